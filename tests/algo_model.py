"""numpy model of the exact arithmetic the CUDA kernels perform (test-only).

It restates, in f64, the device algorithm of paper_2009_13977_b200/csrc:
  * wy_build2.cu : T~ = (diag(V^T V) + 2 striu(V^T V))^{-1} on RAW vectors
  * chain_v2.cu  : Z = V^T X ; Z' = T~ Z (fwd) / T~^T Z (bwd) ; X -= 2 V Z'
  * dv2.cu       : dV = -2 (A Z'b^T + G Z'f^T + 2 V striu(Q - Q^T)), Q = Z'f Z'b^T
so the CPU suite can check the kernels' closed forms against the reference
oracle without a GPU (the GPU suite then checks the kernels themselves).
"""
import numpy as np


def blocks(n, b, cap=64):
    b = min(max(b, 1), n)
    b = min(b, cap)  # wider blocks run as 64-wide sub-blocks (chain kernels)
    return [(lo, min(lo + b, n)) for lo in range(0, n, b)]


def t_tilde(Vb):
    """Vb: d x w raw block (columns = vectors)."""
    G = Vb.T @ Vb
    M = np.diag(np.diag(G)) + 2 * np.triu(G, 1)
    return np.linalg.inv(M)


def fwd_bwd(V, X, Gout, b, cap=64):
    """V: (n, d) chain, X, Gout: (d, m).  Returns Y, dX, dV (n, d).
    cap: widest block run as one (64 = the chain kernels; the large-batch path
    of csrc/lb_*.cu runs 128/256/512-wide blocks: cap=None)."""
    n, d = V.shape
    Vt = V.T
    bl = blocks(n, b, cap if cap else n)
    Ts = [t_tilde(Vt[:, lo:hi]) for lo, hi in bl]
    # forward sweep, recording activations A_i (block output) and Z'f
    A = X.copy()
    acts, zf = [None] * len(bl), [None] * len(bl)
    for i in reversed(range(len(bl))):
        lo, hi = bl[i]
        Vb = Vt[:, lo:hi]
        Zp = Ts[i] @ (Vb.T @ A)
        A = A - 2 * Vb @ Zp
        acts[i], zf[i] = A.copy(), Zp
    Y = A
    # backward sweep
    Gs = Gout.copy()
    dV = np.zeros_like(V)
    for i in range(len(bl)):
        lo, hi = bl[i]
        Vb = Vt[:, lo:hi]
        Zb = Ts[i].T @ (Vb.T @ Gs)
        Q = zf[i] @ Zb.T
        Kp = np.triu(Q - Q.T, 1)
        dV[lo:hi] = (-2 * (acts[i] @ Zb.T + Gs @ zf[i].T + 2 * Vb @ Kp)).T
        Gs = Gs - 2 * Vb @ Zb
    return Y, Gs, dV
