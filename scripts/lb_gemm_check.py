"""tcgen05 3xTF32 GEMM (large-batch path) check + timing on cuda:0.

    python scripts/lb_gemm_check.py [--time]

Each case: D = alpha A B^T (+ beta C) against a float64 torch product; prints
max relative (Frobenius) error per output, then (with --time) TFLOP/s of the
hook's GEMM launch alone for the large-batch step's shapes."""
import argparse
import ctypes as C
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch

from paper_2009_13977_b200 import _lib

lib = _lib.load()
f = lib.fasthb_lb_gemm_test
P, I64, I, F = C.c_void_p, C.c_int64, C.c_int, C.c_float
f.argtypes = [P, I64, P, I64, I, I, I, I, P, I64, F, F, P, I64, P, P, I64, P, P, I64, P, I, I]
f.restype = I


def ptr(t):
    return C.c_void_p(t.data_ptr()) if t is not None else None


def run(M, N, K, b_mn, alpha=1.0, beta=0.0, with_c=False, trans=False, ksplit=1, swap=0, seed=0):
    g = torch.Generator(device="cuda").manual_seed(seed)
    A = torch.randn(M, K, device="cuda", generator=g)
    B = torch.randn(K, N, device="cuda", generator=g) if b_mn else torch.randn(N, K, device="cuda", generator=g)
    Cm = torch.randn(M, N, device="cuda", generator=g) if with_c else None
    Bt = B if b_mn else B.t()
    ref = alpha * (A.double() @ Bt.double())
    if with_c:
        ref = ref + beta * Cm.double()
    D = torch.zeros(M, N, device="cuda")
    Dh, Dl = torch.zeros(M, N, device="cuda"), torch.zeros(M, N, device="cuda")
    Th = Tl = None
    if trans:
        Th, Tl = torch.zeros(N, M, device="cuda"), torch.zeros(N, M, device="cuda")
    part = torch.zeros(ksplit, M, N, device="cuda") if ksplit > 1 else None
    rc = f(ptr(A), K, ptr(B), N if b_mn else K, int(b_mn), M, N, K, ptr(Cm), N, alpha, beta,
           None if part is not None else ptr(D), N, None if part is not None else ptr(Dh),
           None if part is not None else ptr(Dl), N, ptr(Th), ptr(Tl), M, ptr(part), ksplit, swap)
    torch.cuda.synchronize()
    out = {"M": M, "N": N, "K": K, "b_mn": b_mn, "beta": beta, "ksplit": ksplit, "swap": swap, "rc": rc}
    rel = lambda x: float((x.double() - ref).norm() / ref.norm())
    if part is not None:
        out["err_partial"] = rel(part.sum(0))
    else:
        out["err_f32"] = rel(D)
        out["err_split"] = rel(Dh.double() + Dl.double())
        if trans:
            out["err_T"] = rel((Th.double() + Tl.double()).t())
    return out


def timed(M, N, K, b_mn, reps=20):
    import time
    A = torch.randn(M, K, device="cuda")
    B = torch.randn(K, N, device="cuda") if b_mn else torch.randn(N, K, device="cuda")
    D = torch.empty(M, N, device="cuda")
    # the hook splits + allocates each call; time it with events around many calls and
    # subtract nothing: report the hook total and the GEMM via the profiler separately
    args = lambda: f(ptr(A), K, ptr(B), N if b_mn else K, int(b_mn), M, N, K, None, N, 1.0, 0.0, ptr(D), N,
                     None, None, N, None, None, M, None, 1, 0)
    args()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        args()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    return {"M": M, "N": N, "K": K, "b_mn": b_mn, "hook_ms": ms, "tflops_hook": 2 * M * N * K / ms / 1e9}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--time", action="store_true")
    a = ap.parse_args()
    cases = [
        dict(M=128, N=256, K=32, b_mn=False),
        dict(M=128, N=256, K=64, b_mn=False),
        dict(M=256, N=512, K=256, b_mn=False),
        dict(M=200, N=300, K=100, b_mn=False),
        dict(M=128, N=256, K=32, b_mn=True),
        dict(M=128, N=256, K=32, b_mn=True, swap=1),
        dict(M=256, N=512, K=256, b_mn=True),
        dict(M=256, N=512, K=256, b_mn=True, swap=1),
        dict(M=512, N=1024, K=512, b_mn=False, alpha=-2.0, beta=1.0, with_c=True),
        dict(M=512, N=512, K=384, b_mn=False, trans=True),
        dict(M=512, N=512, K=2048, b_mn=False, ksplit=8),
        dict(M=512, N=1024, K=2048, b_mn=True, ksplit=4),
        dict(M=1000, N=1000, K=1000, b_mn=False),
        # M >= 1024: CTA-pair (cta_group::2) tiles
        dict(M=1024, N=512, K=256, b_mn=False),
        dict(M=1024, N=512, K=256, b_mn=True),
        dict(M=2048, N=768, K=96, b_mn=False, alpha=-2.0, beta=1.0, with_c=True),
        dict(M=1100, N=300, K=200, b_mn=False, trans=True),
        dict(M=1024, N=1024, K=2048, b_mn=True, ksplit=4),
        dict(M=8192, N=512, K=2048, b_mn=False),
    ]
    for c in cases:
        try:
            print(json.dumps(run(**c)), flush=True)
        except Exception as e:  # noqa: BLE001
            print(json.dumps({"case": c, "error": str(e)}), flush=True)
    if a.time:
        for M, N, K, mn in ((8192, 2048, 512, False), (8192, 512, 2048, False), (512, 2048, 8192, True),
                            (8192, 8192, 2048, False)):
            print(json.dumps(timed(M, N, K, mn)), flush=True)


if __name__ == "__main__":
    main()
