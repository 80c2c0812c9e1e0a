"""Time the FastH fwd+bwd step for each chain geometry (C CTAs per cluster x
WC columns per cluster) at a given (d, b, m); prints one line per config with
per-kernel device times.  Run on the GPU box."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np
import torch

from paper_2009_13977_b200 import fasth as fb
from oracle.oracle import Port, relative_error


def main(d=784, b=32, m=32, steps=100, clusters=(4, 7, 8, 14, 16), wcs=(8, 16)):
    rng = np.random.default_rng(0)
    V, X, G = rng.standard_normal((d, d)), rng.standard_normal((d, m)), rng.standard_normal((d, m))
    want = Port().fasth_fwd_bwd(V, X, G, b)
    Vd = torch.tensor(V, dtype=torch.float32, device="cuda")
    Xd = torch.tensor(X.T.copy(), dtype=torch.float32, device="cuda").t()
    Gd = torch.tensor(G.T.copy(), dtype=torch.float32, device="cuda").t()
    flush = torch.empty(64 * 1024 * 1024, device="cuda")
    ctx = fb.Context(0, deferred=True)
    s = torch.cuda.Stream()
    for C in clusters:
        for WC in wcs:
            os.environ["FASTH_CLUSTER"], os.environ["FASTH_WC"] = str(C), str(WC)
            try:
                with torch.cuda.stream(s):
                    tape = fb.fasth_forward(Vd, Xd, b, ctx=ctx)
                    back = fb.fasth_backward(tape, Gd)
                torch.cuda.synchronize()
                ctx.check()
                err = max(relative_error(t.double().cpu().numpy(), w) for t, w in
                          zip((tape.output(), back.grad_input, back.grad_vectors), want))
                ctx.set_timing(True)
                with torch.cuda.stream(s):
                    for _ in range(steps):
                        flush.zero_()
                        t2 = fb.fasth_forward(Vd, Xd, b, ctx=ctx)
                        fb.fasth_backward(t2, Gd)
                torch.cuda.synchronize()
                kt = ctx.kernel_times()
                ctx.set_timing(False)
                tot = sum(v[0] for v in kt.values()) * 1e3 / steps
                ks = " ".join(f"{k}={v[0] * 1e3 / v[1]:.1f}" for k, v in sorted(kt.items()))
                print(f"C={C:2d} WC={WC:2d}  kernels {tot:8.1f} us  err {err:.1e}  {ks}", flush=True)
            except Exception as e:
                print(f"C={C:2d} WC={WC:2d}  FAILED {type(e).__name__}: {str(e)[:120]}", flush=True)
                torch.cuda.synchronize()


if __name__ == "__main__":
    args = [int(x) for x in sys.argv[1:]]
    main(*args)
