"""SVD layer fwd+bwd (svd_forward_backward) timing at large batch: the
large-batch tcgen05 legs (FASTH_LB=1) against the chain kernels (FASTH_LB=0).

    python scripts/svd_lb_probe.py  -> one JSON line per (d, m, path)"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch

from paper_2009_13977_b200 import fasth as fb


def run(d, m, lb, steps=5):
    os.environ["FASTH_LB"] = "1" if lb else "0"
    g = torch.Generator(device="cuda").manual_seed(0)
    U = torch.randn(d, d, device="cuda", generator=g)
    V = torch.randn(d, d, device="cuda", generator=g)
    s = torch.rand(d, device="cuda", generator=g) + 0.5
    X = torch.randn(m, d, device="cuda", generator=g).t()
    G = torch.randn(m, d, device="cuda", generator=g).t()
    p = fb.SvdParam(d, d, U, V, s)
    ctx = fb.Context(0, deferred=True)
    for _ in range(2):
        fb.svd_forward_backward(p, X, G, 32, ctx=ctx)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        fb.svd_forward_backward(p, X, G, 32, ctx=ctx)
    e1.record()
    torch.cuda.synchronize()
    ctx.check()
    ms = e0.elapsed_time(e1) / steps
    flops = 2 * (12.0 * d * d * m)  # two chains, fwd+bwd
    return {"d": d, "m": m, "path": "large-batch" if lb else "chain", "ms": ms, "tflops": flops / ms / 1e9}




def breakdown(d=2048, m=8192):
    """Per-kernel device times of one large-batch layer step (timing mode)."""
    os.environ["FASTH_LB"] = "1"
    os.environ["FASTH_LB_STREAMS"] = "0"
    g = torch.Generator(device="cuda").manual_seed(0)
    p = fb.SvdParam(d, d, torch.randn(d, d, device="cuda", generator=g), torch.randn(d, d, device="cuda", generator=g),
                    torch.rand(d, device="cuda", generator=g) + 0.5)
    X = torch.randn(m, d, device="cuda", generator=g).t()
    G = torch.randn(m, d, device="cuda", generator=g).t()
    ctx = fb.Context(0, deferred=True)
    fb.svd_forward_backward(p, X, G, 32, ctx=ctx)
    ctx.set_timing(True)
    for _ in range(3):
        fb.svd_forward_backward(p, X, G, 32, ctx=ctx)
    torch.cuda.synchronize()
    kt = ctx.kernel_times()
    ctx.set_timing(False)
    tot = sum(v[0] for v in kt.values()) / 3
    rows = sorted(((k, v[0] / 3, v[1] / 3) for k, v in kt.items()), key=lambda r: -r[1])
    print(json.dumps({"d": d, "m": m, "sum_ms": tot, "kernels": {k: [round(ms, 4), n] for k, ms, n in rows}}))


if __name__ == "__main__":
    if "--breakdown" in sys.argv:
        breakdown()
    else:
        for d, m in ((1024, 4096), (2048, 8192), (2048, 2048), (1024, 1024)):
            for lb in (True, False):
                print(json.dumps(run(d, m, lb)), flush=True)
