"""Config 3 shapes (batch 32): the chain kernels vs the re-blocked tcgen05
path with split-K (FASTH_LB=1), device µs per fused fwd+bwd step + parity
against the float64 model."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch

from paper_2009_13977_b200 import fasth as fb
from tests.test_gpu_lb import model64, rel


def timed(fn, reps=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e3 / reps


SHAPES = [tuple(map(int, a.split('x'))) for a in sys.argv[1:]] or [(1024, 32), (2048, 32), (4096, 32), (2048, 256), (4096, 128)]
for d, m in SHAPES:
    g = torch.Generator(device="cuda").manual_seed(d + m)
    V = torch.randn(d, d, device="cuda", generator=g)
    X = torch.randn(m, d, device="cuda", generator=g).t()
    G = torch.randn(m, d, device="cuda", generator=g).t()
    ctx = fb.Context(0, deferred=True)
    res = {"d": d, "m": m}
    for lb in ("0", "1"):
        os.environ["FASTH_LB"] = lb
        try:
            res[f"us_lb{lb}"] = timed(lambda: fb.fasth_forward_backward(V, X, G, 32, ctx=ctx))
            Y, back = fb.fasth_forward_backward(V, X, G, 32, ctx=ctx)
            torch.cuda.synchronize()
            if d <= 2048 and os.environ.get('PROBE_PARITY', '1') == '1':
                Yr, dXr, dVr = model64(V, X, G, 64)
                res[f"err_lb{lb}"] = max(rel(Y, Yr), rel(back.grad_input, dXr), rel(back.grad_vectors, dVr))
        except Exception as e:  # noqa: BLE001
            res[f"err_lb{lb}"] = str(e)[:100]
    print(json.dumps(res), flush=True)
