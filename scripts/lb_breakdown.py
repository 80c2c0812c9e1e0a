"""Per-kernel breakdown of the re-blocked path (ctx timing mode, one stream)
for one shape: python scripts/lb_breakdown.py D M"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ["FASTH_LB"] = "1"
os.environ["FASTH_LB_STREAMS"] = "0"
import torch

from paper_2009_13977_b200 import fasth as fb

d, m = int(sys.argv[1]), int(sys.argv[2])
g = torch.Generator(device="cuda").manual_seed(0)
V = torch.randn(d, d, device="cuda", generator=g)
X = torch.randn(m, d, device="cuda", generator=g).t()
G = torch.randn(m, d, device="cuda", generator=g).t()
ctx = fb.Context(0, deferred=True)
for _ in range(3):
    fb.fasth_forward_backward(V, X, G, 32, ctx=ctx)
torch.cuda.synchronize()
ctx.set_timing(True)
R = 5
for _ in range(R):
    fb.fasth_forward_backward(V, X, G, 32, ctx=ctx)
torch.cuda.synchronize()
kt = ctx.kernel_times()
ctx.set_timing(False)
tot = 0
for k, (ms, n) in sorted(kt.items(), key=lambda x: -x[1][0]):
    print(f"{k:28s} {ms * 1e3 / R:9.1f} us/step  ({n // R} launches)")
