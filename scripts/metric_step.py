"""Runs the metric-config step (d = n = 784, b = 32, m = 32) a few times:
the target of the ncu captures in profiles/ (kernel filters -k build2 /
sweep2 / dv2)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2009_13977_b200 import fasth as fb  # noqa: E402

d, b, m = (int(x) for x in (sys.argv[1:4] if len(sys.argv) > 3 else (784, 32, 32)))
reps = int(os.environ.get("STEP_REPS", 4))
g = torch.Generator(device="cuda").manual_seed(0)
V = torch.randn(d, d, device="cuda", generator=g)
X = torch.randn(m, d, device="cuda", generator=g).t()
G = torch.randn(m, d, device="cuda", generator=g).t()
ctx = fb.Context(0, deferred=True)
for _ in range(reps):
    fb.fasth_forward_backward(V, X, G, b, ctx=ctx)
torch.cuda.synchronize()
ctx.check()
print("ok")
