"""Run the metric-config fused step a few times as a CUDA graph (L2 flushed)
with FASTH_STEPTRACE set, then dump the last replay's timeline.
STEP_TWO_CALL=1: the fasth_forward + fasth_backward step instead (the trace
then shows the backward sweep and the gradient kernel)."""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2009_13977_b200 import fasth as fb  # noqa: E402

d, m, b = (int(x) for x in (sys.argv[1:4] if len(sys.argv) > 3 else (784, 32, 32)))
g = torch.Generator(device="cuda").manual_seed(0)
V = torch.randn(d, d, device="cuda", generator=g)
X = torch.randn(m, d, device="cuda", generator=g).t()
G = torch.randn(m, d, device="cuda", generator=g).t()
flush = torch.empty(64 * 1024 * 1024, device="cuda")
ctx = fb.Context(0, deferred=True)
outs = (torch.empty(m, d, device="cuda").t(), torch.empty(m, d, device="cuda").t(), torch.empty(d, d, device="cuda"))
s = torch.cuda.Stream()
two_call = os.environ.get("STEP_TWO_CALL", "0") == "1"


def step():
    if two_call:
        t = fb.fasth_forward(V, X, b, ctx=ctx, out=outs[0])
        return fb.fasth_backward(t, G)
    return fb.fasth_forward_backward(V, X, G, b, ctx=ctx, out=outs)


with torch.cuda.stream(s):
    for _ in range(3):
        step()
torch.cuda.synchronize()
gr = torch.cuda.CUDAGraph()
with torch.cuda.graph(gr, stream=s):
    step()
with torch.cuda.stream(s):
    for _ in range(5):
        flush.zero_()
        gr.replay()
torch.cuda.synchronize()
ctx.check()
path = os.environ["FASTH_STEPTRACE"] + ".bin"
print(subprocess.run([sys.executable, os.path.join(ROOT, "scripts", "step_timeline.py"), path],
                     capture_output=True, text=True).stdout)
