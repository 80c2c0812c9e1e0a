"""Per-replay overhead of a CUDA graph as bench.py times it (flush, event,
replay, event): an empty-kernel graph vs the metric step's graph."""
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2009_13977_b200 import fasth as fb  # noqa: E402

flush = torch.empty(64 * 1024 * 1024, device="cuda")
s = torch.cuda.Stream()
t = torch.zeros(1, device="cuda")


def timeit(gr, n=200, fl=True):
    ts = []
    with torch.cuda.stream(s):
        for _ in range(n):
            if fl:
                flush.zero_()
            a, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(s)
            gr.replay()
            e.record(s)
            e.synchronize()
            ts.append(a.elapsed_time(e) * 1e3)
    return statistics.median(ts)


g1 = torch.cuda.CUDAGraph()
with torch.cuda.stream(s):
    t.add_(1)
    torch.cuda.synchronize()
    with torch.cuda.graph(g1, stream=s):
        t.add_(1)
g3 = torch.cuda.CUDAGraph()
with torch.cuda.stream(s):
    with torch.cuda.graph(g3, stream=s):
        t.add_(1)
        t.add_(1)
        t.add_(1)
d, m, b = 784, 32, 32
V = torch.randn(d, d, device="cuda")
X = torch.randn(m, d, device="cuda").t()
G = torch.randn(m, d, device="cuda").t()
ctx = fb.Context(0, deferred=True)
outs = (torch.empty(m, d, device="cuda").t(), torch.empty(m, d, device="cuda").t(), torch.empty(d, d, device="cuda"))
with torch.cuda.stream(s):
    for _ in range(3):
        fb.fasth_forward_backward(V, X, G, b, ctx=ctx, out=outs)
torch.cuda.synchronize()
gs = torch.cuda.CUDAGraph()
with torch.cuda.graph(gs, stream=s):
    fb.fasth_forward_backward(V, X, G, b, ctx=ctx, out=outs)
for name, g in (("1 tiny kernel", g1), ("3 tiny kernels", g3), ("metric step", gs)):
    print(f"{name:16s}: flushed {timeit(g):7.2f} us   unflushed {timeit(g, fl=False):7.2f} us")
