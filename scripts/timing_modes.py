"""The metric step timed as bench.py does (flush, event, step, event; median
over steps) with the step issued three ways: CUDA graph replay, eager calls
of the C ABI entry, and a graph whose replay is preceded by the flush inside
the same graph (event pair around the step nodes only is not possible: the
events here bracket flush + step, then the flush alone is subtracted)."""
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2009_13977_b200 import fasth as fb  # noqa: E402

d, m, b = 784, 32, 32
g = torch.Generator(device="cuda").manual_seed(0)
V = torch.randn(d, d, device="cuda", generator=g)
X = torch.randn(m, d, device="cuda", generator=g).t()
G = torch.randn(m, d, device="cuda", generator=g).t()
flush = torch.empty(64 * 1024 * 1024, device="cuda")
ctx = fb.Context(0, deferred=True)
outs = (torch.empty(m, d, device="cuda").t(), torch.empty(m, d, device="cuda").t(), torch.empty(d, d, device="cuda"))
s = torch.cuda.Stream()


def step():
    fb.fasth_forward_backward(V, X, G, b, ctx=ctx, out=outs)


with torch.cuda.stream(s):
    for _ in range(5):
        step()
torch.cuda.synchronize()
gr = torch.cuda.CUDAGraph()
with torch.cuda.graph(gr, stream=s):
    step()


def med(fn, n=300):
    ts = []
    with torch.cuda.stream(s):
        for _ in range(n):
            flush.zero_()
            a, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(s)
            fn()
            e.record(s)
            e.synchronize()
            ts.append(a.elapsed_time(e) * 1e3)
    return statistics.median(ts), min(ts)


for name, fn in (("graph replay", gr.replay), ("eager C ABI", step), ("graph replay", gr.replay), ("eager C ABI", step)):
    md, mn = med(fn)
    print(f"{name:14s}: median {md:7.2f} us  min {mn:7.2f} us")
ctx.check()
