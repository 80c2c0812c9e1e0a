"""Config 2 as the layer (svd_forward_backward, d = 784, b = 32, batch 32):
eager back-to-back steps (bench.py's config2_layer timing) vs a CUDA graph
of the step replayed back to back and with an L2 flush between steps."""
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2009_13977_b200 import fasth as fb  # noqa: E402

d, b, m = 784, 32, 32
g = torch.Generator(device="cuda").manual_seed(0)
U = torch.randn(d, d, device="cuda", generator=g)
V = torch.randn(d, d, device="cuda", generator=g)
U /= U.norm(dim=1, keepdim=True)
V /= V.norm(dim=1, keepdim=True)
s = torch.rand(d, device="cuda", generator=g) * 1.5 + 0.5
X = torch.randn(m, d, device="cuda", generator=g).t()
G = torch.randn(m, d, device="cuda", generator=g).t()
p = fb.SvdParam(d, d, U, V, s)
ctx = fb.Context(0, deferred=True)
st = torch.cuda.Stream()
flush = torch.empty(64 * 1024 * 1024, device="cuda")


def step():
    return fb.svd_forward_backward(p, X, G, b, ctx=ctx)


with torch.cuda.stream(st):
    for _ in range(5):
        step()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
with torch.cuda.stream(st):
    e0.record(st)
    for _ in range(50):
        step()
    e1.record(st)
torch.cuda.synchronize()
print(f"eager back to back: {e0.elapsed_time(e1) * 1e3 / 50:7.2f} us/step")
gr = torch.cuda.CUDAGraph()
try:
    with torch.cuda.graph(gr, stream=st):
        out = step()
    with torch.cuda.stream(st):
        e0.record(st)
        for _ in range(50):
            gr.replay()
        e1.record(st)
    torch.cuda.synchronize()
    print(f"graph back to back: {e0.elapsed_time(e1) * 1e3 / 50:7.2f} us/step")
    ts = []
    with torch.cuda.stream(st):
        for _ in range(100):
            flush.zero_()
            a, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(st)
            gr.replay()
            e.record(st)
            e.synchronize()
            ts.append(a.elapsed_time(e) * 1e3)
    print(f"graph flushed single: median {statistics.median(ts):7.2f} us")
except Exception as ex:  # noqa: BLE001
    print("graph capture failed:", ex)
ctx.check()
# per-kernel CUDA-event windows (timing mode: launches serialised by the events)
ctx.set_timing(True)
with torch.cuda.stream(st):
    for _ in range(20):
        step()
torch.cuda.synchronize()
kt = ctx.kernel_times()
ctx.set_timing(False)
for k, (ms, n) in sorted(kt.items(), key=lambda kv: -kv[1][0]):
    print(f"  {k:28s} {1e3 * ms / 20:8.2f} us/step  ({n // 20} launches/step)")
