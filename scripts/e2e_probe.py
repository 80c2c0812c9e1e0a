"""Where the host-buffer step's time goes (config 1, d=784, m=32, b=32):
device-time of copies alone (eager and inside a CUDA graph), the device step,
and the library's cached-graph replay of the whole host step."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch

from paper_2009_13977_b200 import fasth as fb

d, b, m = 784, 32, 32
Vh, Xh, Gh = torch.randn(d, d).pin_memory(), torch.randn(m, d).pin_memory(), torch.randn(m, d).pin_memory()
out = tuple(torch.empty(s).pin_memory() for s in ((m, d), (m, d), (d, d)))
Vd, Xd, Gd = torch.empty(d, d, device="cuda"), torch.empty(m, d, device="cuda"), torch.empty(m, d, device="cuda")
Yd, dXd, dVd = torch.empty(m, d, device="cuda"), torch.empty(m, d, device="cuda"), torch.empty(d, d, device="cuda")
s = torch.cuda.Stream()


def dev_time(fn, reps=50):
    with torch.cuda.stream(s):
        for _ in range(5):
            fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        for _ in range(reps):
            fn()
        e1.record(s)
        torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e3 / reps


res = {}
res["h2d_V"] = dev_time(lambda: Vd.copy_(Vh, non_blocking=True))
res["h2d_XG"] = dev_time(lambda: (Xd.copy_(Xh, non_blocking=True), Gd.copy_(Gh, non_blocking=True)))
res["d2h_dV"] = dev_time(lambda: out[2].copy_(dVd, non_blocking=True))
res["d2h_YdX"] = dev_time(lambda: (out[0].copy_(Yd, non_blocking=True), out[1].copy_(dXd, non_blocking=True)))


def copies():
    Vd.copy_(Vh, non_blocking=True)
    Xd.copy_(Xh, non_blocking=True)
    Gd.copy_(Gh, non_blocking=True)
    out[0].copy_(Yd, non_blocking=True)
    out[1].copy_(dXd, non_blocking=True)
    out[2].copy_(dVd, non_blocking=True)


res["all_copies_eager"] = dev_time(copies)
g = torch.cuda.CUDAGraph()
with torch.cuda.stream(s):
    copies()
    torch.cuda.synchronize()
    with torch.cuda.graph(g, stream=s):
        copies()
res["all_copies_graph"] = dev_time(g.replay)
ctx = fb.Context(0, deferred=True)
with torch.cuda.stream(s):
    ctx.bind_stream() if hasattr(ctx, "bind_stream") else None
res["device_step_eager"] = dev_time(lambda: fb.fasth_forward_backward(Vd, Xd.t(), Gd.t(), b, ctx=ctx,
                                                                      out=(Yd.t(), dXd.t(), dVd)))
ctx2 = fb.Context(0)
for _ in range(5):
    fb.forward_backward_host(Vh, Xh, Gh, b, ctx=ctx2, out=out)
t0 = time.perf_counter()
for _ in range(50):
    fb.forward_backward_host(Vh, Xh, Gh, b, ctx=ctx2, out=out)
res["host_step_wall"] = (time.perf_counter() - t0) * 1e6 / 50
os.environ["FASTH_HOST_GRAPH"] = "0"
t0 = time.perf_counter()
for _ in range(50):
    fb.forward_backward_host(Vh, Xh, Gh, b, ctx=ctx2, out=out)
res["host_step_wall_eager"] = (time.perf_counter() - t0) * 1e6 / 50
print(json.dumps({k: round(v, 1) for k, v in res.items()}))
