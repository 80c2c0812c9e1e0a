"""Where the end-to-end (host-buffer) step time goes at the metric config:
wall time of fasth_forward_backward_host, the device time of the same call
(CUDA events on its stream), and the pieces: pinned H2D of V/X/G, the
device-resident step, D2H of Y/dX/dV."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch

from paper_2009_13977_b200 import fasth as fb

d, b, m = 784, 32, 32
Vh = torch.randn(d, d).pin_memory()
Xh = torch.randn(m, d).pin_memory()
Gh = torch.randn(m, d).pin_memory()
out = tuple(torch.empty(s).pin_memory() for s in ((m, d), (m, d), (d, d)))
ctx = fb.Context(0)
for _ in range(5):
    fb.forward_backward_host(Vh, Xh, Gh, b, ctx=ctx, out=out)
torch.cuda.synchronize()
K = 50
s = torch.cuda.current_stream()
ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(K)]
t0 = time.perf_counter()
for k in range(K):
    ev[k][0].record(s)
    fb.forward_backward_host(Vh, Xh, Gh, b, ctx=ctx, out=out)
    ev[k][1].record(s)
torch.cuda.synchronize()
wall = (time.perf_counter() - t0) * 1e6 / K
dev_us = sum(a.elapsed_time(b_) for a, b_ in ev) * 1e3 / K


def timed(fn, reps=50):
    a, b_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    fn()
    torch.cuda.synchronize()
    a.record()
    for _ in range(reps):
        fn()
    b_.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b_) * 1e3 / reps


Vd, Xd, Gd = torch.empty(d, d, device="cuda"), torch.empty(m, d, device="cuda"), torch.empty(m, d, device="cuda")
h2d = timed(lambda: (Vd.copy_(Vh, non_blocking=True), Xd.copy_(Xh, non_blocking=True), Gd.copy_(Gh, non_blocking=True)))
d2h = timed(lambda: (out[0].copy_(Xd, non_blocking=True), out[1].copy_(Gd, non_blocking=True), out[2].copy_(Vd, non_blocking=True)))
dctx = fb.Context(0, deferred=True)
comp = timed(lambda: fb.fasth_forward_backward(Vd, Xd.t(), Gd.t(), b, ctx=dctx))
print(json.dumps({"wall_us": round(wall, 1), "device_us": round(dev_us, 1), "h2d_us": round(h2d, 1),
                  "d2h_us": round(d2h, 1), "device_step_eager_us": round(comp, 1)}))
