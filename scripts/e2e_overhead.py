"""Host-side overhead of the host-buffer entry at the metric config: wall
time per call through the Python mirror (forward_backward_host) vs the bare
ctypes call of fasth_forward_backward_host with prepared arguments, and the
device-side span of one call (CUDA events on the legacy stream around it)."""
import ctypes as C
import json
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2009_13977_b200 import fasth as fb  # noqa: E402

d, b, m = 784, 32, 32
Vh, Xh, Gh = (torch.randn(s).pin_memory() for s in ((d, d), (m, d), (m, d)))
out = tuple(torch.empty(s).pin_memory() for s in ((m, d), (m, d), (d, d)))
ctx = fb.Context(0)
for _ in range(10):
    fb.forward_backward_host(Vh, Xh, Gh, b, ctx=ctx, out=out)
lib = ctx.lib
args = (ctx.h, C.c_void_p(Vh.data_ptr()), d, d, C.c_void_p(Xh.data_ptr()), C.c_void_p(Gh.data_ptr()), m, b,
        C.c_void_p(out[0].data_ptr()), C.c_void_p(out[1].data_ptr()), C.c_void_p(out[2].data_ptr()))
res = {}
for name, fn in (("python_api", lambda: fb.forward_backward_host(Vh, Xh, Gh, b, ctx=ctx, out=out)),
                 ("bare_ctypes", lambda: lib.fasth_forward_backward_host(*args))):
    ts = []
    for _ in range(300):
        t0 = time.perf_counter()
        fn()
        ts.append((time.perf_counter() - t0) * 1e6)
    res[name + "_us"] = round(statistics.median(ts), 1)
ev = []
for _ in range(100):
    a, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    lib.fasth_forward_backward_host(*args)
    e.record()
    e.synchronize()
    ev.append(a.elapsed_time(e) * 1e3)
res["device_span_us"] = round(statistics.median(ev), 1)
print(json.dumps(res))
