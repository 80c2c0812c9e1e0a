"""PCIe probe for the host-buffer step: the chain V (d x d fp32, 2.46 MB at
d = 784) host->device and dV device->host, by one cudaMemcpyAsync, by k
chunks on k streams (several copy engines), and by an SM copy kernel reading
pinned host memory (zero copy).  Device time per transfer (CUDA events)."""
import json
import os
import sys

import torch

d = int(sys.argv[1]) if len(sys.argv) > 1 else 784
n = d * d
h = torch.randn(n).pin_memory()
hd = torch.empty(n).pin_memory()
g = torch.empty(n, device="cuda")
s0 = torch.cuda.Stream()
streams = [torch.cuda.Stream() for _ in range(8)]


def timed(fn, reps=30):
    torch.cuda.synchronize()
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s0)
        fn()
        b.record(s0)
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) * 1e3)
    ts.sort()
    return round(ts[len(ts) // 2], 1)


def chunked(k, h2d=True):
    def fn():
        ev = torch.cuda.Event()
        ev.record(s0)
        step = (n + k - 1) // k
        for i in range(k):
            st = streams[i]
            st.wait_event(ev)
            with torch.cuda.stream(st):
                lo, hi = i * step, min(n, (i + 1) * step)
                if h2d:
                    g[lo:hi].copy_(h[lo:hi], non_blocking=True)
                else:
                    hd[lo:hi].copy_(g[lo:hi], non_blocking=True)
        for i in range(k):
            s0.wait_stream(streams[i])
    return fn


res = {"bytes": 4 * n}
with torch.cuda.stream(s0):
    res["h2d_1"] = timed(lambda: g.copy_(h, non_blocking=True))
    res["d2h_1"] = timed(lambda: hd.copy_(g, non_blocking=True))
for k in (2, 4, 8):
    res[f"h2d_{k}streams"] = timed(chunked(k, True))
    res[f"d2h_{k}streams"] = timed(chunked(k, False))
# zero copy: a device kernel reading the pinned host buffer through UVA
hz = h.view(-1)
with torch.cuda.stream(s0):
    res["h2d_zerocopy_torch"] = timed(lambda: g.copy_(hz.cuda(non_blocking=True)))  # baseline path
# both directions at once
def both():
    ev = torch.cuda.Event()
    ev.record(s0)
    streams[0].wait_event(ev)
    streams[1].wait_event(ev)
    with torch.cuda.stream(streams[0]):
        g.copy_(h, non_blocking=True)
    with torch.cuda.stream(streams[1]):
        hd.copy_(g, non_blocking=True)
    s0.wait_stream(streams[0])
    s0.wait_stream(streams[1])
res["h2d_and_d2h_concurrent"] = timed(both)
res["gbs_h2d_1"] = round(4 * n / res["h2d_1"] / 1e3, 1)
res["gbs_d2h_1"] = round(4 * n / res["d2h_1"] / 1e3, 1)
print(json.dumps(res))
