"""e2e A/B of the host-buffer step (fasth_forward_backward_host at the metric
config): host wall time per call (median) under env variants, interleaved."""
import json
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2009_13977_b200 import fasth as fb  # noqa: E402

d, b, m = 784, 32, 32
variants = sys.argv[1:] or ["base"]
Vh, Xh, Gh = (torch.randn(s).pin_memory() for s in ((d, d), (m, d), (m, d)))
outs = {}
ctxs = {}


def env_of(v):
    return {} if v == "base" else dict(kv.split("=", 1) for kv in v.split(","))


def call(v):
    env = env_of(v)
    old = {k: os.environ.get(k) for k in env}
    os.environ.update(env)
    try:
        t0 = time.perf_counter()
        fb.forward_backward_host(Vh, Xh, Gh, b, ctx=ctxs[v], out=outs[v])
        return time.perf_counter() - t0
    finally:
        for k, val in old.items():
            if val is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = val


for v in variants:
    ctxs[v] = fb.Context(0)
    outs[v] = tuple(torch.empty(s).pin_memory() for s in ((m, d), (m, d), (d, d)))
    for _ in range(5):
        call(v)
ref = outs[variants[0]]
times = {v: [] for v in variants}
for _ in range(int(os.environ.get("E2E_ROUNDS", 6))):
    for v in variants:
        for _ in range(30):
            times[v].append(call(v) * 1e6)
for v in variants:
    err = max(float((a - r).norm() / r.norm()) for a, r in zip(outs[v], ref))
    print(json.dumps({"variant": v, "median_us": round(statistics.median(times[v]), 1),
                      "p10_us": round(sorted(times[v])[len(times[v]) // 10], 1), "vs_first_maxrel": err}), flush=True)
