"""A/B probe: device time of the metric-config step (graph replay, L2
flushed, CUDA events) under environment-knob variants given on the command
line, e.g.  python scripts/step_env.py base FASTH_PIPELINE=1 FASTH_PIPELINE=1,FASTH_BUILDERS=20
Variants are interleaved over several rounds (box noise); prints medians."""
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2009_13977_b200 import fasth as fb  # noqa: E402

d = int(os.environ.get("STEP_D", 784))
m = int(os.environ.get("STEP_M", 32))
b = int(os.environ.get("STEP_B", 32))
two_call = os.environ.get("STEP_TWO_CALL", "0") == "1"
variants = sys.argv[1:] or ["base"]
g = torch.Generator(device="cuda").manual_seed(0)
V = torch.randn(d, d, device="cuda", generator=g)
X = torch.randn(m, d, device="cuda", generator=g).t()
G = torch.randn(m, d, device="cuda", generator=g).t()
flush = torch.empty(64 * 1024 * 1024, device="cuda")
ref = None


def env_of(v):
    return {} if v == "base" else dict(kv.split("=", 1) for kv in v.split(","))


graphs = {}
fine = {}
REP = int(os.environ.get("STEP_REP", 10))
for v in variants:
    env = env_of(v)
    old = {k: os.environ.get(k) for k in env}
    os.environ.update(env)
    ctx = fb.Context(0, deferred=True)
    outs = (torch.empty(m, d, device="cuda").t(), torch.empty(m, d, device="cuda").t(),
            torch.empty(d, d, device="cuda"))
    s = torch.cuda.Stream()

    def fn():
        if two_call:
            t = fb.fasth_forward(V, X, b, ctx=ctx, out=outs[0])
            r = fb.fasth_backward(t, G)
            return r
        if env.get("NODV"):  # step option, not a library knob: no gradient kernel
            return fb.fasth_forward_backward(V, X, G, b, ctx=ctx, out=(outs[0], outs[1], None))
        return fb.fasth_forward_backward(V, X, G, b, ctx=ctx, out=outs)
    try:
        with torch.cuda.stream(s):
            for _ in range(3):
                fn()
        torch.cuda.synchronize()
        ctx.check()
        gr = torch.cuda.CUDAGraph()
        with torch.cuda.graph(gr, stream=s):
            keep = fn()
        torch.cuda.synchronize()
        gr.replay()
        torch.cuda.synchronize()
        # finer resolution: REP x (flush + step) in one graph, minus REP flushes
        g10 = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g10, stream=s):
            for _ in range(REP):
                flush.zero_()
                keep10 = fn()
        torch.cuda.synchronize()
        fine[v] = g10
    except Exception as e:  # noqa: BLE001
        print(json.dumps({"variant": v, "error": str(e)[:200]}), flush=True)
        for k, val in old.items():
            if val is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = val
        continue
    if ref is None:
        ref = [t.clone() for t in outs]
    err = max(float((a - r_).norm() / r_.norm()) for a, r_ in zip(outs, ref))
    graphs[v] = (gr, s, ctx, keep, err)
    for k, val in old.items():
        if val is None:
            os.environ.pop(k, None)
        else:
            os.environ[k] = val

variants = [v for v in variants if v in graphs]
times = {v: [] for v in variants}
for rnd in range(int(os.environ.get("STEP_ROUNDS", 5))):
    for v in variants:
        gr, s, _, _, _ = graphs[v]
        with torch.cuda.stream(s):
            for i in range(40):
                flush.zero_()
                a, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(s)
                gr.replay()
                e.record(s)
                e.synchronize()
                times[v].append(a.elapsed_time(e) * 1e3)
gfl = torch.cuda.CUDAGraph()
sf = torch.cuda.Stream()
with torch.cuda.graph(gfl, stream=sf):
    for _ in range(REP):
        flush.zero_()
torch.cuda.synchronize()


def time_graph(g, st, n=20):
    ts = []
    with torch.cuda.stream(st):
        for _ in range(n):
            a, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(st)
            g.replay()
            e.record(st)
            e.synchronize()
            ts.append(a.elapsed_time(e) * 1e3)
    return statistics.median(ts)


fine_us = {}
for rnd in range(3):
    tf = time_graph(gfl, sf)
    for v in variants:
        fine_us.setdefault(v, []).append((time_graph(fine[v], graphs[v][1]) - tf) / REP)
for v in variants:
    ts = sorted(times[v])
    print(json.dumps({"variant": v, "d": d, "m": m, "b": b, "two_call": two_call, "median_us": statistics.median(ts),
                      "p10_us": ts[len(ts) // 10], "fine_us": round(statistics.median(fine_us[v]), 2), "vs_first_variant_maxrel": graphs[v][4]}), flush=True)
