"""Per-kernel device times of one fasth_forward_backward step (d, b, m from
argv; default the metric config) for each first/second-generation kernel
choice (KT_VARIANTS: comma-separated env knobs set to 1): the step is captured
into a CUDA graph with the context's event timing on (mode 2), replayed with
an L2 flush before each replay, and the per-kernel event times averaged.
Prints one JSON line per variant."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch

from paper_2009_13977_b200 import fasth as fb


def graph_kernel_times(ctx, fn, reps=30, flush=None):
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        for _ in range(3):
            fn()
    torch.cuda.synchronize()
    ctx.set_timing(True, graph=True)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        fn()
    torch.cuda.synchronize()
    tot = 0.0
    with torch.cuda.stream(s):
        for _ in range(reps):
            if flush is not None:
                flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(s)
            g.replay()
            b.record(s)
            b.synchronize()
            tot += a.elapsed_time(b)
            ctx.kernel_times()  # accumulate this replay (collect reads and keeps the events)
    kt = ctx.kernel_times()
    del g
    torch.cuda.synchronize()
    ctx.set_timing(False)
    return tot * 1e3 / reps, {k: round(v[0] * 1e3 / v[1], 2) for k, v in kt.items()}


if __name__ == "__main__":
    d, b, m = (int(x) for x in (sys.argv[1:4] if len(sys.argv) > 3 else (784, 32, 32)))
    V = torch.randn(d, d, device="cuda")
    X = torch.randn(m, d, device="cuda").t()
    G = torch.randn(m, d, device="cuda").t()
    flush = torch.empty(64 * 1024 * 1024, device="cuda")
    variants = os.environ.get("KT_VARIANTS", ",FASTH_PIPELINE,FASTH_NO_PDL").split(",")
    for variant in variants:
        if variant:
            os.environ[variant] = "1"
        ctx = fb.Context(0, deferred=True)
        outs = (torch.empty(m, d, device="cuda").t(), torch.empty(m, d, device="cuda").t(),
                torch.empty(d, d, device="cuda"))
        step_us, kt = graph_kernel_times(ctx, lambda: fb.fasth_forward_backward(V, X, G, b, ctx=ctx, out=outs),
                                         flush=flush)
        ctx.check()
        print(json.dumps({"variant": variant or "v2", "d": d, "b": b, "m": m, "step_us": round(step_us, 2),
                          "kernel_us": kt}), flush=True)
        if variant:
            del os.environ[variant]
