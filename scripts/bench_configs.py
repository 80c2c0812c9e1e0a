"""Secondary BASELINE.json configurations on one B200 (bench.py measures the
headline config 2).  Device time per call via CUDA graph replay with the L2
flushed before every replay; prints one JSON line per measurement.

  config 1  FastH fwd+bwd, d = 64, b = 8, batch 32
  config 3  FastH fwd+bwd d sweep (256 .. 4096, b = 32 / 64, batch 32), and
            the reference's exp / Cayley "paths" at the same sizes: the
            SVD-form layer with f(sigma) timed as a full layer fwd+bwd
            (bench.hpp:166-209, op = exp / cayley)
  config 4  depth-4 MLP of d = 784 SVD layers, one full training step
            (paper_2009_13977_b200/mlp.py)

With --cpu every config-3 line also carries the reference's own CPU time for
the same op / d / b / batch (oracle/_ref = the unmodified reference compiled
here: bench::run_bench, algo fasth, all host threads, bench.hpp:166-209) and
the GPU speed-up over it.

Usage: python scripts/bench_configs.py [--quick] [--cpu]
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch

from paper_2009_13977_b200 import fasth as fb
from paper_2009_13977_b200 import mlp

FLUSH = None


def timed_graph(fn, reps=50, warm=5):
    """Capture fn() once into a CUDA graph, replay with L2 flushed; device µs."""
    global FLUSH
    if FLUSH is None:
        FLUSH = torch.empty(64 * 1024 * 1024, device="cuda")
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        for _ in range(warm):
            keep = fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        keep = fn()
    tot = 0.0
    with torch.cuda.stream(s):
        for _ in range(reps):
            FLUSH.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(s)
            g.replay()
            b.record(s)
            b.synchronize()
            tot += a.elapsed_time(b)
    del keep
    return tot * 1e3 / reps


def fwd_bwd_us(d, b, m, ctx):
    V = torch.randn(d, d, device="cuda")
    X = torch.randn(m, d, device="cuda").t()
    G = torch.randn(m, d, device="cuda").t()

    def step():
        t = fb.fasth_forward(V, X, b, ctx=ctx)
        return t, fb.fasth_backward(t, G)
    return timed_graph(step)


def layer_us(d, b, m, ctx, kind):
    """op = exp / cayley / layer: derived SVD-form parameter, layer fwd+bwd."""
    U = torch.randn(d, d, device="cuda")
    U /= U.norm(dim=1, keepdim=True)
    s = torch.rand(d, device="cuda") * 1.8 - 0.9
    f = {"exp": torch.exp(s), "cayley": (1 - s) / (1 + s), "layer": s.abs() + 0.5}[kind]
    p = fb.SvdParam(d, d, U, U.clone(), f)  # symmetric form U f(Sigma) U^T as bench.hpp:179-185
    X = torch.randn(m, d, device="cuda").t()
    G = torch.randn(m, d, device="cuda").t()

    def step():  # G drawn up front (bench.hpp:166-209): the paired-sweep layer call
        return fb.svd_forward_backward(p, X, G, b, ctx=ctx)
    return timed_graph(step)


def cpu_reference(op, d, b, m):
    """bench::run_bench (bench.hpp:225) for one op on all host threads:
    (mean us, reps, cores, -march of the build)."""
    from oracle.oracle import Ref
    R = Ref()
    reps = 10 if d <= 512 else 5 if d <= 1024 else 2 if d <= 2048 else 1
    R.run_bench(op, "fasth", d, m, b, 1, 0, 0)  # warm-up
    mean, _, _ = R.run_bench(op, "fasth", d, m, b, reps, 0, 0)
    return mean * 1e6, reps, R.hardware_threads(), R.march


def main():
    quick = "--quick" in sys.argv
    with_cpu = "--cpu" in sys.argv
    ctx = fb.Context(0, deferred=True)
    out = []

    def emit(rec):
        if with_cpu and rec.get("config") == 3 and "us" in rec:
            cu, reps, cores, march = cpu_reference(rec["op"], rec["d"], rec["b"], rec["batch"])
            rec.update({"cpu_reference_us": cu, "gpu_speedup": cu / rec["us"],
                        "cpu_sample": f"run_bench op={rec['op']} algo=fasth, {reps} reps, {cores} threads, "
                                      f"-march={march}"})
        print(json.dumps(rec), flush=True)
        out.append(rec)

    us = fwd_bwd_us(64, 8, 32, ctx)
    emit({"config": 1, "op": "mul", "d": 64, "b": 8, "batch": 32, "us": us,
          "tflops": (12 * 64 * 64 * 32 + 4 * 64 * 64 * 8) / us / 1e6})
    dims = [256, 512, 1024, 2048] if quick else [256, 512, 1024, 2048, 3072, 4096]
    for d in dims:
        for b in (32, 64):
            try:
                us = fwd_bwd_us(d, b, 32, ctx)
                emit({"config": 3, "op": "mul", "d": d, "b": b, "batch": 32, "us": us,
                      "tflops": (12.0 * d * d * 32 + 4.0 * d * d * b) / us / 1e6})
            except Exception as e:
                emit({"config": 3, "op": "mul", "d": d, "b": b, "error": str(e)[:200]})
        for kind in ("exp", "cayley"):
            try:
                us = layer_us(d, 32, 32, ctx, kind)
                emit({"config": 3, "op": kind, "d": d, "b": 32, "batch": 32, "us": us,
                      "tflops": 2 * (12.0 * d * d * 32 + 4.0 * d * d * 32) / us / 1e6})
            except Exception as e:
                emit({"config": 3, "op": kind, "d": d, "error": str(e)[:200]})
    cfg = mlp.MLPConfig(d=784, depth=4, block_width=32)
    layers = mlp.random_layers(cfg, seed=0)
    x = torch.randn(32, 784, device="cuda").t()
    tgt = torch.randn(32, 784, device="cuda").t()
    us = timed_graph(lambda: mlp.train_step(layers, x, tgt, cfg, ctx=ctx), reps=20)
    emit({"config": 4, "op": "mlp4_train_step", "d": 784, "b": 32, "batch": 32, "us": us,
          "tflops": mlp.flops_per_step(cfg, 32) / us / 1e6})
    ctx.check()
    with open(os.path.join(ROOT, "gpurun_out", "bench_configs.json"), "w") as f:
        json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
