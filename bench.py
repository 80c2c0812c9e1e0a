"""FastH fwd+bwd benchmark (BASELINE.json metric) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Workload (BASELINE.json configs[1], the metric config): one FastH
forward + backward step — fasth_forward (fasth.hpp:40) then fasth_backward
(fasth.hpp:69) — at d = n = 784 Householder factors, WY block width b = 32
(BASELINE "m"), batch 32 columns (BASELINE "batch"), on the reference's own
synthetic workload (bench.hpp:117-134, op=mul, seed 0: V, X, G ~ N(0, 1)).
A step = WY build + forward chain + backward chain + per-vector gradients;
outputs UX, dX and dV are all produced every step.

Rows of the JSON line:
  value     device time per step (µs), inputs resident in HBM, the step
            replayed from a CUDA graph, L2 flushed (256 MiB write) before
            every timed step, CUDA events on the launch stream, max over ranks.
  e2e       the same step through the reference-facing host-buffer C ABI call
            fasth_forward_backward_host: pinned host V, X, G in, Y, dX, dV out,
            copies inside the timed region.
  roofline  the dominant kernel (the chain sweep) timed per launch with CUDA
            events inside this run (ctx timing mode), algorithmic flops per
            launch = 4 d n m, against the 3xTF32 tensor-pipe
            peak derived from MEASURED_PEAKS.json (bf16 dense / 6).
  cpu_baseline  the reference's own CPU FastH (oracle/_ref: the unmodified
            headers compiled as-is) via bench::run_bench on all host threads.

--impl reference times that CPU reference alone (rank 0 only) on the same
config (the whole job's batch, 32 x N columns) and prints the same line with
"impl": "reference".
N > 1: weak scaling, each rank runs the batch-32 step on its own shard and the
summed dV is all-reduced over NCCL inside the timed step.  Launched under
torchrun (the driver's form) or directly as ``python bench.py --gpus N``, in
which case it re-executes itself under torch.distributed.run with N ranks.
The `config5` object is BASELINE configs[4] as the north_star states it:
d = 2048, global batch 65536 sharded over the N ranks (strong scaling; the
1-GPU point runs the whole batch).
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "FastH fwd+bwd µs/step at d=784,m=32,batch=32; TFLOP/s vs tensor-pipe roofline"
D, B, M = 784, 32, 32
SEED = 0


def flops_alg(d, n, m, b):
    """F_alg = 12 d n m + 4 d n b useful fp32 flops per fwd+bwd."""
    return 12.0 * d * n * m + 4.0 * d * n * b


def peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        p = json.load(open(path))
        return {"bf16": p["bf16_tflops"], "bf16_sustained": p["bf16_tflops_sustained"],
                "hbm": p["hbm_gbs"], "src": "measured"}
    except Exception:
        return {"bf16": 1590.0, "bf16_sustained": 1400.0, "hbm": 6650.0, "src": "fallback"}


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.p = None

    def __enter__(self):
        try:
            self.p = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                       "--format=csv,noheader,nounits", "-lms", "50"],
                                      stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.p = None
        time.sleep(0.15)
        return self

    def __exit__(self, *a):
        self.out = ""
        if self.p is not None:
            time.sleep(0.1)
            self.p.terminate()
            try:
                self.out, _ = self.p.communicate(timeout=5)
            except Exception:
                self.p.kill()

    def summary(self):
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in (self.out or "").splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) < 6:
                continue
            try:
                sm.append(float(f[0]))
                mx = max(mx, float(f[1]))
            except ValueError:
                continue
            for nm, v in zip(names, f[2:6]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        sm.sort()
        med = sm[len(sm) // 2] if sm else None
        return {"sm_mhz": med, "sm_max_mhz": mx or None, "reasons": sorted(reasons),
                "samples": len(sm)}


def workload(d=D, m=M, seed=SEED):
    """The reference's own generator (bench.hpp:117-134) when oracle/_ref is
    present, else a numpy stand-in of the same distribution."""
    import numpy as np
    try:
        from oracle.oracle import Ref
        V, X, G = Ref().gen_mul(seed, d, m)
        src = "reference bench.hpp:117 op=mul"
    except Exception:
        rng = np.random.default_rng(seed + d)
        V, X, G = rng.standard_normal((d, d)), rng.standard_normal((d, m)), rng.standard_normal((d, m))
        src = "numpy N(0,1)"
    return V, X, G, src


def cpu_reference(d, m, b, reps, warm=1):
    """bench::run_bench (bench.hpp:225) on all host threads: (mean µs, std µs, cores, kind)."""
    from oracle.oracle import Ref
    R = Ref()
    for _ in range(max(warm - 1, 0)):
        R.run_bench("mul", "fasth", d, m, b, 1, SEED, 0)
    mean, std, _ = R.run_bench("mul", "fasth", d, m, b, reps, SEED, 0)
    return mean * 1e6, std * 1e6, R.hardware_threads(), "reference", R.march


def cpu_sequential(d, m, b, reps=8):
    """The reference's sequential-Householder path (run_bench algo=sequential:
    single-threaded by construction, reference.hpp), timed beside FastH as
    the north_star asks: (mean µs, std µs)."""
    from oracle.oracle import Ref
    R = Ref()
    mean, std, _ = R.run_bench("mul", "sequential", d, m, b, reps, SEED, 0)
    return mean * 1e6, std * 1e6


def headline_config(world):
    """The `config` object of both arms (same keys, same values)."""
    return {"workload": "FastH fwd+bwd op=mul (fasth_forward + fasth_backward, bench.hpp:147-151)",
            "d": D, "n": D, "block_width": B, "batch_per_gpu": M, "global_batch": M * world,
            "parallelism": f"batch-sharded dp{world}" if world > 1 else "single GPU"}


def run_reference_impl(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    world = max(args.gpus, int(os.environ.get("WORLD_SIZE", "1")))
    try:  # the whole job's batch (32 per GPU) on the host's cores
        us, std, cores, kind, march = cpu_reference(D, M * world, B, max(args.steps, 1), args.warmup)
    except Exception as e:  # the reference always builds here; report, don't fake
        print(json.dumps({"impl": "reference", "unavailable": f"oracle/_ref failed: {e}"}))
        return
    line = {
        "impl": "reference", "metric": METRIC, "value": us, "unit": "us/step", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": us / 1e3,
        "higher_is_better": False, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (reference generator bench.hpp:117, seed 0)",
        "config": headline_config(world),
        "algo": "fasth (reference CPU, all host threads)",
        "tflops": flops_alg(D, D, M * world, B) / (us * 1e-6) / 1e12,
        "cpu_baseline": {"value": us, "unit": "us/step", "cores": cores, "kind": kind,
                         "sample": f"run_bench op=mul d={D} m={M * world} k={B} algo=fasth, "
                                   f"{args.steps} reps after warm-up (std {std:.1f} us), built -march={march}"},
        "e2e": {"value": us, "unit": "us/step", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))


def layer_line(local, steps=50, warmup=5):
    """BASELINE configs[1] read as the layer: the SVD-reparameterised layer
    W = U Sigma V^T at d = 784, b = 32, batch 32 (svd_layer.hpp:106-154):
    svd_forward + svd_backward per step (two FastH chains each way, Sigma,
    dSigma), device time with CUDA events, inputs resident.  Synthetic:
    normalised N(0,1) vectors, sigma ~ U(0.5, 2) (bench.hpp:129-131)."""
    import torch

    from paper_2009_13977_b200 import fasth as fb
    d, b, m = D, B, M
    g = torch.Generator(device="cuda").manual_seed(SEED)
    U = torch.randn(d, d, device="cuda", generator=g)
    V = torch.randn(d, d, device="cuda", generator=g)
    U /= U.norm(dim=1, keepdim=True)
    V /= V.norm(dim=1, keepdim=True)
    s = torch.rand(d, device="cuda", generator=g) * 1.5 + 0.5
    X = torch.randn(m, d, device="cuda", generator=g).t()
    G = torch.randn(m, d, device="cuda", generator=g).t()
    p = fb.SvdParam(d, d, U, V, s)
    ctx = fb.Context(local, deferred=True)

    def step():  # G drawn up front, as the reference's layer benchmark (bench.hpp:166-209)
        return fb.svd_forward_backward(p, X, G, b, ctx=ctx)

    for _ in range(warmup):
        step()
    torch.cuda.synchronize()
    n0 = ctx.launch_count
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        step()
    e1.record()
    torch.cuda.synchronize()
    ctx.check()
    us = e0.elapsed_time(e1) * 1e3 / steps
    return {"workload": "BASELINE configs[1] as the layer: svd_forward + svd_backward as "
                        "fasth_svd_forward_backward (paired sweeps), W = U Sigma V^T",
            "d": d, "block_width": b, "batch": m, "us_per_step": us,
            "tflops": 2 * flops_alg(d, d, m, b) / (us * 1e-6) / 1e12,
            "gpu_launches_per_step": (ctx.launch_count - n0) / steps, "steps": steps, "warmup": warmup,
            "timing": "eager, CUDA events on the context stream, inputs resident",
            "data": "synthetic: normalised N(0,1) vectors, sigma ~ U(0.5, 2)"}


def large_batch_line(world, rank, local, peak_3xtf32, global_batch=65536, steps=10, warmup=3):
    """BASELINE.json configs[4]: d = 2048 FastH fwd+bwd on a global batch of
    65536 columns sharded over the ranks (strong scaling: 65536 on one GPU,
    8192 per GPU on eight), dV all-reduced over NCCL when world > 1 (row
    buckets overlapped with the backward).  Runs the tcgen05 large-batch path
    (lb.h).  Synthetic N(0,1) inputs on the device; CUDA events around
    `steps` steps, max over ranks; every step touches GBs, so L2 (126 MB)
    holds nothing across steps."""
    import torch
    import torch.distributed as dist

    from paper_2009_13977_b200 import fasth as fb
    from paper_2009_13977_b200.sharding import shard_range
    d, b = 2048, 32
    lo, hi = shard_range(global_batch, world, rank)
    m = hi - lo
    g = torch.Generator(device="cuda").manual_seed(0)
    V = torch.randn(d, d, device="cuda", generator=g)
    g.manual_seed(1000 + rank)
    X = torch.randn(m, d, device="cuda", generator=g).t()
    G = torch.randn(m, d, device="cuda", generator=g).t()
    ctx = fb.Context(local, deferred=True)
    outs = (torch.empty(m, d, device="cuda").t(), torch.empty(m, d, device="cuda").t(),
            torch.empty(d, d, device="cuda"))
    comm = None
    if world > 1:  # dV all-reduced per 512-row bucket as the backward finishes it
        from paper_2009_13977_b200.sharding import allreduce_dv_buckets
        ctx.set_dv_buckets(4)
        comm = torch.cuda.Stream()

    def step():
        _, back = fb.fasth_forward_backward(V, X, G, b, ctx=ctx, out=outs)
        if world > 1:
            allreduce_dv_buckets(back.grad_vectors, ctx.dv_buckets(), comm)
            torch.cuda.current_stream().wait_stream(comm)

    for _ in range(warmup):
        step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    n0 = ctx.launch_count
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        step()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / steps
    launches = (ctx.launch_count - n0) // steps
    if world > 1:
        t = torch.tensor([ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    ctx.check()
    flops = 12.0 * d * d * global_batch + 4.0 * d * d * b * world
    tf = flops / (ms * 1e-3) / 1e12
    # per-kernel: CUDA events around every launch of the large-batch path
    # (ctx timing mode), untimed steps, one stream (concurrent kernels would
    # stretch each other's event windows); algorithmic flops per launch below
    saved = os.environ.get("FASTH_LB_STREAMS")
    os.environ["FASTH_LB_STREAMS"] = "0"
    ctx.set_timing(True)
    for _ in range(3):
        step()
    torch.cuda.synchronize()
    kt = ctx.kernel_times()
    ctx.set_timing(False)
    if saved is None:
        del os.environ["FASTH_LB_STREAMS"]
    else:
        os.environ["FASTH_LB_STREAMS"] = saved
    Bw, nb = 512, d // 512
    fl = {"lb_f1_zf": 2.0 * m * Bw * d, "lb_k1_zb": 2.0 * m * Bw * d, "lb_f2_update": 2.0 * m * d * Bw,
          "lb_k4_update": 2.0 * m * d * Bw, "lb_dv": 2.0 * Bw * d * (2 * m + Bw), "lb_q": 2.0 * Bw * Bw * m,
          "lb_build_gram": 2.0 * Bw * Bw * d * nb, "lb_build_w": 2.0 * Bw * d * Bw * nb}
    kern = {k: {"us_per_launch": v[0] * 1e3 / v[1], "launches_per_step": v[1] / 3,
                "tflops": fl[k] / (v[0] * 1e-3 / v[1]) / 1e12 if k in fl else None}
            for k, v in kt.items() if k.startswith("lb_")}
    top = max((k for k in kern if k in fl), key=lambda k: kern[k]["us_per_launch"] * kern[k]["launches_per_step"])
    traffic = None
    try:
        traffic = json.load(open(os.path.join(ROOT, "profiles", "roofline_traffic.json"))).get(top)
    except Exception:
        pass
    roof = {"bound": "tensor", "kernel": top, "achieved": kern[top]["tflops"], "peak": peak_3xtf32,
            "unit": "TFLOP/s", "frac": kern[top]["tflops"] / peak_3xtf32, "traffic": traffic,
            "flops_per_launch": fl[top],
            "note": "3xTF32 useful flops; CUDA events per launch on the context stream (kernels serialised "
                    "for this pass); ncu tensor-pipe activity of these GEMMs in profiles/r01_lb_*_full.txt"}
    return {"workload": "BASELINE configs[4]: FastH fwd+bwd d=2048, global batch 65536 batch-sharded, dV "
                        "all-reduced (NCCL, 4 row buckets overlapped with the backward)",
            "scaling": "strong", "roofline": roof, "kernels": kern,
            "d": d, "batch_per_gpu": m, "global_batch": global_batch, "n_gpus": world,
            "us_per_step": ms * 1e3, "tflops": tf, "frac_3xtf32_peak": tf / (peak_3xtf32 * world),
            "steps": steps, "warmup": warmup, "gpu_launches_per_step": launches,
            "path": "large-batch: 512-wide WY blocks on the tcgen05 3xTF32 GEMM (cta_group::2)",
            "data": "synthetic N(0,1) on device", "l2": "working set ~1.5 GB per step (> L2)"}


def relaunch(args):
    """`python bench.py --gpus N` outside torchrun: re-execute under
    torch.distributed.run with N ranks on this node (the driver's form)."""
    import socket
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")        # NCCL's init log (rings / NVLS) stays visible on stderr
    env.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    return subprocess.call(cmd, env=env)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--cpu-reps", type=int, default=150, help="reps of the cpu_baseline sample")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-config5", action="store_true", help="skip the large-batch (config 5) line")
    ap.add_argument("--config5-batch", type=int, default=65536, help="config 5 global batch (strong scaling)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if args.impl == "reference":
        return run_reference_impl(args)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(relaunch(args))

    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_2009_13977_b200 import fasth as fb

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)

    V, X, G, src = workload()
    if world > 1:  # weak scaling: each rank its own batch-32 shard of a 32*world batch
        rng = np.random.default_rng(1000 + rank)
        X, G = rng.standard_normal(X.shape), rng.standard_normal(G.shape)
    Vd = torch.tensor(V, dtype=torch.float32, device=dev)            # (n, d) = col-major d x n
    Xd = torch.tensor(X.T.copy(), dtype=torch.float32, device=dev).t()  # (d, m) col-major
    Gd = torch.tensor(G.T.copy(), dtype=torch.float32, device=dev).t()

    ctx = fb.Context(local, deferred=True)
    stream = torch.cuda.Stream(dev)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)

    Yd = torch.empty((M, D), dtype=torch.float32, device=dev).t()
    dXd = torch.empty((M, D), dtype=torch.float32, device=dev).t()
    dVd = torch.empty((D, D), dtype=torch.float32, device=dev)

    def step():
        """fasth_forward + fasth_backward of the reference benchmark step
        (bench.hpp:147-151, G drawn up front) as the one-call
        fasth_forward_backward: build, both sweeps in one launch, gradients."""
        Y, back = fb.fasth_forward_backward(Vd, Xd, Gd, B, ctx=ctx, out=(Yd, dXd, dVd))
        if world > 1:
            dist.all_reduce(back.grad_vectors)
        return Y, back

    def step_two_calls():
        tape = fb.fasth_forward(Vd, Xd, B, ctx=ctx)
        return tape, fb.fasth_backward(tape, Gd)

    # parity gate on this very workload before timing anything
    with torch.cuda.stream(stream):
        Y0, back = step()
    torch.cuda.synchronize()
    ctx.check()
    parity = None
    if world == 1:
        try:
            from oracle.oracle import Port, relative_error
            want = Port().sequential_fwd_bwd(V, X, G)
            got = (Y0, back.grad_input, back.grad_vectors)
            parity = max(relative_error(g.double().cpu().numpy(), w) for g, w in zip(got, want))
            assert parity <= 1e-4, parity
        except ImportError:
            parity = None

    # capture the device step once (fwd+bwd; the NCCL all-reduce stays eager)
    with torch.cuda.stream(stream):
        for _ in range(args.warmup):
            step()
    torch.cuda.synchronize()
    launches0 = ctx.launch_count
    # the NCCL all-reduce of dV is captured into the same graph (N > 1); if
    # the capture is refused it stays eager after the replay
    ar_in_graph = world > 1
    try:
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph, stream=stream):
            g_y, g_back = fb.fasth_forward_backward(Vd, Xd, Gd, B, ctx=ctx, out=(Yd, dXd, dVd))
            if ar_in_graph:
                dist.all_reduce(g_back.grad_vectors)
    except Exception:  # noqa: BLE001
        if not ar_in_graph:
            raise
        torch.cuda.synchronize()
        ar_in_graph = False
        launches0 = ctx.launch_count
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph, stream=stream):
            g_y, g_back = fb.fasth_forward_backward(Vd, Xd, Gd, B, ctx=ctx, out=(Yd, dXd, dVd))
    launches_per_step = ctx.launch_count - launches0
    torch.cuda.synchronize()
    # the same work as the reference's two calls (fasth_forward, then
    # fasth_backward on the tape), for comparison
    graph2 = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph2, stream=stream):
        g2 = step_two_calls()
    torch.cuda.synchronize()

    def timed_graph(gr, k):
        tot = 0.0
        with torch.cuda.stream(stream):
            for _ in range(3):
                gr.replay()
            for i in range(k):
                flush.zero_()
                a_, b_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a_.record(stream)
                gr.replay()
                b_.record(stream)
                b_.synchronize()
                tot += a_.elapsed_time(b_)
        return tot * 1e3 / k

    def timed_loop(k):
        total = 0.0
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
              for _ in range(k)]
        with torch.cuda.stream(stream):
            for i in range(k):
                flush.zero_()
                ev[i][0].record(stream)
                graph.replay()
                if world > 1 and not ar_in_graph:
                    dist.all_reduce(g_back.grad_vectors)
                ev[i][1].record(stream)
        torch.cuda.synchronize()
        for a, b in ev:
            total += a.elapsed_time(b)
        return total

    for _ in range(args.warmup):
        graph.replay()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        t_ms = timed_loop(args.steps)
        # keep the GPU busy long enough for the clock sampler to see load
        t_end = time.time() + 0.4
        while time.time() < t_end:
            timed_loop(50)
    torch.cuda.synchronize()
    if world > 1:
        t = torch.tensor([t_ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        t_ms = float(t.item())
    us_per_step = t_ms * 1e3 / args.steps

    two_call_us = timed_graph(graph2, min(args.steps, 100))
    del g2

    # eager (no graph) device time, for reference
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(stream):
        e0.record(stream)
        for _ in range(50):
            step()
        e1.record(stream)
    torch.cuda.synchronize()
    eager_us = e0.elapsed_time(e1) * 1e3 / 50

    # per-kernel timing (dominant kernel share + roofline)
    ctx.set_timing(True)
    with torch.cuda.stream(stream):
        for _ in range(50):
            flush.zero_()
            step()
    torch.cuda.synchronize()
    ktimes = ctx.kernel_times()
    ctx.set_timing(False)

    # e2e: the reference-facing host-buffer C ABI call
    Vh = torch.tensor(V, dtype=torch.float32).pin_memory()
    Xh = torch.tensor(X.T.copy(), dtype=torch.float32).pin_memory()
    Gh = torch.tensor(G.T.copy(), dtype=torch.float32).pin_memory()
    hctx = fb.Context(local)
    hout = (torch.empty((M, D), dtype=torch.float32).pin_memory(),
            torch.empty((M, D), dtype=torch.float32).pin_memory(),
            torch.empty((D, D), dtype=torch.float32).pin_memory())
    # after the device-resident runs the first calls ramp down from ~190 us
    # over ~15 ms (the PCIe link and host waking up; BENCH_E2E_DUMP): untimed
    # calls for at least 0.2 s and W steps
    t_w = time.perf_counter() + 0.2
    n_w = 0
    while n_w < args.warmup or time.perf_counter() < t_w:
        fb.forward_backward_host(Vh, Xh, Gh, B, ctx=hctx, out=hout)
        n_w += 1
    e2e_steps = max(20, min(args.steps, 200))
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    walls = []
    for _ in range(e2e_steps):
        t0 = time.perf_counter()
        Yh, dXh, dVh = fb.forward_backward_host(Vh, Xh, Gh, B, ctx=hctx, out=hout)
        if world > 1:  # the batch-summed dV of the sharded job
            dvd = dVh.to(dev, non_blocking=True)
            dist.all_reduce(dvd)
            dVh.copy_(dvd)
            torch.cuda.synchronize()
        walls.append(time.perf_counter() - t0)
    if os.environ.get("BENCH_E2E_DUMP"):  # diagnostics: the per-call wall times in call order
        print("e2e walls us:", " ".join(f"{w * 1e6:.0f}" for w in walls), file=sys.stderr)
    walls.sort()
    # median of per-step wall times (each call returns synchronised results)
    e2e_us = walls[len(walls) // 2] * 1e6
    e2e_mean_us = sum(walls) / len(walls) * 1e6
    if world > 1:
        t = torch.tensor([e2e_us], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_us = float(t.item())
    h2d = 4 * (D * D + 2 * D * M)
    d2h = 4 * (D * D + 2 * D * M)

    # roofline of the dominant kernel (chain sweeps; flops per launch = 4 d n m)
    pk = peaks()
    # the fused sweep launch carries both chains: 8 d n m flops per launch
    sweep_ms = sum(v[0] for k, v in ktimes.items() if k.startswith("sweep"))
    sweep_n = sum(v[1] for k, v in ktimes.items() if k.startswith("sweep"))
    chains_per_launch = 2 if any(k.startswith("sweep(fwd+bwd)") for k in ktimes) else 1
    step_ms = sum(v[0] for v in ktimes.values())
    sweep_us = sweep_ms * 1e3 / max(sweep_n, 1)
    achieved = chains_per_launch * 4.0 * D * D * M / (sweep_us * 1e-6) / 1e12
    peak_3xtf32 = pk["bf16"] / 6.0
    traffic = None
    tfile = os.path.join(ROOT, "profiles", "roofline_traffic.json")
    if os.path.exists(tfile):
        try:
            traffic = json.load(open(tfile)).get("sweep_dram_bytes_per_launch")
        except Exception:
            traffic = None

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        try:
            us_c, std_c, cores, kind, march = cpu_reference(D, M, B, args.cpu_reps)
            cpu = {"value": us_c, "unit": "us/step", "cores": cores, "kind": kind,
                   "sample": f"reference bench::run_bench op=mul d={D} m={M} k={B} algo=fasth, "
                             f"{args.cpu_reps} reps (std {std_c:.0f} us), all host threads, built -march={march}"}
            us_s, std_s = cpu_sequential(D, M, B)
            cpu["sequential"] = {"value": us_s, "unit": "us/step", "cores": 1,
                                 "sample": f"run_bench op=mul d={D} m={M} algo=sequential (the reference's "
                                           f"reflection-by-reflection path), 8 reps (std {std_s:.0f} us)"}
        except Exception as e:
            cpu = {"value": None, "unit": "us/step", "cores": os.cpu_count(), "kind": "reference",
                   "sample": f"unavailable: {e}"}

    line = {
        "metric": METRIC, "value": us_per_step, "unit": "us/step", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": us_per_step / 1e3,
        "higher_is_better": False, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
        "data": f"synthetic ({src}, seed {SEED})",
        "config": headline_config(world),
        "api": "fasth_forward_backward (fasth_forward + fasth_backward in one call, G known up front as in "
               "bench.hpp:147-151)",
        "timing": {"l2": "flushed (256 MiB write) before every timed step",
                   "how": "CUDA graph replay, CUDA events on the launch stream, max over ranks"},
        "tflops": flops_alg(D, D, M * world, B) / (us_per_step * 1e-6) / 1e12,
        "eager_us_per_step": eager_us,
        "two_call": {"value": two_call_us, "unit": "us/step",
                     "api": "fasth_forward then fasth_backward on its tape (the training-path call pair, "
                            "fasth.hpp:40,69), CUDA graph, L2 flushed"},
        "two_call_us_per_step": two_call_us,
        "parity_max_rel_err": parity,
        "kernel_share": {k: round(v[0] / step_ms, 4) for k, v in ktimes.items()} if step_ms else {},
        "kernel_us": {k: v[0] * 1e3 / v[1] for k, v in ktimes.items()},
        "roofline": {"bound": "tensor", "achieved": achieved, "peak": peak_3xtf32,
                     "unit": "TFLOP/s", "frac": achieved / peak_3xtf32, "traffic": traffic,
                     "kernel": "sweep (forward and backward chains, one launch)",
                     "flops_per_launch": chains_per_launch * 4.0 * D * D * M,
                     "peak_note": f"3xTF32 useful = bf16 dense/6 of {pk['src']} "
                                  f"MEASURED_PEAKS ({pk['bf16']} TFLOP/s); the sweep runs 3xTF32 mma.sync "
                                  "and is latency bound at batch 32 (25 dependent block steps per chain)"},
        "e2e": {"value": e2e_us, "unit": "us/step", "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": d2h, "mean_us": e2e_mean_us, "steps": e2e_steps,
                "timing": "host wall clock per call (median), copies and sync inside",
                "api": "fasth_forward_backward_host (C ABI, pinned host buffers)"},
        "gpu_launches": launches_per_step * args.steps,
        "allreduce": ("NCCL all-reduce(SUM) of dV captured in the step's CUDA graph" if ar_in_graph else
                      "eager NCCL all-reduce(SUM) of dV after the graph replay") if world > 1 else None,
        "clocks": clk.summary(),
        "cpu_baseline": cpu,
    }
    if world == 1:
        try:
            line["config2_layer"] = layer_line(local)
            if cpu is not None and cpu.get("value"):
                from oracle.oracle import Ref
                mean, std, _ = Ref().run_bench("layer", "fasth", D, M, B, 20, SEED, 0)
                line["config2_layer"]["cpu_reference_us"] = mean * 1e6
                line["config2_layer"]["cpu_reference_sample"] = (
                    f"run_bench op=layer d={D} m={M} k={B} algo=fasth, 20 reps (std {std * 1e6:.0f} us), "
                    "all host threads")
        except Exception as e:  # noqa: BLE001
            line["config2_layer"] = {"unavailable": str(e)[:200]}
    if not args.no_config5:
        try:
            line["config5"] = large_batch_line(world, rank, local, peak_3xtf32, args.config5_batch)
        except Exception as e:  # noqa: BLE001 - the headline line must still print
            line["config5"] = {"unavailable": str(e)[:200]}
    if rank == 0:
        print(json.dumps(line))
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
