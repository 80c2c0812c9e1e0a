"""BASELINE.json configs[4]: d = 2048 FastH fwd+bwd on a large batch, batch-
sharded (weak: each rank its own m-column shard; dV all-reduced over NCCL).

    python scripts/bench_config5.py [--m-per-gpu 8192] [--steps 5]
    python -m torch.distributed.run --nproc-per-node N scripts/bench_config5.py ...

Synthetic N(0,1) inputs generated on the device; the step (build, both
sweeps, gradients, all-reduce of dV) is timed with CUDA events, max over
ranks.  Prints one JSON line (rank 0): us/step, TFLOP/s (F_alg = 12 d n m +
4 d n b per fwd+bwd) and the fraction of the 3xTF32 peak."""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import torch.distributed as dist

from paper_2009_13977_b200 import fasth as fb


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--d", type=int, default=2048)
    ap.add_argument("--b", type=int, default=32)
    ap.add_argument("--m-per-gpu", type=int, default=8192)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=2)
    args = ap.parse_args()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    d, b, m = args.d, args.b, args.m_per_gpu
    g = torch.Generator(device="cuda").manual_seed(0)
    V = torch.randn(d, d, device="cuda", generator=g)  # same chain on every rank
    g.manual_seed(1000 + rank)
    X = torch.randn(m, d, device="cuda", generator=g).t()
    G = torch.randn(m, d, device="cuda", generator=g).t()
    ctx = fb.Context(local, deferred=True)
    outs = (torch.empty(m, d, device="cuda").t(), torch.empty(m, d, device="cuda").t(),
            torch.empty(d, d, device="cuda"))

    def step():
        _, back = fb.fasth_forward_backward(V, X, G, b, ctx=ctx, out=outs)
        if world > 1:
            dist.all_reduce(back.grad_vectors)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(args.steps):
        step()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / args.steps
    if world > 1:
        t = torch.tensor([ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    ctx.check()
    flops = (12.0 * d * d * m + 4.0 * d * d * b) * world
    peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["bf16_tflops"] / 6.0
    tf = flops / (ms * 1e-3) / 1e12
    if rank == 0:
        print(json.dumps({"config": 5, "d": d, "b": b, "m_per_gpu": m, "global_batch": m * world, "n_gpus": world,
                          "us_per_step": ms * 1e3, "tflops": tf, "frac_3xtf32_peak": tf / peak,
                          "scaling": "weak", "data": "synthetic N(0,1) on device",
                          "path": {"0": "chain/panel", "1": "large_batch"}.get(os.environ.get("FASTH_LB", ""), "auto")}))
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
