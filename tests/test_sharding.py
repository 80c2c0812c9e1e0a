"""Batch-sharded FastH across ranks (world_size 2, gloo, CPU): per-rank
column shards + one all-reduce(SUM) of dV reproduce the full-batch result.
The per-rank compute here is the f64 oracle (no GPU in this container); the
GPU path uses the same sharding helpers with NCCL (bench.py --gpus N)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2009_13977_b200.sharding import shard_range


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, d, m, b, out_q, bucketed=False):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle.oracle import Port
    from paper_2009_13977_b200.sharding import allreduce_dv_buckets, allreduce_grads
    rng = np.random.default_rng(7)
    V, X, G = rng.standard_normal((d, d)), rng.standard_normal((d, m)), rng.standard_normal((d, m))
    lo, hi = shard_range(m, world, rank)
    Y, dX, dV = Port().fasth_fwd_bwd(V, X[:, lo:hi], G[:, lo:hi], b)
    dVt = torch.tensor(dV)
    if bucketed:  # row buckets as Context.dv_buckets() reports them (events: GPU only)
        allreduce_dv_buckets(dVt, [(0, 3, None), (3, 3, None), (3, 10, None), (10, d, None)])
    else:
        allreduce_grads([dVt])
    out_q.put((rank, lo, hi, Y, dX, dVt.numpy()))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("m,bucketed", [(8, False), (7, False), (7, True)])
def test_batch_sharded_dV_allreduce_gloo(m, bucketed):
    from oracle.oracle import Port, relative_error
    d, b, world = 24, 5, 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, d, m, b, q, bucketed)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    rng = np.random.default_rng(7)
    V, X, G = rng.standard_normal((d, d)), rng.standard_normal((d, m)), rng.standard_normal((d, m))
    Y, dX, dV = Port().fasth_fwd_bwd(V, X, G, b)
    for rank, lo, hi, y, dx, dv in res:
        assert relative_error(y, Y[:, lo:hi]) < 1e-12
        assert relative_error(dx, dX[:, lo:hi]) < 1e-12
        assert relative_error(dv, dV) < 1e-12  # summed over ranks == full-batch sum


def test_shard_range_covers_batch():
    for m in (0, 1, 7, 32, 65536):
        for world in (1, 2, 3, 8):
            spans = [shard_range(m, world, r) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == m
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
            assert max(h - l for l, h in spans) - min(h - l for l, h in spans) <= 1
