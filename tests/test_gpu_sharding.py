"""Batch-sharded FastH through the PRODUCT on the GPU at world size 2.

Both ranks run on cuda:0 (one GPU per gpurun box) over gloo: each computes
its column shard with the sm_100a kernels (fasth_forward_backward), then the
dV row buckets the context reports are all-reduced with
sharding.allreduce_dv_buckets on a comm stream that waits on each bucket's
event — the bench's multi-GPU step with gloo in place of NCCL.  The result
must equal the full-batch GPU step (dV is a batch sum, householder.hpp:144-147;
UX and dX are per column).
"""
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _inputs(d, m):
    import torch
    g = torch.Generator(device="cpu").manual_seed(7)
    V = torch.randn(d, d, generator=g)
    X = torch.randn(m, d, generator=g).t()
    G = torch.randn(m, d, generator=g).t()
    return V, X, G


def _worker(rank, world, port, d, m, b, nbuckets, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import torch
    import torch.distributed as dist
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        from paper_2009_13977_b200 import fasth as fb
        from paper_2009_13977_b200.sharding import allreduce_dv_buckets, shard_range
        V, X, G = _inputs(d, m)
        lo, hi = shard_range(m, world, rank)
        ctx = fb.Context(0, deferred=True)
        ctx.set_dv_buckets(nbuckets)
        comm = torch.cuda.Stream()
        Y, back = fb.fasth_forward_backward(V.cuda(), X[:, lo:hi].cuda(), G[:, lo:hi].cuda(), b, ctx=ctx)
        buckets = ctx.dv_buckets()
        allreduce_dv_buckets(back.grad_vectors, buckets, comm)
        torch.cuda.current_stream().wait_stream(comm)
        torch.cuda.synchronize()
        ctx.check()
        out_q.put((rank, lo, hi, len(buckets), Y.cpu().numpy(), back.grad_input.cpu().numpy(),
                   back.grad_vectors.cpu().numpy()))
        dist.barrier()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("d,m,b,lb", [(1024, 512, 32, True), (784, 64, 32, False)])
def test_sharded_product_equals_full_batch(d, m, b, lb):
    import torch
    import torch.multiprocessing as mp

    from paper_2009_13977_b200 import fasth as fb
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, d, m, b, 4, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    V, X, G = _inputs(d, m)
    Y, back = fb.fasth_forward_backward(V.cuda(), X.cuda(), G.cuda(), b)
    Y, dX, dV = (t.cpu().double().numpy() for t in (Y, back.grad_input, back.grad_vectors))
    rel = lambda a, w: float(np.linalg.norm(a - w) / max(np.linalg.norm(w), 1.0))  # noqa: E731
    for rank, lo, hi, nb, y, dx, dv in res:
        assert nb == (min(4, d // 512) if lb else 1)  # large-batch: one bucket per 512-wide block (<= 4)
        assert rel(y, Y[:, lo:hi]) <= 2e-5
        assert rel(dx, dX[:, lo:hi]) <= 2e-5
        assert rel(dv, dV) <= 2e-5  # the summed shards == the full-batch batch sum
    assert torch.cuda.is_available()
