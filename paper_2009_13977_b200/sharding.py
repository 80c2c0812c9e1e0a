"""Batch sharding of the FastH step across GPUs.

UX and dX are column-wise independent, so each rank owns a contiguous column
slice of X / G (column-major layout makes the slice contiguous).  The only
exchange is the batch sum of the vector gradients dV (Eq. (5) sums over the
batch, householder.hpp:145-147) and of dSigma (svd_layer.hpp:131-137): one
all-reduce(SUM) over NCCL (NVLink / NVSwitch) per step.
"""
from __future__ import annotations


def shard_range(m: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous column slice [lo, hi) of a batch of m columns for `rank`;
    the first m % world ranks get one extra column."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad world/rank")
    base, extra = divmod(m, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def allreduce_grads(tensors, group=None):
    """Sum the batch-summed gradients over the ranks (in place)."""
    import torch.distributed as dist
    for t in tensors:
        if t is not None and t.numel():
            dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
    return tensors


def allreduce_dv_buckets(dV, buckets, comm_stream=None, group=None):
    """Bucketed batch sum of dV, overlapped with the backward.

    ``buckets`` = Context.dv_buckets(): [(row_begin, row_end, event)] in
    completion order.  Each row slice of the (n, d) row-major dV is
    all-reduced on ``comm_stream`` after that stream waits on the bucket's
    event, so the first buckets travel over NVLink while the large-batch
    backward still computes the later ones.  The caller's stream must wait on
    ``comm_stream`` before reading dV (returned for convenience).  With
    ``comm_stream=None`` (CPU / gloo) the slices are reduced in order on the
    current stream."""
    import contextlib

    import torch
    import torch.distributed as dist
    if comm_stream is not None:
        ctx = torch.cuda.stream(comm_stream)
    else:
        ctx = contextlib.nullcontext()
    with ctx:
        for lo, hi, ev in buckets:
            if hi <= lo:
                continue
            if comm_stream is not None and ev is not None:
                comm_stream.wait_event(ev)
            dist.all_reduce(dV[lo:hi], op=dist.ReduceOp.SUM, group=group)
    return comm_stream
