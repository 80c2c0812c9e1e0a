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
