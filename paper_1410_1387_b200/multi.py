"""Multi-GPU bootstrap over torch.distributed (one process per GPU).

The y-slab path's only collective is the per-step halo exchange, done by the
library with NCCL on its own communicator (include/vti.h, vti_step). torch's
process group is plumbing: it carries the 128-byte ncclUniqueId from rank 0
to every rank, and the max-over-ranks reduction of timings.
"""
from __future__ import annotations


def broadcast_nccl_id(dist, rank: int, world: int) -> bytes | None:
    """A fresh ncclUniqueId from rank 0 (ids are single-use: one per communicator)."""
    if world == 1:
        return None
    from . import nccl_unique_id
    obj = [nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    return obj[0]


def max_over_ranks(dist, world: int, x: float, device="cpu") -> float:
    """Max of a scalar over all ranks (the contract's timing rule for N > 1)."""
    if world == 1:
        return x
    import torch
    t = torch.tensor([float(x)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())
