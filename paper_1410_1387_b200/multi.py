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
    try:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    except RuntimeError:   # a backend without device-tensor support (gloo builds): host tensor
        t = t.cpu()
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def connect_peer(dist, handle, rank: int, world: int) -> bool:
    """Connect a rank's handle to its y-neighbours for the fused peer-memory halo transport
    (vti_ipc_export / vti_ipc_connect): every rank publishes its CUDA-IPC blob, then
    opens the blobs of rank-1 and rank+1. Returns True on every rank only if every
    rank succeeded (the decision is collective, so nobody waits on a peer that fell
    back to NCCL)."""
    if world == 1:
        return False
    blob = handle.ipc_export()
    blobs = [None] * world
    dist.all_gather_object(blobs, blob)
    ok = 1
    try:
        handle.ipc_connect(blobs[rank - 1] if rank > 0 else None, blobs[rank + 1] if rank < world - 1 else None)
    except Exception:
        ok = 0
    import torch
    t = torch.tensor([ok], dtype=torch.int32)
    try:
        dist.all_reduce(t, op=dist.ReduceOp.MIN)
    except RuntimeError:   # process groups whose backend needs device tensors
        t = t.cuda()
        dist.all_reduce(t, op=dist.ReduceOp.MIN)
    return bool(int(t.item()))


def sync_or_die(handle, timeout_s: float, what: str = "halo exchange", query=None, die=None) -> None:
    """Wait for the handle's enqueued steps, polling its stream, and exit the process
    loudly if they do not finish within timeout_s (a peer that never delivers its halo
    must fail the run, not hang it). The main stream waits on every exchange, so its
    completion covers the comm stream's work too.

    ``handle.stream`` is the cudaStream_t (an int property, vti_stream). ``query`` /
    ``die`` default to torch's stream query and os._exit(3); tests substitute them.
    """
    import os
    import sys
    import time

    if query is None:
        import torch
        query = torch.cuda.ExternalStream(handle.stream).query
    if die is None:
        die = os._exit
    t0 = time.monotonic()
    while not query():
        if time.monotonic() - t0 > timeout_s:
            print(f"error: {what} did not complete within {timeout_s:.0f} s "
                  f"(transport {handle.halo_transport}); aborting", file=sys.stderr, flush=True)
            die(3)
            return
        time.sleep(0.01)
    handle.sync()
