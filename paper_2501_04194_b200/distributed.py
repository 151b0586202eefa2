"""Batch sharding across GPUs.

Rows of a batch are independent (``trace_var`` treats leading axes as batch,
masking.py:310; SPEC "independent batch items may run in parallel"), so each
rank evaluates a contiguous block of rows with no communication.  The only
exchange is one all-reduce (sum) of the smooth-interval parameter gradients
``(d_a, d_b, d_c)`` — 24 bytes in fp64, for determinism — plus any scalar
loss the caller averages over the batch.

One process per GPU; ``torch.distributed`` with the NCCL backend on B200
(gloo works the same on CPU, which the tests use).
"""

from __future__ import annotations

from typing import Iterable, Optional

import torch

__all__ = ["shard_rows", "allreduce_interval_grads", "sharded_trace"]


def shard_rows(batch: int, rank: int, world: int) -> slice:
    """Contiguous row block of ``rank``: sizes differ by at most one row."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} / world {world}")
    base, extra = divmod(batch, world)
    lo = rank * base + min(rank, extra)
    hi = lo + base + (1 if rank < extra else 0)
    return slice(lo, hi)


def allreduce_interval_grads(tensors: Iterable[Optional[torch.Tensor]], group=None) -> None:
    """Sum the ``.grad`` of the (a, b, c) binding tensors over ranks, in place.

    The gradients are packed into one fp64 buffer so the whole exchange is a
    single all-reduce.
    """
    import torch.distributed as dist
    ts = [t for t in tensors if t is not None and t.grad is not None]
    if not ts or not dist.is_available() or not dist.is_initialized() or dist.get_world_size() == 1:
        return
    flat = torch.stack([t.grad.reshape(()).to(torch.float64) for t in ts])
    dist.all_reduce(flat, op=dist.ReduceOp.SUM, group=group)
    for t, v in zip(ts, flat):
        t.grad.copy_(v.to(t.grad.dtype).reshape(t.grad.shape))


def sharded_trace(f, channels, cfg, smooth_binding=None, rank=None, world=None):
    """Evaluate this rank's rows of ``channels`` (full-batch tensors or already-local).

    Returns ``(local_trace, row_slice)``.  Call ``allreduce_interval_grads`` on
    the binding tensors after ``backward`` to finish the interval gradients.
    """
    import torch.distributed as dist
    from .engine import trace
    if rank is None:
        rank = dist.get_rank() if dist.is_initialized() else 0
    if world is None:
        world = dist.get_world_size() if dist.is_initialized() else 1
    B = next(iter(channels.values())).shape[0]
    sl = shard_rows(B, rank, world)
    local = {k: v[sl] for k, v in channels.items()}
    return trace(f, local, cfg, smooth_binding=smooth_binding), sl
