"""Batch sharding across GPUs.

Rows of a batch are independent (``trace_var`` treats leading axes as batch,
masking.py:310; SPEC "independent batch items may run in parallel"), so each
rank evaluates a contiguous block of rows with no communication.  The only
exchange is one all-reduce (sum) of the smooth-interval parameter gradients
``(d_a, d_b, d_c)`` — 24 bytes in fp64 — plus any scalar loss the caller
averages over the batch (``apps.py:279``'s mean over the dataset).

One process per GPU; ``torch.distributed`` with the NCCL backend on B200
(gloo works the same on CPU, which the host tests use).
"""

from __future__ import annotations

from typing import Mapping, Optional, Sequence

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


def _rank_world(rank, world):
    import torch.distributed as dist
    init = dist.is_available() and dist.is_initialized()
    if rank is None:
        rank = dist.get_rank() if init else 0
    if world is None:
        world = dist.get_world_size() if init else 1
    return rank, world


def allreduce_interval_grads(tensors: Sequence[Optional[torch.Tensor]], group=None) -> None:
    """Sum the ``.grad`` of the (a, b, c) binding tensors over ranks, in place.

    Collective: every initialised rank must call it with the same number of entries.
    A rank whose entry is ``None`` or has no ``.grad`` (e.g. it had no smooth-interval
    gradient to contribute) still joins the all-reduce with zeros, so no rank blocks.
    The gradients travel packed in one fp64 buffer (one all-reduce per call); entries
    that had no ``.grad`` receive the reduced value as a fresh ``.grad``.
    """
    import torch.distributed as dist
    if not dist.is_available() or not dist.is_initialized() or dist.get_world_size(group) == 1:
        return
    ts = list(tensors)
    dev = next((t.device for t in ts if t is not None), None)
    if dist.get_backend(group) == "nccl":
        dev = torch.device("cuda", torch.cuda.current_device())
    elif dev is None:
        dev = torch.device("cpu")
    flat = torch.zeros(len(ts), dtype=torch.float64, device=dev)
    for i, t in enumerate(ts):
        if t is not None and t.grad is not None:
            flat[i] = t.grad.reshape(()).to(torch.float64)
    dist.all_reduce(flat, op=dist.ReduceOp.SUM, group=group)
    for t, v in zip(ts, flat):
        if t is None:
            continue
        if t.grad is None:
            t.grad = v.to(dtype=t.dtype, device=t.device).reshape(t.shape)
        else:
            t.grad.copy_(v.to(t.grad.dtype).reshape(t.grad.shape))


def sharded_trace(f, channels: Mapping[str, torch.Tensor], cfg, smooth_binding=None, *,
                  local: bool = False, rank: Optional[int] = None, world: Optional[int] = None):
    """This rank's rows of the robustness trace (``engine.trace``, differentiable).

    ``local=False``: ``channels`` hold the FULL batch ``[B, T]`` (1-D ``[T]`` is one row)
    and this rank takes ``shard_rows(B, rank, world)``; ``B < world`` is rejected, since a
    rank with no rows could not join the interval-gradient all-reduce meaningfully.
    ``local=True``: ``channels`` already hold this rank's rows and are used as given.

    Returns ``(local_trace, row_slice)`` (``row_slice`` is ``None`` when ``local``).  After
    ``backward``, call ``allreduce_interval_grads`` on the binding tensors on every rank.
    """
    from .engine import trace
    rank, world = _rank_world(rank, world)
    if local:
        return trace(f, channels, cfg, smooth_binding=smooth_binding), None
    rows = {k: (v.unsqueeze(0) if v.dim() == 1 else v) for k, v in channels.items()}
    B = next(iter(rows.values())).shape[0]
    if any(v.shape[0] != B for v in rows.values()):
        raise ValueError("channels disagree on the batch size")
    if B < world:
        raise ValueError(f"batch of {B} rows cannot be sharded over {world} ranks")
    sl = shard_rows(B, rank, world)
    local_rows = {k: v[sl] for k, v in rows.items()}
    return trace(f, local_rows, cfg, smooth_binding=smooth_binding), sl
