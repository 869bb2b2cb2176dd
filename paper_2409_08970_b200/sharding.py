"""Batch sharding across GPUs (one process per GPU, torch.distributed).

DCT+ signals are independent, so a batch splits into contiguous row slices
with no data-path collective.  torch.distributed is used only
for the plumbing: barriers and the max-over-ranks timing reduction.
"""
from __future__ import annotations

from typing import Tuple


def shard_rows(batch: int, rank: int, world: int) -> Tuple[int, int]:
    """Contiguous slice [start, start + count) of `batch` rows for `rank`:
    the first batch % world ranks take one extra row."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("shard_rows: need 0 <= rank < world")
    base, extra = divmod(batch, world)
    start = rank * base + min(rank, extra)
    return start, base + (1 if rank < extra else 0)


def max_over_ranks(value: float, device=None) -> float:
    """max of a per-rank scalar (device time) over all ranks; identity when
    torch.distributed is not initialised."""
    import torch
    import torch.distributed as dist

    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def forward_shard(plan, signals, rank: int, world: int, **kw):
    """This rank's share of a batched forward: rows shard_rows(...) of
    `signals` (a host array or a tensor on this rank's device)."""
    start, count = shard_rows(signals.shape[0], rank, world)
    return start, plan.forward(signals[start:start + count], **kw)
