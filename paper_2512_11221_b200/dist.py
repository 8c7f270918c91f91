"""Multi-GPU plumbing for the sequence-sharded mode.

Sequences are independent (one ledger per sequence, R-layer), so the batch is partitioned across
ranks with no collective on the hot path: rank r owns sequences [r*B/N, (r+1)*B/N) in its own
context (pool, ledger, host mirror on its GPU).  torch.distributed is used only for the barrier
around timed regions and to reduce the timings (max over ranks) — plumbing, not the product.
"""
from __future__ import annotations

import os


def env_rank() -> tuple[int, int, int]:
    """(rank, world_size, local_rank) from the torchrun environment (defaults: single process)."""
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")),
            int(os.environ.get("LOCAL_RANK", "0")))


def shard(total: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous block partition of `total` sequences: (first, count) of this rank.
    The first total % world ranks get one extra sequence; every sequence has exactly one owner."""
    if world <= 0 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    q, r = divmod(total, world)
    first = rank * q + min(rank, r)
    return first, q + (1 if rank < r else 0)


def max_over_ranks(value: float, device=None) -> float:
    """Max of a per-rank float over the process group (identity without one)."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def sum_over_ranks(value: float, device=None) -> float:
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())
