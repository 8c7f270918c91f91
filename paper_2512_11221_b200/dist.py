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


def head_shard(Hq: int, Hkv: int, rank: int, world: int) -> tuple[int, int, int, int]:
    """Head-sharded mode: (q_lo, q_hi, kv_lo, kv_hi) of this rank.  KV heads are split evenly and each
    rank keeps the query heads that read them (GQA groups stay whole)."""
    if Hkv % world or Hq % Hkv:
        raise ValueError("need n_kv_heads % world == 0 and n_q_heads % n_kv_heads == 0")
    hk = Hkv // world
    g = Hq // Hkv
    return rank * hk * g, (rank + 1) * hk * g, rank * hk, (rank + 1) * hk


def share_nccl_id(make_id) -> bytes:
    """Rank 0 calls make_id() (e.g. asr_nccl_unique_id) and broadcasts the 128 bytes to every rank over
    the torch.distributed process group (plumbing; any backend)."""
    import torch.distributed as dist
    obj = [make_id() if dist.get_rank() == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    return obj[0]


def ledger_digest(ctx, batch: int) -> str:
    """Hex digest of every sequence's ledger and attended list (head-sharded mode: every rank must take
    bitwise the same decisions — the digests are all-gathered and compared)."""
    import hashlib
    h = hashlib.sha256()
    for b in range(batch):
        st = ctx.stats(b, detail=True)
        for k in ("residency", "timer", "count", "freeze_step"):
            h.update(st["ledger"][k].tobytes())
        h.update(st["active_list"].tobytes())
    return h.hexdigest()


def ranks_agree(digest: str) -> bool:
    """All-gather a per-rank digest over the process group; True iff every rank has the same one."""
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return True
    out = [None] * dist.get_world_size()
    dist.all_gather_object(out, digest)
    return all(x == out[0] for x in out)
