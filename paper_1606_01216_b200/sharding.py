"""Shift sharding across ranks: the l shifted systems are independent,
so rank r of N takes shifts r, r+N, ... and solves them with no collective on the
data path.  Only timing (max over ranks) and, optionally, the solution blocks
(all-gather, for a global Arnoldi block downstream) cross ranks."""
from __future__ import annotations

from typing import List, Sequence


def log_shifts(count: int, lo: float = 10.0, hi: float = 1e4) -> List[float]:
    """count real shifts log-spaced in [lo, hi] (BASELINE configs: 10^(1 + 3 i / (count - 1)))."""
    if count == 1:
        return [lo]
    a, b = __import__("math").log10(lo), __import__("math").log10(hi)
    return [10.0 ** (a + (b - a) * i / (count - 1)) for i in range(count)]


def shard(items: Sequence, rank: int, world: int) -> list:
    """Round-robin shard of items for rank (disjoint, covering, balanced to +-1)."""
    if not (0 <= rank < world):
        raise ValueError("rank out of range")
    return list(items[rank::world])


def owner(index: int, world: int) -> int:
    return index % world


def max_over_ranks(values: Sequence[float], dist=None, device=None) -> List[float]:
    """Element-wise max over ranks (device-timed ms per rank -> job time)."""
    if dist is None or not dist.is_initialized() or dist.get_world_size() == 1:
        return [float(v) for v in values]
    import torch
    t = torch.tensor(list(values), dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return [float(x) for x in t.tolist()]


def gather_blocks(local_blocks: Sequence, local_index: Sequence[int], total: int, dist=None):
    """All-gather per-shift solution blocks so every rank holds the full list (index order)."""
    if dist is None or not dist.is_initialized() or dist.get_world_size() == 1:
        out = [None] * total
        for i, b in zip(local_index, local_blocks):
            out[i] = b
        return out
    gathered = [None] * dist.get_world_size()
    dist.all_gather_object(gathered, list(zip(local_index, local_blocks)))
    out = [None] * total
    for part in gathered:
        for i, b in part:
            out[i] = b
    return out
