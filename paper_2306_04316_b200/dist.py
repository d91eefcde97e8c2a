"""Multi-GPU helpers: one process per GPU (torch.distributed), points sharded,
polygon replicated, bit planes gathered once at the end.

The reference parallelises with contiguous std::thread chunks over points
(proj/include/polycast/batch.hpp:217-227) and guarantees identical output for
any worker count; the same holds here for any world size: shards are
contiguous and 32-point aligned, so every rank owns whole flag words and the
gathered plane is bit-identical to the single-GPU one.
"""
from __future__ import annotations

import numpy as np


def shard_range(n: int, rank: int, world: int, align: int = 32) -> tuple[int, int]:
    """Contiguous [lo, hi) of n units for `rank`, boundaries multiples of `align`."""
    per = -(-n // world)
    per = -(-per // align) * align
    lo = min(n, rank * per)
    hi = min(n, (rank + 1) * per)
    return lo, hi


def gather_bit_planes(local_words, n_total: int, world: int, group=None):
    """All-gather per-rank bit planes (rank r covers shard_range(n_total, r, world))
    into the full plane.  `local_words` is a 1-D int32 torch tensor; returns a
    uint32 numpy array of ceil(n_total/32) words (on every rank)."""
    import torch
    import torch.distributed as dist

    per_words = -(-shard_range(n_total, 0, world)[1] // 32) if world > 1 else len(local_words)
    buf = torch.zeros(per_words, dtype=torch.int32, device=local_words.device)
    buf[: len(local_words)] = local_words
    out = torch.zeros(world * per_words, dtype=torch.int32, device=local_words.device)
    dist.all_gather_into_tensor(out, buf, group=group)
    full = np.zeros((n_total + 31) // 32, np.uint32)
    host = out.cpu().numpy().view(np.uint32)
    for r in range(world):
        lo, hi = shard_range(n_total, r, world)
        if hi > lo:
            w0, nw = lo // 32, (hi - lo + 31) // 32
            full[w0:w0 + nw] = host[r * per_words:r * per_words + nw]
    return full


def job_totals(units: float, points: float, world: int, device=None, group=None) -> tuple[float, float]:
    """(units, points) summed over all ranks."""
    if world <= 1:
        return float(units), float(points)
    import torch
    import torch.distributed as dist

    t = torch.tensor([units, points], dtype=torch.float64, device=device)
    dist.all_reduce(t, group=group)
    return float(t[0]), float(t[1])


def max_over_ranks(value: float, world: int, device=None, group=None) -> float:
    if world <= 1:
        return float(value)
    import torch
    import torch.distributed as dist

    t = torch.tensor([value], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t.item())
