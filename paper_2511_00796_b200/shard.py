"""Multi-GPU sharding of one constrained_search.

The layout rank space [0, total) is split into world contiguous ranges; each rank
scans its own range (gp_constrained_search_range) and the (cost, rank, feasible)
triples are all-gathered — 24 bytes per rank — and reduced lexicographically:
the smallest rank among equal costs is the single-GPU / reference answer.
Works with any torch.distributed backend (NCCL on B200 boxes, gloo in CPU tests).
"""
from __future__ import annotations

import math


def shard_range(total: int, rank: int, world: int) -> tuple[int, int]:
    return total * rank // world, total * (rank + 1) // world


def reduce_winners(rows):
    """rows: iterable of (cost, rank, feasible) with rank < 0 meaning "no feasible layout".
    Returns (cost, rank, feasible_total) of the lexicographic minimum."""
    best = None
    feasible = 0
    for cost, rank, feas in rows:
        feasible += int(feas)
        if rank < 0:
            continue
        key = (cost, int(rank))
        if best is None or key < best:
            best = key
    if best is None:
        return math.inf, -1, feasible
    return best[0], best[1], feasible


def gather_winner(found: bool, cost: float, rank: int, feasible: int, device=None):
    """All-gather this rank's (cost, rank, feasible) and reduce; identity when not distributed."""
    import torch
    import torch.distributed as dist
    row = (cost if found else math.inf, float(rank if found else -1), float(feasible))
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return reduce_winners([row])
    t = torch.tensor(row, dtype=torch.float64, device=device)
    out = torch.empty(dist.get_world_size() * 3, dtype=torch.float64, device=device)
    dist.all_gather_into_tensor(out, t)
    return reduce_winners((c, int(r), int(f)) for c, r, f in out.view(-1, 3).tolist())
