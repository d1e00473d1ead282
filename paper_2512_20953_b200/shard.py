"""Multi-GPU sharding of plan searches: one process per GPU.

The path shards without a data-path collective: the TP-dimension searches of
one plan (and the snapshots of a replanning sweep) are independent problems,
assigned to ranks (longest-first by estimated cost, or round-robin); each rank runs its share on its own GPU and the
per-problem results are exchanged once at the end (torch.distributed
all_gather over NCCL on the B200 box, gloo in the CPU tests), after which every
rank holds the full, identically ordered result list and can replay the
reference selection deterministically.
"""
from __future__ import annotations

from typing import Callable, List, Optional, Sequence, TypeVar

T = TypeVar("T")
R = TypeVar("R")


def shard_indices(n: int, rank: int, world: int,
                  costs: Optional[Sequence[float]] = None) -> List[int]:
    """Problem indices owned by `rank`, ascending.

    Without costs: round-robin (the snapshots of a sweep). With costs: greedy
    longest-first (LPT) — each problem, most expensive first (ties: lower
    index), goes to the least-loaded rank (ties: lower rank). For one plan's
    TP dimensions the budgeted searches dominate, so the slowest (most units)
    gets a GPU to itself when there are enough ranks. Deterministic: every rank
    computes the same assignment."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} / world {world}")
    if costs is None:
        return list(range(rank, n, world))
    if len(costs) != n:
        raise ValueError(f"{len(costs)} costs for {n} problems")
    load = [0.0] * world
    owner = [0] * n
    for i in sorted(range(n), key=lambda i: (-costs[i], i)):
        r = min(range(world), key=lambda r: (load[r], r))
        owner[i] = r
        load[r] += costs[i]
    return [i for i in range(n) if owner[i] == rank]


def merge_shards(per_rank: Sequence[Sequence[R]], n: int,
                 costs: Optional[Sequence[float]] = None) -> List[R]:
    """Inverse of shard_indices: per-rank result lists back into problem order."""
    world = len(per_rank)
    out: List[R] = [None] * n  # type: ignore[list-item]
    for r, res in enumerate(per_rank):
        idx = shard_indices(n, r, world, costs)
        if len(idx) != len(res):
            raise ValueError(f"rank {r} returned {len(res)} results for {len(idx)} problems")
        for i, x in zip(idx, res):
            out[i] = x
    return out


def sharded_map(items: Sequence[T], fn: Callable[[List[T]], List[R]], dist=None,
                costs: Optional[Sequence[float]] = None) -> List[R]:
    """Run fn on this rank's shard and all-gather the results (object collective).

    Without torch.distributed (or at world size 1) this is fn(items)."""
    if dist is None or not dist.is_initialized() or dist.get_world_size() == 1:
        return list(fn(list(items)))
    rank, world = dist.get_rank(), dist.get_world_size()
    mine = [items[i] for i in shard_indices(len(items), rank, world, costs)]
    local = list(fn(mine)) if mine else []
    gathered: List[List[R]] = [None] * world  # type: ignore[list-item]
    dist.all_gather_object(gathered, local)
    return merge_shards(gathered, len(items), costs)


def search_cost(problem) -> float:
    """Relative cost of one grouping search for shard_indices: a budget-truncated
    search (more units than exact_threshold) scales with its unit count, an
    exhaustive one (<= exact_threshold units) is negligible."""
    return float(problem.n) * (1000.0 if problem.n > problem.exact_threshold else 1.0)
