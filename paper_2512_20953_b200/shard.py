"""Multi-GPU sharding of plan searches: one process per GPU.

The path shards without a data-path collective: the TP-dimension searches of
one plan (and the snapshots of a replanning sweep) are independent problems,
assigned round-robin to ranks; each rank runs its share on its own GPU and the
per-problem results are exchanged once at the end (torch.distributed
all_gather over NCCL on the B200 box, gloo in the CPU tests), after which every
rank holds the full, identically ordered result list and can replay the
reference selection deterministically.
"""
from __future__ import annotations

from typing import Callable, List, Sequence, TypeVar

T = TypeVar("T")
R = TypeVar("R")


def shard_indices(n: int, rank: int, world: int) -> List[int]:
    """Problem indices owned by `rank` (round-robin: budgeted TP dims, which come
    first in ascending-tp order, land on different ranks)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} / world {world}")
    return list(range(rank, n, world))


def merge_shards(per_rank: Sequence[Sequence[R]], n: int) -> List[R]:
    """Inverse of shard_indices: per-rank result lists back into problem order."""
    world = len(per_rank)
    out: List[R] = [None] * n  # type: ignore[list-item]
    for r, res in enumerate(per_rank):
        idx = shard_indices(n, r, world)
        if len(idx) != len(res):
            raise ValueError(f"rank {r} returned {len(res)} results for {len(idx)} problems")
        for i, x in zip(idx, res):
            out[i] = x
    return out


def sharded_map(items: Sequence[T], fn: Callable[[List[T]], List[R]], dist=None) -> List[R]:
    """Run fn on this rank's shard and all-gather the results (object collective).

    Without torch.distributed (or at world size 1) this is fn(items)."""
    if dist is None or not dist.is_initialized() or dist.get_world_size() == 1:
        return list(fn(list(items)))
    rank, world = dist.get_rank(), dist.get_world_size()
    mine = [items[i] for i in shard_indices(len(items), rank, world)]
    local = list(fn(mine)) if mine else []
    gathered: List[List[R]] = [None] * world  # type: ignore[list-item]
    dist.all_gather_object(gathered, local)
    return merge_shards(gathered, len(items))
