"""The N>1 path's host logic on CPU: round-robin sharding of independent
searches over 2 gloo ranks, one all-gather, identical merged results on every
rank and equal to the serial run (the oracle stands in for the per-rank GPU
search here; the GPU search itself is covered by the gpu tests)."""
import os
import random

import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2512_20953_b200 import cases
from paper_2512_20953_b200.shard import merge_shards, shard_indices, sharded_map


def _problems():
    rng = random.Random(7)
    return [p for p in cases.grouping_cases(rng, 40) if len(p["power"]) <= 9][:9]


def _solve(batch):
    from oracle.binding import Oracle
    o = Oracle()
    out = []
    for p in batch:
        r = o.solve_grouping(p["power"], p["memory"], p["K"], p["min_mem"], p["type_key"],
                             p["node_key"], p["exact_threshold"], p["node_budget"],
                             max(1, p["top_k"]))
        out.append((r.visited, r.optimal, [list(x) for x in r.rgs], list(r.objective)))
    return out


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        got = sharded_map(_problems(), _solve, dist)
        q.put((rank, got))
    finally:
        dist.destroy_process_group()


def test_shard_indices_partition():
    for n in range(0, 12):
        for world in (1, 2, 3, 8):
            idx = sorted(i for r in range(world) for i in shard_indices(n, r, world))
            assert idx == list(range(n))
    assert merge_shards([[0, 2, 4], [1, 3]], 5) == [0, 1, 2, 3, 4]
    with pytest.raises(ValueError):
        merge_shards([[0], [1]], 5)


def test_two_rank_gloo_matches_serial():
    serial = _solve(_problems())
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + random.Random(os.getpid()).randint(0, 999)
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert res[0] == res[1] == serial


def test_longest_first_sharding_isolates_the_slowest_search():
    # cfg4's TP dims: tp1 (64 units), tp2 (32), tp4 (16) budgeted, tp8 (8) exhaustive
    from types import SimpleNamespace
    from paper_2512_20953_b200.shard import search_cost
    probs = [SimpleNamespace(n=n, exact_threshold=8) for n in (64, 32, 16, 8)]
    costs = [search_cost(p) for p in probs]
    assert [shard_indices(4, r, 2, costs) for r in range(2)] == [[0], [1, 2, 3]]
    assert [shard_indices(4, r, 4, costs) for r in range(4)] == [[0], [1], [2], [3]]
    parts = [shard_indices(4, r, 3, costs) for r in range(3)]
    assert sorted(i for p in parts for i in p) == [0, 1, 2, 3]
    assert merge_shards([["a"], ["b", "c", "d"]], 4, costs) == ["a", "b", "c", "d"]
