"""GPU parity of the grouping search (the hot loop) against the oracle and the
reference's golden vectors: winner RGS, objective and z bit-exact, visits and
the optimal flag identical — exhaustive and budget-truncated, both engines."""
import math
import random

import pytest

from paper_2512_20953_b200.configs import min_mem_for, units_for
from paper_2512_20953_b200 import configs
from paper_2512_20953_b200.engine import GroupingProblem

pytestmark = pytest.mark.gpu


def _same(r, o):
    if o.status != 0:
        return r.status == o.status
    return (r.status == 0 and r.count == o.count and r.rgs == o.rgs
            and r.objective == o.objective and r.z == o.z and r.visited == o.visited
            and r.optimal == o.optimal)


def _random_problems(seed, count, nmax=11, top_ks=(1,)):
    rng = random.Random(seed)
    out = []
    for t in range(count):
        topk = rng.choice(top_ks) if len(top_ks) > 1 else top_ks[0]
        n = rng.randint(1, nmax)
        if t % 5 == 0:
            P = [2.0] * n  # heavy ties
            M = [8.0] * n
        else:
            P = [rng.choice([0.5, 1.0, 1.5, 2.0, 3.0]) for _ in range(n)]
            M = [float(rng.randint(4, 20)) for _ in range(n)]
        T = [int(p * 2) for p in P]
        N = sorted(rng.randint(0, 3) for _ in range(n))
        K = rng.randint(1, 16)
        MIN = sum(M) * rng.uniform(0.1, 0.9) / rng.randint(1, 4)
        if rng.random() < 0.5:
            MIN = float(round(MIN))
        thr = rng.choice([0, 4, 8])
        B = rng.choice([0, 1, 2, 17, 300, 3000, 20000])
        out.append(GroupingProblem(P, M, K, MIN, T, N, thr, B, topk))
    return out


@pytest.mark.parametrize("cap", [3, 64, 2048])
def test_wave_engine_random_batch(engine, oracle, cap):
    probs = _random_problems(cap, 160, nmax=10 if cap < 16 else 11)
    res = engine.grouping_search(probs, segment_cap=cap, max_seconds=60)
    bad = []
    for pb, r in zip(probs, res):
        o = oracle.solve_grouping(pb.power, pb.memory, pb.n_microbatches, pb.min_mem,
                                  pb.type_key, pb.node_key, pb.exact_threshold, pb.node_budget)
        if not _same(r, o):
            bad.append((pb, r, o.rgs, o.objective, o.visited, o.optimal))
        assert r.engine == 0
    assert not bad, bad[:2]


@pytest.mark.parametrize("cap", [3, 64, 2048])
def test_wave_engine_top_k_random_batch(engine, oracle, cap):
    """top_k > 1 on the wave engine: the cutoff state is the top_k vector
    (grouping.cpp:117-132); every returned candidate, visits and the optimal
    flag match the oracle."""
    probs = _random_problems(1000 + cap, 160, nmax=10 if cap < 16 else 11,
                             top_ks=(2, 3, 4, 8, 13, 16))
    res = engine.grouping_search(probs, segment_cap=cap, max_seconds=60)
    bad = []
    for pb, r in zip(probs, res):
        o = oracle.solve_grouping(pb.power, pb.memory, pb.n_microbatches, pb.min_mem,
                                  pb.type_key, pb.node_key, pb.exact_threshold, pb.node_budget,
                                  pb.top_k)
        if not _same(r, o):
            bad.append((pb, r, o.rgs, o.objective, o.visited, o.optimal))
        assert r.engine == 0
    assert not bad, bad[:2]


@pytest.mark.parametrize("name,k", [("cfg2", 2), ("cfg3", 3), ("cfg4", 2), ("cfg4", 8),
                                    ("cfg2", 12), ("cfg3", 16)])
def test_configs_top_k_every_tp_dimension(engine, oracle, name, k):
    w = configs.get(name)
    g = 0
    for nd in w.cluster["nodes"]:
        g = math.gcd(g, nd["count"])
    probs = []
    for tp in [t for t in range(1, g + 1) if g % t == 0]:
        P, M, T, N = units_for(w.cluster, tp)
        probs.append(GroupingProblem(P, M, w.model["n_microbatches"], min_mem_for(w.model), T, N,
                                     top_k=k))
    res = engine.grouping_search(probs, max_seconds=60)
    for pb, r in zip(probs, res):
        o = oracle.solve_grouping(pb.power, pb.memory, pb.n_microbatches, pb.min_mem,
                                  pb.type_key, pb.node_key, top_k=k)
        assert r.engine == 0
        assert _same(r, o), (name, k, pb.n, r.objective, o.objective, r.visited, o.visited)


def test_serial_engine_random_batch(engine, oracle):
    probs = _random_problems(99, 120, nmax=10)
    res = engine.grouping_search(probs, force_serial=True, max_seconds=60)
    for pb, r in zip(probs, res):
        o = oracle.solve_grouping(pb.power, pb.memory, pb.n_microbatches, pb.min_mem,
                                  pb.type_key, pb.node_key, pb.exact_threshold, pb.node_budget)
        assert r.engine == 1
        assert _same(r, o), (pb, r)


def test_golden_grouping_vectors(engine, golden_grouping):
    probs = [GroupingProblem(g["power"], g["memory"], g["K"], g["min_mem"], g["type_key"],
                             g["node_key"], g["exact_threshold"], g["node_budget"], g["top_k"])
             for g in golden_grouping]
    res = engine.grouping_search(probs, max_seconds=60)
    for g, r in zip(golden_grouping, res):
        assert r.status == g["status"], g
        if g["status"] != 0:
            continue
        assert r.count == g["count"]
        assert r.rgs == g["rgs"]
        assert [x.hex() for x in r.objective] == g["objective"]
        assert [x.hex() for x in r.z] == g["z"]
        assert r.optimal == g["optimal"] and r.visited == g["visited"]


@pytest.mark.parametrize("name", ["cfg1", "cfg2", "cfg3", "cfg4"])
def test_configs_every_tp_dimension(engine, oracle, name):
    w = configs.get(name)
    g = 0
    for nd in w.cluster["nodes"]:
        g = math.gcd(g, nd["count"])
    probs = []
    for tp in [t for t in range(1, g + 1) if g % t == 0]:
        P, M, T, N = units_for(w.cluster, tp)
        probs.append(GroupingProblem(P, M, w.model["n_microbatches"], min_mem_for(w.model), T, N))
    res = engine.grouping_search(probs, max_seconds=60)
    for pb, r in zip(probs, res):
        o = oracle.solve_grouping(pb.power, pb.memory, pb.n_microbatches, pb.min_mem,
                                  pb.type_key, pb.node_key)
        assert _same(r, o), (name, pb.n)
        # the filter must decide almost every child check itself: a compiler that
        # folds the PASS outcome away stays exact but shows up here
        if r.engine == 0:
            assert r.exact_checks <= max(16, r.segment_visits // 1000), (name, pb.n)


def test_non_dyadic_and_large_top_k(engine, oracle):
    nd = GroupingProblem([1.0, 1.0, 2.0, 0.7, 1.3], [8.0, 8.0, 8.0, 9.0, 7.0], 8, 6.0,
                         [0, 0, 1, 2, 3], [0, 0, 1, 2, 3], top_k=3)
    big = GroupingProblem([1.0, 1.0, 2.0, 0.5, 1.5, 2.0], [8.0, 8.0, 8.0, 9.0, 7.0, 4.0], 8, 6.0,
                          [0, 0, 1, 2, 3, 1], [0, 0, 1, 2, 3, 3], top_k=20)
    mid = GroupingProblem(big.power, big.memory, 8, 6.0, big.type_key, big.node_key, top_k=12)
    small = GroupingProblem(big.power, big.memory, 8, 6.0, big.type_key, big.node_key, top_k=3)
    # top_k <= 16 runs on the wave engine; larger top_k (beyond the old limit,
    # the reference accepts any) on the serial replica with a top_k-long list
    res = engine.grouping_search([nd, big, mid, small])
    # non-dyadic sums: the wave engine if no += drifts, else the serial replica
    assert [r.engine for r in res][1:] == [1, 0, 0] and res[0].engine in (0, 1)
    assert res[1].count > 16
    for pb, r in zip([nd, big, mid, small], res):
        o = oracle.solve_grouping(pb.power, pb.memory, 8, 6.0, pb.type_key, pb.node_key,
                                  top_k=pb.top_k)
        assert _same(r, o)


def _host_decide(A, D, rem, cut, mb, md):
    has_cut = cut >= 0
    if (has_cut and A + mb < cut) or (D - md > rem):
        return 1
    b_pass = (not has_cut) or (A - mb >= cut)
    return 0 if (b_pass and D + md <= rem) else 2


def test_device_filter_decision_matches_host(engine):
    """Pins decide(): an equivalent if/else-chain formulation was miscompiled
    by nvcc 12.9 for sm_100a (never returned PASS) — DESIGN.md 2.3."""
    import ctypes as C
    rm = [0.0, 0.0, 100.0, 0.0]
    cases = []
    for A in (10.0, 50.0, 50.0 + 1e-12, 90.0):
        for D in (50.0, 100.0, 100.0 + 1e-12, 150.0):
            for cut in (-1.0, 0.0, 50.0, 60.0):
                cases.append((A, D, cut))
    flat = [v for c in cases for v in c]
    lib = engine.lib
    lib.hpk_selftest_decide.argtypes = [C.POINTER(C.c_double), C.c_int, C.POINTER(C.c_double),
                                        C.c_double, C.c_double, C.POINTER(C.c_int)]
    for mb in (0.0, 1e-9):
        for md in (0.0, 1e-9):
            out = (C.c_int * len(cases))()
            rc = lib.hpk_selftest_decide((C.c_double * len(flat))(*flat), len(cases),
                                         (C.c_double * 4)(*rm), mb, md, out)
            assert rc == 0
            want = [_host_decide(A, D, 100.0, cut, mb, md) for (A, D, cut) in cases]
            assert list(out) == want


def test_enumeration_engine_matches_the_dfs_winner(engine, oracle):
    """Exhaustive top-1 searches on the enumeration engine (planner path): the
    winner (RGS, objective, z) equals the reference DFS's — SURVEY.md fact 4."""
    probs = [GroupingProblem(pb.power, pb.memory, pb.n_microbatches, pb.min_mem, pb.type_key,
                             pb.node_key, 12, pb.node_budget)
             for pb in _random_problems(77, 300, nmax=12)]
    res = engine.grouping_search(probs, enumeration=True, max_seconds=60)
    for pb, r in zip(probs, res):
        o = oracle.solve_grouping(pb.power, pb.memory, pb.n_microbatches, pb.min_mem,
                                  pb.type_key, pb.node_key, 12, pb.node_budget)
        assert r.engine == 2
        if o.status != 0:
            assert r.status == o.status
            continue
        assert (r.status, r.rgs, r.objective, r.z, r.optimal) == \
            (0, o.rgs, o.objective, o.z, o.optimal), pb


def test_enumeration_engine_top_k(engine, oracle):
    """Exhaustive top-k on the enumeration engine: the global top k when at least
    k feasible leaves reach the prune floor, else the wave engine takes over —
    either way the list equals the reference DFS's."""
    probs = [GroupingProblem(pb.power, pb.memory, pb.n_microbatches, pb.min_mem, pb.type_key,
                             pb.node_key, 12, pb.node_budget, pb.top_k)
             for pb in _random_problems(78, 300, nmax=12, top_ks=(2, 3, 5, 8))]
    res = engine.grouping_search(probs, enumeration=True, max_seconds=60)
    engines = set()
    for pb, r in zip(probs, res):
        o = oracle.solve_grouping(pb.power, pb.memory, pb.n_microbatches, pb.min_mem,
                                  pb.type_key, pb.node_key, 12, pb.node_budget, pb.top_k)
        engines.add(r.engine)
        if o.status != 0:
            assert r.status == o.status
            continue
        assert (r.status, r.count, r.rgs, r.objective, r.z, r.optimal) == \
            (0, o.count, o.rgs, o.objective, o.z, o.optimal), pb
    assert 2 in engines


def test_wave_engine_up_to_128_units(engine, oracle):
    """65..128 TP units run on the wave engine (lanes own groups g and g+32, so a
    node may hold up to 64 groups); budgeted searches over such clusters match
    the oracle exactly (visits, optimal flag, winner)."""
    import random
    rng = random.Random(72)
    probs = []
    for n in (65, 72, 96, 128, 72, 80):
        P = [rng.choice([1.0, 1.5, 2.0]) for _ in range(n)]
        M = [rng.choice([40e9, 80e9, 100e9]) for _ in range(n)]
        T = [int(p * 2) for p in P]
        N = [i // 8 for i in range(n)]
        MIN = sum(M) / rng.choice([3, 6, 12])
        probs.append(GroupingProblem(P, M, rng.choice([16, 64]), MIN, T, N,
                                     node_budget=rng.choice([20000, 300000])))
    res = engine.grouping_search(probs, max_seconds=120)
    for pb, r in zip(probs, res):
        o = oracle.solve_grouping(pb.power, pb.memory, pb.n_microbatches, pb.min_mem,
                                  pb.type_key, pb.node_key, pb.exact_threshold, pb.node_budget)
        assert r.engine == 0, pb.n
        assert _same(r, o), (pb.n, r.visited, o.visited)


def test_more_than_63_groups_falls_back_exactly(engine, oracle):
    """K = 1 and equal powers: every merge is pruned by the singletons seed, so
    the DFS walks straight down opening a new group per unit and reaches an
    internal node with 64 groups (65 children) — beyond the lanes' slots. The
    wave engine hands such a problem to the serial replica; the result stays
    the reference's."""
    n = 70
    pb = GroupingProblem([1.0] * n, [8.0] * n, 1, 1.0, [0] * n, list(range(n)))
    r = engine.grouping_search([pb], max_seconds=120)[0]
    o = oracle.solve_grouping(pb.power, pb.memory, 1, 1.0, pb.type_key, pb.node_key)
    assert r.engine == 1
    assert _same(r, o)


def test_non_dyadic_sums_exact_with_drift_check(engine, oracle):
    """Unit powers outside the exact-sum contract (derive_power ratios): the
    wave engine runs them while checking every += for drift
    (fl(fl(x+p)-p) != x, the reference's path-dependent sums, grouping.cpp:184-198)
    and hands drifting problems to the serial replica. Either way the result is
    the reference's; both engines must actually occur in the batch."""
    rng = random.Random(314)
    probs = []
    for _ in range(160):
        n = rng.randint(4, 11)
        base = rng.choice([[1.0, 2.0, 1.5], [1.0, 0.7, 1.3], [1.0, 1 / 3, 2 / 3],
                           [1.0, 1.4999999999999998, 2.0000000000000004], [0.1, 0.2, 0.3]])
        P = [rng.choice(base) for _ in range(n)]
        M = [rng.choice([8.0, 10.0, 16.0]) for _ in range(n)]
        T = [base.index(x) for x in P]
        N = sorted(rng.randint(0, 3) for _ in range(n))
        K = rng.choice([1, 4, 16])
        MIN = float(rng.choice([8, 16, 24, 32]))
        probs.append(GroupingProblem(P, M, K, MIN, T, N, exact_threshold=rng.choice([0, 8]),
                                     node_budget=rng.choice([50, 500, 5000])))
    res = engine.grouping_search(probs, segment_cap=rng.choice([3, 64]), max_seconds=120)
    engines = set()
    for pb, r in zip(probs, res):
        o = oracle.solve_grouping(pb.power, pb.memory, pb.n_microbatches, pb.min_mem,
                                  pb.type_key, pb.node_key, pb.exact_threshold, pb.node_budget)
        assert _same(r, o), (pb, r.engine)
        engines.add(r.engine)
    assert engines == {0, 1}
