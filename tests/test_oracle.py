"""The oracle (oracle/hetplan_oracle.c) pinned to the reference: against the
committed golden vectors (generated from the reference library by
tools/make_golden.py) and, when the reference probe is built, directly."""
import ctypes as C
import os
import random

import pytest

from oracle.binding import PROBE_LIB
from paper_2512_20953_b200.configs import min_mem_for, units_for
from paper_2512_20953_b200 import cases, configs


def _f(h):
    return float.fromhex(h)


def test_oracle_matches_golden_grouping(oracle, golden_grouping):
    assert len(golden_grouping) >= 300
    for rec in golden_grouping:
        o = oracle.solve_grouping(rec["power"], rec["memory"], rec["K"], rec["min_mem"],
                                  rec["type_key"], rec["node_key"], rec["exact_threshold"],
                                  rec["node_budget"], rec["top_k"])
        assert o.status == rec["status"], rec
        if rec["status"] != 0:
            continue
        assert o.count == rec["count"]
        assert o.rgs == rec["rgs"]
        assert [x.hex() for x in o.objective] == rec["objective"]
        assert [x.hex() for x in o.z] == rec["z"]
        assert o.optimal == rec["optimal"]
        assert o.visited == rec["visited"]


def test_oracle_matches_golden_partition(oracle, golden_partition):
    for rec in golden_partition:
        rc, layers, times, bn, _, _ = oracle.balance_workload(
            rec["n_layers"], rec["prof"], rec["mem_capacity"], rec["stage_index"], rec["tp"],
            rec["ppb"], rec["pab"], rec["opt_mult"], rec["k_total"])
        assert rc == rec["status"], rec
        if rc == 0:
            assert layers == rec["layers"]
            assert [t.hex() for t in times] == rec["times"]
            assert bn.hex() == rec["bottleneck"]


# The reference's own known answers (P/tests/test_grouping.cpp, test_partition.cpp,
# test_profile.cpp, acceptance.cpp C9).
def test_known_answer_two_a100_one_h800(oracle):
    o = oracle.solve_grouping([1.0, 1.0, 2.0], [10.0, 10.0, 10.0], 8, 5.0, [0, 0, 1], [0, 0, 1])
    assert o.count == 1 and o.optimal
    assert o.rgs[0][0] == o.rgs[0][1] != o.rgs[0][2]
    assert abs(o.objective[0] - 32.0 / 9.0) < 1e-12
    assert abs(o.z[0] - 16.0 / 9.0) < 1e-12


def test_known_answer_budget_abort(oracle):
    # test_grouping.cpp:222-247: 12 identical units, threshold 4, budget 50
    o = oracle.solve_grouping([1.0] * 12, [8.0] * 12, 8, 4.0, [0] * 12, list(range(12)), 4, 50)
    assert not o.optimal and o.objective[0] > 0 and o.visited == 50
    full = oracle.solve_grouping([1.0] * 12, [8.0] * 12, 8, 4.0, [0] * 12, list(range(12)), 12,
                                 50_000_000)
    assert full.optimal and full.objective[0] >= o.objective[0]


def test_known_answer_tie_break(oracle):
    # test_grouping.cpp:202-220: K=1, two identical devices -> two singletons, objective 2
    o = oracle.solve_grouping([1.0, 1.0], [4.0, 4.0], 1, 2.0, [0, 0], [0, 0])
    assert o.rgs[0] == [0, 1] and o.objective[0] == 2.0


def test_known_answer_proportional_partition(oracle):
    # acceptance.cpp C4 tail: powers (1,1,2,2), 24 layers -> (4,4,8,8); linear profile
    rows = []
    for pw in (1.0, 1.0, 2.0, 2.0):
        rows.append([(1 << b) / pw for b in range(5)])
    rc, layers, times, bn, _, _ = oracle.balance_workload(24, rows, [1e300] * 4, [1, 2, 3, 4], 1,
                                                          0.0, 0.0, 0.0, 8)
    assert rc == 0 and layers == [4, 4, 8, 8] and len(set(times)) == 1


def test_binary_decomposition_exact(oracle):
    # acceptance.cpp C9: T(n) == c*n for c = 0.25 over n in 1..64
    row = [0.25 * (1 << b) for b in range(7)]
    rowp = (C.c_double * 7)(*row)
    for n in range(1, 65):
        assert oracle.lib.hpo_stage_time(rowp, 7, n) == 0.25 * n


def test_stage_time_is_ascending_bit_sum(oracle):
    # test_profile.cpp:51-66 style: 5 layers = T(1) + T(4) in that order
    row = [0.1, 0.7, 5.0]
    rowp = (C.c_double * 3)(*row)
    assert oracle.lib.hpo_stage_time(rowp, 3, 5) == 0.1 + 5.0
    assert oracle.lib.hpo_stage_time(rowp, 3, 7) == (0.1 + 0.7) + 5.0


@pytest.mark.skipif(not os.path.exists(PROBE_LIB), reason="reference probe not built")
@pytest.mark.parametrize("name", ["cfg1", "cfg2", "cfg3", "cfg4"])
def test_oracle_matches_reference_on_configs(oracle, name):
    probe = C.CDLL(PROBE_LIB)
    w = configs.get(name)
    import math
    g = 0
    for nd in w.cluster["nodes"]:
        g = math.gcd(g, nd["count"])
    for tp in [t for t in range(1, g + 1) if g % t == 0]:
        P, M, T, N = units_for(w.cluster, tp)
        n = len(P)
        mm = min_mem_for(w.model)
        K = w.model["n_microbatches"]
        o = oracle.solve_grouping(P, M, K, mm, T, N)
        cnt = C.c_int()
        rgs = (C.c_int * n)()
        obj = (C.c_double * 1)()
        z = (C.c_double * 1)()
        opt = C.c_int()
        vis = C.c_longlong()
        D = lambda a: (C.c_double * len(a))(*a)  # noqa: E731
        I = lambda a: (C.c_int * len(a))(*a)  # noqa: E731
        rc = probe.ref_solve_grouping(n, D(P), D(M), I(T), I(N), K, C.c_double(mm), 8,
                                      C.c_longlong(5_000_000), 1, C.byref(cnt), rgs, obj, z,
                                      C.byref(opt), C.byref(vis))
        assert rc == 0
        assert o.rgs[0] == list(rgs)
        assert o.objective[0] == obj[0] and o.z[0] == z[0]
        assert o.visited == vis.value and o.optimal == bool(opt.value)
