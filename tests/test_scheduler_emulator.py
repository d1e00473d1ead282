"""The wave scheduler's algorithm (tests/emu/wave_emulator.cpp: ordered
segments, speculative waves, splitting, commit walk, end-marker re-runs,
budget cut) is exact: it reproduces the serial DFS (the oracle) on random
instances, with tiny caps and list capacities so every path is exercised."""
import ctypes as C
import os
import random
import subprocess

import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "emu", "wave_emulator.cpp")
LIB = os.path.join(HERE, "..", "build", "emu", "libwave_emu.so")


@pytest.fixture(scope="module")
def emu():
    os.makedirs(os.path.dirname(LIB), exist_ok=True)
    if not os.path.exists(LIB) or os.path.getmtime(LIB) < os.path.getmtime(SRC):
        subprocess.check_call(["g++", "-std=c++17", "-O2", "-fPIC", "-shared",
                               "-ffp-contract=off", "-o", LIB, SRC])
    return C.CDLL(LIB)


def _d(a):
    return (C.c_double * len(a))(*a)


def _i(a):
    return (C.c_int * len(a))(*a)


def emulate(emu, oracle, P, M, T, N, K, MIN, thr, B, nw, cap, maxl):
    n = len(P)
    srgs = (C.c_int * n)()
    sz = C.c_double()
    floor = oracle.lib.hpo_seed_floor(n, _d(P), _d(M), _i(T), _i(N), K, C.c_double(MIN), srgs,
                                      C.byref(sz))
    if sum(M) < MIN:
        return (3,)
    budget = -1 if n <= thr else B
    rgs = (C.c_int * n)()
    obj = C.c_double()
    has = C.c_int()
    vis = C.c_longlong()
    ab = C.c_int()
    waves = C.c_int()
    runs = C.c_longlong()
    rv = C.c_longlong()
    ml = C.c_int()
    emu.emu_search(n, _d(P), _d(M), K, C.c_double(MIN), C.c_longlong(budget), C.c_double(floor),
                   nw, C.c_longlong(cap), maxl, rgs, C.byref(obj), C.byref(has), C.byref(vis),
                   C.byref(ab), C.byref(waves), C.byref(runs), C.byref(rv), C.byref(ml))
    if not has.value:
        if floor < 0:
            return (3,)
        return (0, list(srgs), floor, 0, vis.value)
    if ab.value and floor > obj.value:
        return (0, list(srgs), floor, 0, vis.value)
    return (0, list(rgs), obj.value, 0 if ab.value else 1, vis.value)


def test_emulator_matches_oracle(emu, oracle):
    rng = random.Random(11)
    for _ in range(600):
        n = rng.randint(1, 9)
        P = [rng.choice([0.5, 1.0, 1.5, 2.0, 3.0]) for _ in range(n)]
        M = [float(rng.randint(4, 20)) for _ in range(n)]
        T = [int(p * 2) for p in P]
        N = sorted(rng.randint(0, 3) for _ in range(n))
        K = rng.randint(1, 16)
        MIN = sum(M) * rng.uniform(0.1, 0.9) / rng.randint(1, 4)
        if rng.random() < 0.5:
            MIN = float(round(MIN))
        thr = rng.choice([0, 8, 100])
        B = rng.randint(1, 2000)
        nw = rng.choice([1, 2, 3, 8, 64])
        cap = rng.choice([1, 2, 3, 5, 17, 100])
        maxl = rng.choice([4, 16, 1000])
        o = oracle.solve_grouping(P, M, K, MIN, T, N, thr, B)
        e = emulate(emu, oracle, P, M, T, N, K, MIN, thr, B, nw, cap, maxl)
        if o.status != 0:
            assert e[0] == o.status
        else:
            assert e == (0, o.rgs[0], o.objective[0], int(o.optimal), o.visited)


ASYNC_SRC = os.path.join(HERE, "emu", "async_emulator.cpp")
ASYNC_LIB = os.path.join(HERE, "..", "build", "emu", "libasync_emu.so")


@pytest.fixture(scope="module")
def async_emu():
    os.makedirs(os.path.dirname(ASYNC_LIB), exist_ok=True)
    if not os.path.exists(ASYNC_LIB) or os.path.getmtime(ASYNC_LIB) < os.path.getmtime(ASYNC_SRC):
        subprocess.check_call(["g++", "-std=c++17", "-O2", "-fPIC", "-shared",
                               "-ffp-contract=off", "-o", ASYNC_LIB, ASYNC_SRC])
    return C.CDLL(ASYNC_LIB)


def test_async_scheduler_emulator_matches_oracle(async_emu, oracle):
    """The asynchronous (wave-free) scheduler design — on-demand splits of the
    front-most runs, time-slice preemption into a preorder-ordered ready set,
    stale-run restarts, ordered commit with end-marker re-runs and the budget
    cut (tests/emu/async_emulator.cpp) — is exact."""
    rng = random.Random(5)
    checked = 0
    while checked < 250:
        n = rng.randint(2, 10)
        P = [rng.choice([0.5, 1.0, 1.5, 2.0]) for _ in range(n)]
        M = [rng.choice([4.0, 8.0, 10.0, 16.0]) for _ in range(n)]
        T = [rng.randint(0, 2) for _ in range(n)]
        N = [rng.randint(0, 4) for _ in range(n)]
        K = rng.choice([1, 2, 8, 16])
        MIN = rng.choice([4.0, 8.0, 16.0, 24.0])
        if sum(M) < MIN:
            continue
        B = rng.choice([3, 10, 50, 300, 3000, 10 ** 9])
        o = oracle.solve_grouping(P, M, K, MIN, T, N, 0, B)
        srgs = (C.c_int * n)()
        sz = C.c_double()
        floor = oracle.lib.hpo_seed_floor(n, _d(P), _d(M), _i(T), _i(N), K, C.c_double(MIN),
                                          srgs, C.byref(sz))
        rgs = (C.c_int * n)()
        obj, has, vis, ab, tt = C.c_double(), C.c_int(), C.c_longlong(), C.c_int(), C.c_double()
        st = (C.c_longlong * 5)()
        async_emu.async_emu_search(
            n, _d(P), _d(M), K, C.c_double(MIN), C.c_longlong(B), C.c_double(floor),
            rng.choice([1, 2, 4, 16]), C.c_double(rng.choice([0, 1, 5])),
            C.c_double(rng.choice([0, 2, 9])), C.c_double(rng.choice([0, 1, 3])), C.c_double(2),
            rng.choice([0, 1]), rng.choice([0, 1]), C.c_longlong(rng.choice([1, 4])),
            C.c_longlong(rng.choice([0, 0, 50, 200])), C.c_longlong(rng.choice([0, 0, 7, 40])),
            rgs, C.byref(obj), C.byref(has),
            C.byref(vis), C.byref(ab), C.byref(tt), st)
        assert vis.value == o.visited and bool(ab.value) == (not o.optimal)
        if o.status == 0 and has.value and not (ab.value and floor > obj.value):
            assert list(rgs) == o.rgs[0] and obj.value == o.objective[0]
        checked += 1
