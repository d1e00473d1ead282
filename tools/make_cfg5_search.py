"""Golden grouping-search results of the whole cfg5 sweep (tests/golden/cfg5_search.json):
for every snapshot and valid TP dimension, the reference's nodes_visited, optimal flag,
winner objective (hex) and winner RGS, from the REFERENCE itself: solve_grouping_topk
(P/src/grouping.cpp:269-335) through the probe oracle/_ref/libhetplan_probe.so.
The GPU test runs all 1167 searches in one batch and compares each.
Run: python tools/make_cfg5_search.py   (~1 min on 8 cores)"""
import json
import math
import os
import sys
from multiprocessing import Pool

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import ctypes as C

from oracle.binding import PROBE_LIB
from paper_2512_20953_b200.configs import min_mem_for, units_for  # noqa: E402
from paper_2512_20953_b200 import configs  # noqa: E402


def problems(count=1000):
    out = []
    for si, w in enumerate(configs.cfg5_snapshots(count)):
        g = 0
        for nd in w.cluster["nodes"]:
            g = math.gcd(g, nd["count"])
        for tp in [t for t in range(1, g + 1) if g % t == 0]:
            P, M, T, N = units_for(w.cluster, tp)
            out.append((si, tp, P, M, w.model["n_microbatches"], min_mem_for(w.model), T, N))
    return out


def solve(pb):
    si, tp, P, M, K, MIN, T, N = pb
    probe = C.CDLL(PROBE_LIB)
    n = len(P)
    D = lambda a: (C.c_double * len(a))(*a)  # noqa: E731
    I = lambda a: (C.c_int * len(a))(*a)  # noqa: E731
    cnt, opt, vis = C.c_int(), C.c_int(), C.c_longlong()
    rgs, obj, z = (C.c_int * n)(), (C.c_double * 1)(), (C.c_double * 1)()
    rc = probe.ref_solve_grouping(n, D(P), D(M), I(T), I(N), K, C.c_double(MIN), 8,
                                  C.c_longlong(5_000_000), 1, C.byref(cnt), rgs, obj, z,
                                  C.byref(opt), C.byref(vis))
    rec = {"snapshot": si, "tp": tp, "status": rc}
    if rc == 0:
        rec.update({"visited": vis.value, "optimal": bool(opt.value), "objective": obj[0].hex(),
                    "rgs": "".join(chr(48 + x) for x in rgs)})
    return rec


if __name__ == "__main__":
    with Pool(os.cpu_count()) as pool:
        recs = pool.map(solve, problems(), chunksize=4)
    with open(os.path.join(ROOT, "tests", "golden", "cfg5_search.json"), "w") as f:
        json.dump(recs, f, separators=(",", ":"))
    print("wrote", len(recs), "searches,", sum(r.get("visited", 0) for r in recs), "visits")
