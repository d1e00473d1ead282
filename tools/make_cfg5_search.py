"""Golden grouping-search results of the whole cfg5 sweep (tests/golden/cfg5_search.json):
for every snapshot and valid TP dimension, the reference's nodes_visited, optimal flag,
winner objective (hex) and winner RGS, from the pinned C restatement
(oracle/_ref/libhpo.so, checked against the reference probe by tests/test_oracle.py).
The GPU test runs all 1167 searches in one batch and compares each.
Run: python tools/make_cfg5_search.py   (~1 min on 8 cores)"""
import json
import math
import os
import sys
from multiprocessing import Pool

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle.binding import Oracle
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
    r = Oracle().solve_grouping(P, M, K, MIN, T, N)
    rec = {"snapshot": si, "tp": tp, "status": r.status}
    if r.status == 0:
        rec.update({"visited": r.visited, "optimal": r.optimal,
                    "objective": r.objective[0].hex(),
                    "rgs": "".join(chr(48 + x) for x in r.rgs[0])})
    return rec


if __name__ == "__main__":
    with Pool(os.cpu_count()) as pool:
        recs = pool.map(solve, problems(), chunksize=4)
    with open(os.path.join(ROOT, "tests", "golden", "cfg5_search.json"), "w") as f:
        json.dump(recs, f, separators=(",", ":"))
    print("wrote", len(recs), "searches,", sum(r.get("visited", 0) for r in recs), "visits")
