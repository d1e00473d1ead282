"""Reference grouping-visit counts of the first cfg5 snapshots (tests/golden/cfg5_visits.json).

bench.py --impl reference --workload cfg5 times the reference planner on a
sample of these snapshots and needs each plan's candidate count (the sum of
GroupingSolution::nodes_visited over TP dimensions); the reference C ABI does
not report it, so it is computed here once with the reference probe
(oracle/_ref/libhetplan_probe.so). Run: python tools/make_cfg5_visits.py
"""
import json
import math
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle.binding import Oracle
from paper_2512_20953_b200.configs import min_mem_for, units_for  # noqa: E402
from paper_2512_20953_b200 import configs  # noqa: E402


def main(count=64):
    o = Oracle()
    out = []
    for w in configs.cfg5_snapshots(count):
        g = 0
        for nd in w.cluster["nodes"]:
            g = math.gcd(g, nd["count"])
        vis = 0
        for tp in [t for t in range(1, g + 1) if g % t == 0]:
            P, M, T, N = units_for(w.cluster, tp)
            if sum(M) < min_mem_for(w.model):
                continue
            r = o.solve_grouping(P, M, w.model["n_microbatches"], min_mem_for(w.model), T, N)
            vis += r.visited
        out.append({"name": w.name, "visits": vis})
    with open(os.path.join(ROOT, "tests", "golden", "cfg5_visits.json"), "w") as f:
        json.dump(out, f, indent=0)
    print("wrote", len(out), "snapshots")


if __name__ == "__main__":
    main()
