"""A/B the grouping-search kernel of two library builds on one config.
usage: python tools/ab_search.py CFG LIB_A LIB_B [reps]"""
import math
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2512_20953_b200.configs import min_mem_for, units_for  # noqa: E402
from paper_2512_20953_b200 import configs  # noqa: E402
from paper_2512_20953_b200.engine import Engine, GroupingProblem  # noqa: E402
w = configs.get(sys.argv[1])
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 5
g = 0
for nd in w.cluster["nodes"]:
    g = math.gcd(g, nd["count"])
probs = []
for tp in [t for t in range(1, g + 1) if g % t == 0]:
    P, M, T, N = units_for(w.cluster, tp)
    probs.append(GroupingProblem(P, M, w.model["n_microbatches"], min_mem_for(w.model), T, N))
for lib in sys.argv[2:4]:
    eng = Engine(lib)
    ts = []
    for _ in range(reps):
        eng.reset_timing()
        res = eng.grouping_search(probs, max_seconds=30)
        ts.append(eng.timing().search_ms)
    print(f"{lib}: min {min(ts):.2f} ms median {sorted(ts)[len(ts) // 2]:.2f} ms waves {[r.waves for r in res]}",
          flush=True)
