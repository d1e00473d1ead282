"""cfg5 snapshot grouping searches in one wave-kernel launch (profiling target)."""
import math
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2512_20953_b200.configs import min_mem_for, units_for
from paper_2512_20953_b200 import configs
from paper_2512_20953_b200.engine import Engine, GroupingProblem
n = int(sys.argv[1]) if len(sys.argv) > 1 else 100
eng = Engine()
probs = []
for w in configs.cfg5_snapshots(n):
    g = 0
    for nd in w.cluster["nodes"]:
        g = math.gcd(g, nd["count"])
    for tp in [t for t in range(1, g + 1) if g % t == 0]:
        P, M, T, N = units_for(w.cluster, tp)
        probs.append(GroupingProblem(P, M, w.model["n_microbatches"], min_mem_for(w.model), T, N))
res = eng.grouping_search(probs, max_seconds=60)
t = eng.timing()
v = sum(r.visited for r in res)
print("ok", len(probs), "problems", v, "visits", t.search_ms, "ms", v / t.search_ms / 1e6, "Gvis/s",
      "exec", sum(r.segment_visits for r in res))
