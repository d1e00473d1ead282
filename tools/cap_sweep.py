import sys, time
sys.path.insert(0, '/root/repo')
from oracle.binding import min_mem_for, units_for
from paper_2512_20953_b200 import configs
from paper_2512_20953_b200.engine import Engine, GroupingProblem
import math
eng = Engine()
name = sys.argv[1]
w = configs.get(name)
g = 0
for nd in w.cluster["nodes"]:
    g = math.gcd(g, nd["count"])
probs = []
for tp in [t for t in range(1, g + 1) if g % t == 0]:
    P, M, T, N = units_for(w.cluster, tp)
    probs.append(GroupingProblem(P, M, w.model["n_microbatches"], min_mem_for(w.model), T, N))
for cap in [int(x) for x in sys.argv[2].split(",")]:
    best = 1e9
    for rep in range(3):
        eng.reset_timing()
        res = eng.grouping_search(probs, segment_cap=cap, max_seconds=30)
        t = eng.timing()
        best = min(best, t.search_ms)
    print(f"{name} cap {cap}: best kernel {best:.2f} ms, waves {[r.waves for r in res]}, run_visits {[r.segment_visits for r in res]}, max_list {[r.max_list for r in res]}", flush=True)
