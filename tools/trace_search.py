"""Grouping-search kernel time of a config's TP dimensions on a given library
build (e.g. a -DHPK_TRACE_LEVEL=n trace build: its per-wave log goes to stdout).
usage: python tools/trace_search.py LIB CFG TP[,TP...] [reps] [max_ctas] [max_list]"""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2512_20953_b200 import configs  # noqa: E402
from paper_2512_20953_b200.configs import min_mem_for, units_for  # noqa: E402
from paper_2512_20953_b200.engine import Engine, GroupingProblem  # noqa: E402

lib, name, tps = sys.argv[1], sys.argv[2], [int(x) for x in sys.argv[3].split(",")]
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 3
max_ctas = int(sys.argv[5]) if len(sys.argv) > 5 else 0
max_list = int(sys.argv[6]) if len(sys.argv) > 6 else 0
w = configs.get(name)
probs = []
for tp in tps:
    P, M, T, N = units_for(w.cluster, tp)
    probs.append(GroupingProblem(P, M, w.model["n_microbatches"], min_mem_for(w.model), T, N))
eng = Engine(lib)
for _ in range(reps):
    eng.reset_timing()
    res = eng.grouping_search(probs, device=0, max_ctas=max_ctas, max_list=max_list)
    t = eng.timing()
    print(f"[trace_search] {name} tp {tps}: search {t.search_ms:.2f} ms, waves "
          f"{[r.waves for r in res]}, visits {[r.visited for r in res]}, runs "
          f"{[r.segment_runs for r in res]}, run visits {[r.segment_visits for r in res]}",
          flush=True)
