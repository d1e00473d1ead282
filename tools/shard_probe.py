"""Search time of a subset of a config's TP dimensions (what one rank runs at N>1)."""
import sys
sys.path.insert(0, "/root/repo")
from oracle.binding import min_mem_for, units_for  # noqa: E402
from paper_2512_20953_b200 import configs  # noqa: E402
from paper_2512_20953_b200.engine import Engine, GroupingProblem  # noqa: E402
eng = Engine()
w = configs.get(sys.argv[1])
for group in sys.argv[2:]:
    probs = []
    for tp in [int(x) for x in group.split(",")]:
        P, M, T, N = units_for(w.cluster, tp)
        probs.append(GroupingProblem(P, M, w.model["n_microbatches"], min_mem_for(w.model), T, N))
    ts = []
    for _ in range(5):
        eng.reset_timing()
        res = eng.grouping_search(probs, max_seconds=30)
        ts.append(eng.timing().search_ms)
    print(f"{sys.argv[1]} tp {group}: min {min(ts):.2f} ms waves {[r.waves for r in res]}", flush=True)
