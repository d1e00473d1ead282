import sys
sys.path.insert(0, '/root/repo')
from oracle.binding import min_mem_for, units_for
from paper_2512_20953_b200 import configs
from paper_2512_20953_b200.engine import Engine, GroupingProblem
eng = Engine()
w = configs.get(sys.argv[1]); tps = [int(x) for x in sys.argv[2].split(",")]
probs = []
for tp in tps:
    P, M, T, N = units_for(w.cluster, tp)
    probs.append(GroupingProblem(P, M, w.model["n_microbatches"], min_mem_for(w.model), T, N))
res = eng.grouping_search(probs, max_seconds=60)
print("ok", [r.visited for r in res], [r.waves for r in res], eng.timing().search_ms, flush=True)
