import sys, os, time, math
sys.path.insert(0, '/root/repo')
from oracle.binding import Oracle, min_mem_for, units_for
from paper_2512_20953_b200 import configs
from paper_2512_20953_b200.engine import Engine, GroupingProblem
eng = Engine(); orc = Oracle()
name = sys.argv[1]; cap = int(sys.argv[2]); maxw = int(sys.argv[3])
tps = [int(x) for x in sys.argv[4].split(",")]
w = configs.get(name)
probs = []
for tp in tps:
    P, M, T, N = units_for(w.cluster, tp)
    probs.append(GroupingProblem(P, M, w.model["n_microbatches"], min_mem_for(w.model), T, N))
t = time.time()
try:
    rs = eng.grouping_search(probs, segment_cap=cap, max_waves=maxw, max_seconds=15)
    for r in rs:
        print("RESULT", r.visited, r.objective, r.optimal, r.waves, r.segment_runs, r.segment_visits, r.max_list, flush=True)
except Exception as e:
    print("ERR", e, flush=True)
print("time %.2f s kernel %.2f ms" % (time.time() - t, eng.timing().search_ms), flush=True)
