import sys
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
from oracle.binding import Oracle
from paper_2512_20953_b200.engine import Engine
from test_gpu_grouping import _random_problems
eng = Engine(); orc = Oracle()
probs = _random_problems(3, 160, nmax=10)
pb = probs[143]
print(pb, flush=True)
o = orc.solve_grouping(pb.power, pb.memory, pb.n_microbatches, pb.min_mem, pb.type_key, pb.node_key, pb.exact_threshold, pb.node_budget)
print("oracle", o.rgs, o.objective, o.visited, o.optimal, flush=True)
for rep in range(3):
    try:
        r = eng.grouping_search(probs, segment_cap=3, max_seconds=10, max_waves=3000)
        print("batch rep", rep, "p143", r[143].visited, r[143].rgs, flush=True)
    except Exception as e:
        print("batch rep", rep, "ERR", e, flush=True)
