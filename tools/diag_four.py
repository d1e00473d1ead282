import sys
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
from oracle.binding import Oracle
from paper_2512_20953_b200.engine import Engine
from test_gpu_grouping import _random_problems
eng = Engine(); orc = Oracle()
cap = int(sys.argv[1]); reps = int(sys.argv[2])
probs = _random_problems(cap, 160, nmax=10 if cap < 16 else 11)
want = [orc.solve_grouping(pb.power, pb.memory, pb.n_microbatches, pb.min_mem, pb.type_key, pb.node_key, pb.exact_threshold, pb.node_budget) for pb in probs]
bad_total = 0
for rep in range(reps):
    res = eng.grouping_search(probs, segment_cap=cap, max_seconds=60)
    for i, (pb, r, o) in enumerate(zip(probs, res, want)):
        if o.status != 0:
            continue
        if (r.rgs, r.objective, r.visited, r.optimal) != (o.rgs, o.objective, o.visited, o.optimal):
            bad_total += 1
            if bad_total <= 6:
                print("rep", rep, "MISMATCH", i, "n", pb.n, "thr", pb.exact_threshold, "B", pb.node_budget)
                print("  gpu", r.rgs, r.objective, r.visited, r.optimal, "waves", r.waves, "runs", r.segment_runs, "maxlist", r.max_list)
                print("  orc", o.rgs, o.objective, o.visited, o.optimal, flush=True)
print("total mismatches", bad_total, "over", reps, "reps", flush=True)
