import sys
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
from oracle.binding import Oracle
from paper_2512_20953_b200.engine import Engine
from test_gpu_grouping import _random_problems
eng = Engine(); orc = Oracle()
cap = int(sys.argv[1])
probs = _random_problems(cap, 160, nmax=10 if cap < 16 else 11)
res = eng.grouping_search(probs, segment_cap=cap, max_seconds=60)
for i, (pb, r) in enumerate(zip(probs, res)):
    o = orc.solve_grouping(pb.power, pb.memory, pb.n_microbatches, pb.min_mem, pb.type_key, pb.node_key, pb.exact_threshold, pb.node_budget)
    if o.status != 0:
        continue
    if (r.rgs, r.objective, r.visited, r.optimal) != (o.rgs, o.objective, o.visited, o.optimal):
        print("MISMATCH", i, pb)
        print("  gpu", r.rgs, r.objective, r.visited, r.optimal, "waves", r.waves)
        print("  orc", o.rgs, o.objective, o.visited, o.optimal)
        # single-problem rerun at several caps
        for c2 in (1, 2, 3, 7, 64, 100000):
            rr = eng.grouping_search([pb], segment_cap=c2, max_seconds=30)[0]
            print("   cap", c2, rr.rgs, rr.objective, rr.visited, rr.optimal)
