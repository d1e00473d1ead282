import sys, os
sys.path.insert(0, '/root/repo')
from oracle.binding import Oracle
from paper_2512_20953_b200.engine import Engine, GroupingProblem
eng = Engine(); orc = Oracle()
cases = [
 (GroupingProblem([1.5, 0.5, 3.0, 1.5, 3.0, 2.0, 0.5], [7.0, 12.0, 7.0, 8.0, 14.0, 14.0, 17.0], 2, 5.697513308353003, [3, 1, 6, 3, 6, 4, 1], [0, 0, 0, 1, 2, 2, 3], 8, 1424), 5),
 (GroupingProblem([1.0, 1.5, 3.0, 1.5, 1.5, 1.0], [17.0, 5.0, 14.0, 4.0, 17.0, 5.0], 3, 1.7252175601686401, [2, 3, 6, 3, 3, 2], [0, 0, 3, 3, 3, 3], 100, 637), 64),
]
for pb, cap in cases:
    r = eng.grouping_search([pb], segment_cap=cap, max_seconds=20)[0]
    o = orc.solve_grouping(pb.power, pb.memory, pb.n_microbatches, pb.min_mem, pb.type_key, pb.node_key, pb.exact_threshold, pb.node_budget)
    print("GPU", r.visited, r.rgs, "ORACLE", o.visited, o.rgs, flush=True)
    r = eng.grouping_search([pb], segment_cap=1000000, max_seconds=20)[0]
    print(" uncapped GPU", r.visited, flush=True)
