import sys
sys.path.insert(0, '/root/repo')
from paper_2512_20953_b200.engine import Engine, GroupingProblem
eng = Engine()
pb = GroupingProblem([1.0, 1.5, 3.0, 1.5, 1.5, 1.0], [17.0, 5.0, 14.0, 4.0, 17.0, 5.0], 3, 1.7252175601686401, [2, 3, 6, 3, 3, 2], [0, 0, 3, 3, 3, 3], 100, 637)
r = eng.grouping_search([pb], segment_cap=1000000, max_seconds=20)[0]
print("GPU", r.visited, flush=True)
