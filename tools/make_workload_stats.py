"""Per-workload constants bench.py reports against (profiles/workload_stats.json):
the reference's candidate count per plan search (sum over TP dimensions of
GroupingSolution::nodes_visited, P/include/hetplan/grouping.hpp:64) and the
SURVEY 8(d) fp64-op model of those visits, both from the pinned C restatement's
instrumentation (oracle/_ref/libhpo.so; its visits equal the reference probe's,
tests/test_oracle.py). cfg5: the sweep's total from tests/golden/cfg5_search.json
(reference probe) and the op model sampled on the first 16 snapshots.
bench.py only reads this file: it never executes the oracle outside its CPU legs.
Run: python tools/make_workload_stats.py"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle.binding import Oracle  # noqa: E402
from paper_2512_20953_b200 import configs  # noqa: E402
from paper_2512_20953_b200.configs import min_mem_for, tp_dims_of, units_for  # noqa: E402


def plan_stats(o, w):
    per_tp = {}
    for tp in tp_dims_of(w.cluster):
        P, M, T, N = units_for(w.cluster, tp)
        if sum(M) < min_mem_for(w.model):
            continue
        r = o.solve_grouping(P, M, w.model["n_microbatches"], min_mem_for(w.model), T, N)
        per_tp[str(tp)] = {"visits": r.visited, "model_ops": r.stats.model_ops}
    return {"visits": sum(v["visits"] for v in per_tp.values()),
            "model_ops": sum(v["model_ops"] for v in per_tp.values()), "per_tp": per_tp}


if __name__ == "__main__":
    o = Oracle()
    out = {name: plan_stats(o, configs.get(name)) for name in ("cfg1", "cfg2", "cfg3", "cfg4")}
    with open(os.path.join(ROOT, "tests", "golden", "cfg5_search.json")) as f:
        golden = json.load(f)
    sample = [plan_stats(o, w) for w in configs.cfg5_snapshots(16)]
    sv = sum(s["visits"] for s in sample)
    so = sum(s["model_ops"] for s in sample)
    per_snap = [0] * 1000
    for r in golden:
        per_snap[r["snapshot"]] += r.get("visited", 0)
    out["cfg5"] = {"snapshots": 1000, "visits": sum(per_snap),
                   "model_ops_per_visit": so / sv, "sample_visits": per_snap,
                   "source": "visits: tests/golden/cfg5_search.json (reference probe); "
                             "ops per visit: oracle instrumentation on snapshots 0..15"}
    with open(os.path.join(ROOT, "profiles", "workload_stats.json"), "w") as f:
        json.dump(out, f, indent=1)
    print({k: v["visits"] for k, v in out.items()})
