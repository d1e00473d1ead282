"""Golden plans of the whole cfg5 replanning sweep (tests/golden/cfg5_plans.json):
for each of the 1000 snapshots (seed 2512), the status and the SHA-256 of the plan
JSON (hp_plan_to_json) that the REFERENCE planner returns — oracle/_ref/libhetplan.so,
compiled from /root/reference/proj/src by oracle/Makefile, reference default options.
tests/test_gpu_batch.py plans all 1000 through hp_plan_compute_batch and compares.
Run: python tools/make_cfg5_plans.py   (~30 s on 8 cores)"""
import hashlib
import json
import os
import sys
from multiprocessing import get_context

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def plan_one(i):
    from oracle.binding import REF_LIB
    from paper_2512_20953_b200 import configs
    from paper_2512_20953_b200.capi import HetplanError, HetplanLib
    w = configs.cfg5_snapshots(i + 1)[i]
    lib = HetplanLib(REF_LIB)
    try:
        js = lib.plan_json(w.cluster_json(), w.model_json(), w.max_layers)
        return {"snapshot": i, "status": 0, "sha256": hashlib.sha256(js.encode()).hexdigest()}
    except HetplanError as e:
        return {"snapshot": i, "status": e.status,
                "sha256": hashlib.sha256(e.message.encode()).hexdigest()}


if __name__ == "__main__":
    with get_context("spawn").Pool(os.cpu_count()) as pool:
        recs = pool.map(plan_one, range(1000), chunksize=8)
    with open(os.path.join(ROOT, "tests", "golden", "cfg5_plans.json"), "w") as f:
        json.dump(recs, f, separators=(",", ":"))
    print("wrote", len(recs), "plans;", sum(r["status"] == 0 for r in recs), "feasible")
