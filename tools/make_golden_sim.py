"""Golden 1F1B simulations (tests/golden/sim.json) from the REFERENCE library
(oracle/_ref/libhetplan.so, compiled from /root/reference/proj/src): for every
feasible plan case's golden plan (tests/golden/plans.json) and four simulator
option sets, hp_simulate's JSON (hp_sim_result_to_json) and timeline CSV
(hp_sim_timeline_csv), as SHA-256 digests, plus the makespan (hex). The GPU test
simulates the same plans through the product (hp_simulate and
hp_simulate_batch) and compares.
Run: python tools/make_golden_sim.py"""
import hashlib
import json
import os
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle.binding import REF_LIB  # noqa: E402
from paper_2512_20953_b200 import cases  # noqa: E402
from paper_2512_20953_b200.capi import HetplanLib  # noqa: E402

# (combined_time, fb_ratio, zero_comm): the planner's validation mode, the
# defaults, a split ratio, and zero communication
SIM_OPTIONS = [(True, None, False), (False, None, False), (False, 1.5, False), (False, 3.0, True)]


def sha(s):
    return hashlib.sha256(s.encode()).hexdigest()


if __name__ == "__main__":
    with open(os.path.join(ROOT, "tests", "golden", "plans.json")) as f:
        golden = {r["name"]: r for r in json.load(f)}
    lib = HetplanLib(REF_LIB)
    out = []
    for case in cases.plan_cases():
        g = golden.get(case.name)
        if not g or g["status"] != 0:
            continue
        with tempfile.NamedTemporaryFile("w", suffix=".json", delete=False) as f:
            f.write(g["json"])
            path = f.name
        cl = lib.cluster_parse(case.cluster)
        md = lib.model_parse(case.model)
        pr = lib.profile_synth(cl, case.base_seconds, case.max_layers)
        plan = lib.plan_load(path)
        os.unlink(path)
        for opt in SIM_OPTIONS:
            js, csv, mk = lib.simulate(plan, cl, md, pr, *opt)
            out.append({"case": case.name, "options": list(opt), "json": sha(js),
                        "csv": sha(csv), "makespan": mk.hex()})
    with open(os.path.join(ROOT, "tests", "golden", "sim.json"), "w") as f:
        json.dump(out, f, indent=0)
    print("wrote", len(out), "simulations")
