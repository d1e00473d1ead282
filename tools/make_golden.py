"""Generate the golden fixtures under tests/golden/ from the REFERENCE library
compiled from its own sources (oracle/_ref/libhetplan.so, built by
oracle/Makefile from /root/reference/proj/src) and the reference probe.

The fixtures let the tests pin the oracle and the B200 product without the
reference being present at run time (it is absent on the GPU box):

* plans.json     — full hp_plan_compute outputs (plan JSON text, or status +
                   hp_last_error) for the BASELINE configs, the reference's own
                   test fixtures and acceptance clusters, and option variants.
* grouping.json  — solve_grouping_topk outputs on seeded random unit sets
                   (exhaustive and budget-truncated), via the probe.
* partition.json — balance_workload outputs on seeded random stage sets.

Run: python tools/make_golden.py   (needs oracle/_ref built; ~1 min)
"""
import ctypes as C
import json
import os
import random
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle.binding import PROBE_LIB, REF_LIB  # noqa: E402
from paper_2512_20953_b200 import configs  # noqa: E402
from paper_2512_20953_b200.capi import HetplanError, HetplanLib, PlanOptions  # noqa: E402
from paper_2512_20953_b200 import cases  # noqa: E402

GOLDEN = os.path.join(ROOT, "tests", "golden")


def gen_plans(ref):
    out = []
    for case in cases.plan_cases():
        rec = {"name": case.name}
        try:
            rec["json"] = ref.plan_json(case.cluster, case.model, case.max_layers, case.options,
                                        case.base_seconds)
            rec["status"] = 0
        except HetplanError as e:
            rec["status"] = e.status
            rec["error"] = e.message
        out.append(rec)
    return out


def gen_grouping(probe):
    rng = random.Random(2512)
    out = []
    for inst in cases.grouping_cases(rng, 400):
        n = len(inst["power"])
        k = max(1, inst["top_k"])
        cnt = C.c_int()
        rgs = (C.c_int * (n * k))()
        obj = (C.c_double * k)()
        z = (C.c_double * k)()
        opt = C.c_int()
        vis = C.c_longlong()
        D = lambda a: (C.c_double * len(a))(*a)  # noqa: E731
        I = lambda a: (C.c_int * len(a))(*a)  # noqa: E731
        rc = probe.ref_solve_grouping(n, D(inst["power"]), D(inst["memory"]), I(inst["type_key"]),
                                      I(inst["node_key"]), inst["K"], C.c_double(inst["min_mem"]),
                                      inst["exact_threshold"], C.c_longlong(inst["node_budget"]),
                                      inst["top_k"], C.byref(cnt), rgs, obj, z, C.byref(opt),
                                      C.byref(vis))
        rec = dict(inst)
        rec["status"] = rc
        if rc == 0:
            c = cnt.value
            rec["count"] = c
            rec["rgs"] = [[rgs[j * n + u] for u in range(n)] for j in range(c)]
            rec["objective"] = [obj[j].hex() for j in range(c)]
            rec["z"] = [z[j].hex() for j in range(c)]
            rec["optimal"] = bool(opt.value)
            rec["visited"] = vis.value
        out.append(rec)
    return out


def gen_partition(probe):
    rng = random.Random(404)
    out = []
    for inst in cases.partition_cases(rng, 200):
        P = len(inst["mem_capacity"])
        n_bits = len(inst["prof"][0])
        flat = [v for row in inst["prof"] for v in row]
        layers = (C.c_int * P)()
        times = (C.c_double * P)()
        bn = C.c_double()
        D = lambda a: (C.c_double * len(a))(*a)  # noqa: E731
        I = lambda a: (C.c_int * len(a))(*a)  # noqa: E731
        rc = probe.ref_balance_workload(inst["n_layers"], P, n_bits, D(flat),
                                        D(inst["mem_capacity"]), I(inst["stage_index"]),
                                        inst["tp"], C.c_double(inst["ppb"]),
                                        C.c_double(inst["pab"]), C.c_double(inst["opt_mult"]),
                                        inst["k_total"], inst["k_total"], 0, layers, times,
                                        C.byref(bn))
        rec = dict(inst)
        rec["status"] = rc
        if rc == 0:
            rec["layers"] = list(layers)
            rec["times"] = [times[i].hex() for i in range(P)]
            rec["bottleneck"] = bn.value.hex()
        out.append(rec)
    return out


def main():
    os.makedirs(GOLDEN, exist_ok=True)
    ref = HetplanLib(REF_LIB)
    probe = C.CDLL(PROBE_LIB)
    with open(os.path.join(GOLDEN, "plans.json"), "w") as f:
        json.dump(gen_plans(ref), f, indent=0, sort_keys=True)
    with open(os.path.join(GOLDEN, "grouping.json"), "w") as f:
        json.dump(gen_grouping(probe), f, indent=0, sort_keys=True)
    with open(os.path.join(GOLDEN, "partition.json"), "w") as f:
        json.dump(gen_partition(probe), f, indent=0, sort_keys=True)
    print("golden fixtures written to", GOLDEN)


if __name__ == "__main__":
    main()
