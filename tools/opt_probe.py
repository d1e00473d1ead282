"""Time plan_compute under non-default options (top_k, derive_power) on the
product library vs the reference library; checks the JSON is identical.

usage: python tools/opt_probe.py [cfg ...]
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle.binding import REF_LIB  # noqa: E402
from paper_2512_20953_b200 import configs  # noqa: E402
from paper_2512_20953_b200.capi import HetplanLib, PlanOptions  # noqa: E402
from paper_2512_20953_b200.engine import LIB_PATH  # noqa: E402

prod = HetplanLib(LIB_PATH)
ref = HetplanLib(REF_LIB)
names = sys.argv[1:] or ["cfg2", "cfg3", "cfg4"]
variants = [("default", PlanOptions()), ("top_k=2", PlanOptions(top_k=2)),
            ("top_k=4", PlanOptions(top_k=4)), ("top_k=12", PlanOptions(top_k=12)),
            ("derive_power", PlanOptions(derive_power=True))]


def timed(lib, w, o, reps):
    best = 1e9
    out = None
    for _ in range(reps):
        t = time.perf_counter()
        try:
            out = lib.plan_json(w.cluster_json(), w.model_json(), w.max_layers, o)
        except Exception as e:  # noqa: BLE001
            out = "ERR " + str(e)
        best = min(best, time.perf_counter() - t)
    return best * 1e3, out


for nm in names:
    w = configs.get(nm)
    for vn, o in variants:
        tp, jp = timed(prod, w, o, 3)
        tr, jr = timed(ref, w, o, 1)
        print(f"{nm:5s} {vn:13s} b200 {tp:9.1f} ms  ref {tr:9.1f} ms  same={jp == jr}", flush=True)
