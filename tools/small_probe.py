"""Kernel and plan latency of the small configs (cfg1, accept clusters)."""
import os
import sys
import time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2512_20953_b200 import configs  # noqa: E402
from paper_2512_20953_b200.capi import HetplanLib  # noqa: E402
from paper_2512_20953_b200.engine import LIB_PATH, Engine  # noqa: E402
lib = HetplanLib(LIB_PATH)
eng = Engine()
for nm in sys.argv[1:] or ["cfg1"]:
    w = configs.get(nm)
    cl = lib.cluster_parse(w.cluster_json())
    md = lib.model_parse(w.model_json())
    pr = lib.profile_synth(cl, 0.05, w.max_layers)
    best = 1e9
    for i in range(20):
        eng.reset_timing()
        t = time.perf_counter()
        lib.plan_compute(cl, md, pr).close()
        best = min(best, time.perf_counter() - t)
    tm = eng.timing()
    print(f"{nm}: plan {best * 1e3:.3f} ms (last: search {tm.search_ms:.3f} ms, partition {tm.partition_ms:.3f} ms)", flush=True)
