"""Per-phase host timing of hp_plan_compute on a -DHPK_HOST_TRACE=1 build
(plan_jobs prints one line per plan on stderr).
usage: python tools/host_phases.py LIB CFG [reps]"""
import os
import sys
import time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2512_20953_b200 import configs  # noqa: E402
from paper_2512_20953_b200.capi import HetplanLib  # noqa: E402

lib = HetplanLib(sys.argv[1])
w = configs.get(sys.argv[2])
cl = lib.cluster_parse(w.cluster_json())
md = lib.model_parse(w.model_json())
pr = lib.profile_synth(cl, w.base_seconds, w.max_layers)
for _ in range(int(sys.argv[3]) if len(sys.argv) > 3 else 5):
    t0 = time.perf_counter()
    p = lib.plan_compute(cl, md, pr)
    t1 = time.perf_counter()
    js = lib.plan_to_json(p)
    t2 = time.perf_counter()
    print(f"[host_phases] {w.name}: plan_compute {(t1 - t0) * 1e3:.3f} ms, to_json "
          f"{(t2 - t1) * 1e3:.3f} ms", file=sys.stderr, flush=True)
