"""Per-phase host timing of hp_plan_compute (HPK_HOST_TRACE=1) for the configs."""
import os
import sys
import time
os.environ["HPK_HOST_TRACE"] = "1"
sys.path.insert(0, "/root/repo")
from paper_2512_20953_b200 import configs  # noqa: E402
from paper_2512_20953_b200.capi import HetplanLib  # noqa: E402
from paper_2512_20953_b200.engine import LIB_PATH  # noqa: E402
lib = HetplanLib(LIB_PATH)
for nm in sys.argv[1:] or ["cfg1", "cfg4"]:
    w = configs.get(nm)
    cl = lib.cluster_parse(w.cluster_json())
    md = lib.model_parse(w.model_json())
    pr = lib.profile_synth(cl, 0.05, w.max_layers)
    for i in range(4):
        t = time.perf_counter()
        lib.plan_compute(cl, md, pr).close()
        print(nm, f"plan_compute {1e3 * (time.perf_counter() - t):.2f} ms", flush=True)
