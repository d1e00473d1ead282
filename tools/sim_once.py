"""One cfg4 plan with validate_with_sim through the product C ABI, then the
1F1B simulation of the cfg5 sweep's first plans in one hp_simulate_batch call
(profiling target for the pipeline simulator kernel)."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2512_20953_b200 import configs  # noqa: E402
from paper_2512_20953_b200.capi import HetplanLib, PlanOptions  # noqa: E402
from paper_2512_20953_b200.engine import LIB_PATH  # noqa: E402

lib = HetplanLib(LIB_PATH)
w = configs.get("cfg4")
lib.plan_json(w.cluster_json(), w.model_json(), w.max_layers, PlanOptions(validate_with_sim=True))
snaps = configs.cfg5_snapshots(64)
cl = [lib.cluster_parse(s.cluster_json()) for s in snaps]
md = lib.model_parse(snaps[0].model_json())
pr = [lib.profile_synth(c, s.base_seconds, s.max_layers) for c, s in zip(cl, snaps)]
plans = [h for _, h, _ in lib.plan_compute_batch(cl, md, pr)]
out = lib.simulate_batch(plans, cl, md, pr, combined_time=True)
print("ok", len(out), max(o[2] for o in out))
