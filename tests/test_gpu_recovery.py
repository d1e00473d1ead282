"""the replanning sweep feeds the reference's recovery engine.

Consecutive cfg5 snapshots are planned with the batched B200 planner
(hp_plan_compute_batch); each old plan is checkpointed (hp_checkpoint_save) and
the recovery from the old plan to the new one is computed against its layer
bitmap (hp_recovery_compute) — the reference's own checkpoint / recovery code,
untouched, consuming our plans. The same pipeline through the reference library
must give the same recovery document (or the same status and error)."""
import os

import pytest

from paper_2512_20953_b200 import configs
from paper_2512_20953_b200.capi import HetplanError

pytestmark = pytest.mark.gpu


def _recover(lib, plans, clusters, root):
    out = []
    for i in range(len(plans) - 1):
        ck = os.path.join(root, f"ck_{i}")
        os.makedirs(ck, exist_ok=True)
        try:
            lib.checkpoint_save(plans[i], ck, step=100 + i, hidden_dim=4)
            out.append((0, lib.recovery_json(plans[i], plans[i + 1],
                                             os.path.join(ck, "bitmap.json"), clusters[i + 1])))
        except HetplanError as e:
            out.append((e.status, e.message))
    return out


def test_replan_then_recover_matches_reference(product_lib, ref_lib, tmp_path):
    snaps = configs.cfg5_snapshots(6)
    md_p = product_lib.model_parse(snaps[0].model_json())
    cl_p = [product_lib.cluster_parse(w.cluster_json()) for w in snaps]
    pr_p = [product_lib.profile_synth(c, w.base_seconds, w.max_layers) for c, w in zip(cl_p, snaps)]
    batch = product_lib.plan_compute_batch(cl_p, md_p, pr_p)
    assert all(st == 0 for st, _, _ in batch), [m for _, _, m in batch]
    got = _recover(product_lib, [p for _, p, _ in batch], cl_p, str(tmp_path))

    md_r = ref_lib.model_parse(snaps[0].model_json())
    cl_r = [ref_lib.cluster_parse(w.cluster_json()) for w in snaps]
    pr_r = [ref_lib.profile_synth(c, w.base_seconds, w.max_layers) for c, w in zip(cl_r, snaps)]
    plans_r = [ref_lib.plan_compute(c, md_r, p) for c, p in zip(cl_r, pr_r)]
    want = _recover(ref_lib, plans_r, cl_r, str(tmp_path))
    assert got == want
    assert any(st == 0 for st, _ in got)  # at least one recovery document was produced
