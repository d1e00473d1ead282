"""hp_plan_compute_batch (the replanning-sweep extension of the drop-in ABI):
one call over many clusters returns, per cluster, exactly what hp_plan_compute
returns — the reference's plan JSON byte for byte, or its status and message."""
import json

import pytest

from paper_2512_20953_b200 import cases, configs
from paper_2512_20953_b200.capi import HetplanError

pytestmark = pytest.mark.gpu


def _batch(lib, clusters, model_text, max_layers, threads=0):
    cl = [lib.cluster_parse(c) for c in clusters]
    md = lib.model_parse(model_text)
    pr = [lib.profile_synth(c, 0.05, max_layers) for c in cl]
    out = []
    for st, h, msg in lib.plan_compute_batch(cl, md, pr, host_threads=threads):
        out.append((st, lib.plan_to_json(h) if h is not None else msg))
    return out


def _single(lib, cluster, model_text, max_layers):
    try:
        return 0, lib.plan_json(cluster, model_text, max_layers)
    except HetplanError as e:
        return e.status, e.message


def test_batch_cfg5_sweep_matches_golden(product_lib, golden_plans):
    snaps = [c for c in cases.plan_cases() if c.name.startswith("cfg5-")]
    assert len(snaps) >= 24
    got = _batch(product_lib, [c.cluster for c in snaps], snaps[0].model, snaps[0].max_layers)
    for case, (st, out) in zip(snaps, got):
        g = golden_plans[case.name]
        assert st == g["status"], case.name
        assert out == (g["json"] if st == 0 else g["error"]), case.name


def test_batch_with_failing_clusters_matches_reference(product_lib, ref_lib):
    w = configs.cfg3()
    tiny = json.loads(w.cluster_json())
    for t in tiny["gpu_types"].values():
        t["memory_bytes"] = 1e9  # no DP group can hold the model: InfeasibleError
    odd = json.loads(w.cluster_json())
    odd["nodes"][0]["count"] = 3  # tp dims shrink to [1]
    clusters = [w.cluster_json(), json.dumps(tiny), json.dumps(odd), w.cluster_json()]
    got = _batch(product_lib, clusters, w.model_json(), w.max_layers, threads=3)
    want = [_single(ref_lib, c, w.model_json(), w.max_layers) for c in clusters]
    assert got == want
    assert got[1][0] != 0 and got[0][0] == 0


def test_batch_equals_single_calls(product_lib):
    snaps = configs.cfg5_snapshots(8)
    got = _batch(product_lib, [s.cluster_json() for s in snaps], snaps[0].model_json(),
                 snaps[0].max_layers, threads=1)
    for s, g in zip(snaps, got):
        assert g == _single(product_lib, s.cluster_json(), s.model_json(), s.max_layers)
