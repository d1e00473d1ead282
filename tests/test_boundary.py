"""The drop-in boundary: libhetplan_b200.so loads, exports every entry point
include/hetplan_b200.h declares (the reference C ABI + the hpk_* kernel ABI),
fails loudly without a GPU, and keeps the reference's behaviour for every
non-planner entry point (same bytes as the reference library)."""
import ctypes as C
import json
import os
import re

import pytest

from paper_2512_20953_b200.capi import HP_INTERNAL_ERROR, HetplanError, HetplanLib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "hetplan_b200.h")


def declared_functions():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    names = set(re.findall(r"\b(hpk?_[a-z0-9_]+)\s*\(", text))
    return sorted(n for n in names if not n.endswith("_t"))


def test_header_declares_the_reference_abi_and_kernels():
    names = declared_functions()
    for must in ("hp_plan_compute", "hp_plan_to_json", "hp_cluster_parse", "hp_recovery_compute",
                 "hpk_grouping_search", "hpk_partition_cost", "hpk_last_error"):
        assert must in names


def test_library_exports_every_declared_symbol(product_lib):
    lib = C.CDLL(product_lib.path)
    missing = [n for n in declared_functions() if not hasattr(lib, n)]
    assert not missing, missing


def test_no_gpu_fails_loudly(product_lib):
    from paper_2512_20953_b200.engine import Engine
    if Engine(product_lib.path).device_count() > 0:
        pytest.skip("GPU present: covered by the gpu tests")
    from paper_2512_20953_b200 import configs
    w = configs.cfg1()
    with pytest.raises(HetplanError) as ei:
        product_lib.plan_json(w.cluster_json(), w.model_json(), w.max_layers)
    assert ei.value.status == HP_INTERNAL_ERROR
    assert "no CUDA device" in ei.value.message


def test_no_gpu_batch_fails_loudly_per_cluster(product_lib):
    from paper_2512_20953_b200.engine import Engine
    if Engine(product_lib.path).device_count() > 0:
        pytest.skip("GPU present: covered by the gpu tests")
    from paper_2512_20953_b200 import configs
    snaps = configs.cfg5_snapshots(3)
    cl = [product_lib.cluster_parse(w.cluster_json()) for w in snaps]
    md = product_lib.model_parse(snaps[0].model_json())
    pr = [product_lib.profile_synth(c, 0.05, snaps[0].max_layers) for c in cl]
    out = product_lib.plan_compute_batch(cl, md, pr, host_threads=2)
    assert [(st, h) for st, h, _ in out] == [(HP_INTERNAL_ERROR, None)] * 3
    assert all("no CUDA device" in msg for _, _, msg in out)


def test_non_planner_abi_matches_reference(product_lib, ref_lib, golden_plans):
    # parse errors: same status and message
    for lib in (product_lib, ref_lib):
        with pytest.raises(HetplanError) as ei:
            lib.cluster_parse("{not json")
        assert ei.value.status == 2
    msgs = []
    for lib in (product_lib, ref_lib):
        try:
            lib.model_parse('{"n_layers": 0}')
        except HetplanError as e:
            msgs.append((e.status, e.message))
    assert msgs[0] == msgs[1]
    # plan JSON round trip + explain + estimate through both libraries
    rec = golden_plans["fixture-small"]
    import tempfile
    from paper_2512_20953_b200.cases import CLUSTER_SMALL, MODEL_SMALL
    outs = []
    for lib in (product_lib, ref_lib):
        with tempfile.NamedTemporaryFile("w", suffix=".json", delete=False) as f:
            f.write(rec["json"])
            path = f.name
        h = C.c_void_p()
        st = lib.lib.hp_plan_load_file(path.encode(), C.byref(h))
        assert st == 0
        from paper_2512_20953_b200.capi import Handle
        plan = Handle(lib, h, "hp_plan_free")
        cl = lib.cluster_parse(json.dumps(CLUSTER_SMALL))
        md = lib.model_parse(json.dumps(MODEL_SMALL))
        pr = lib.profile_synth(cl, 0.05, 32)
        outs.append((lib.plan_to_json(plan), lib.plan_explain(plan),
                     lib.estimate_to_json(plan, cl, md, pr)))
        os.unlink(path)
    assert outs[0] == outs[1]
    assert outs[0][0] == rec["json"]


def test_hpk_abi_without_gpu(engine):
    if engine.device_count() > 0:
        pytest.skip("GPU present")
    from paper_2512_20953_b200.engine import EngineError, GroupingProblem
    with pytest.raises(EngineError) as ei:
        engine.grouping_search([GroupingProblem([1.0], [2.0], 1, 1.0)])
    assert ei.value.code == 5 and "no CUDA device" in ei.value.message
