"""the 1F1B simulator on the B200 (hpk_pipeline.cu, sim_b200.cpp).

hp_simulate in the product runs every DP group of a plan in one GPU launch
(the reference's simulate_1f1b is replaced at link time); hp_simulate_batch runs
every group of every plan in one launch. Both must give the reference's JSON
and timeline CSV byte for byte (tests/golden/sim.json from the reference
library, tools/make_golden_sim.py), for the planner's validation options and
the split / zero-communication modes. The acceptance suite's C2/C3 (closed-form
identity and bubble-ratio grid through simulate_pipeline) run against the
product in tests/test_gpu_kernels.py."""
import hashlib
import json
import os
import tempfile

import pytest

from paper_2512_20953_b200 import cases

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))


def _sha(s):
    return hashlib.sha256(s.encode()).hexdigest()


@pytest.fixture(scope="module")
def sim_golden():
    with open(os.path.join(HERE, "golden", "sim.json")) as f:
        return json.load(f)


def _load(lib, golden_plans, case):
    with tempfile.NamedTemporaryFile("w", suffix=".json", delete=False) as f:
        f.write(golden_plans[case.name]["json"])
        path = f.name
    try:
        plan = lib.plan_load(path)
    finally:
        os.unlink(path)
    cl = lib.cluster_parse(case.cluster)
    md = lib.model_parse(case.model)
    pr = lib.profile_synth(cl, case.base_seconds, case.max_layers)
    return plan, cl, md, pr


def test_hp_simulate_matches_reference(product_lib, golden_plans, sim_golden):
    by_case = {c.name: c for c in cases.plan_cases()}
    loaded = {}
    assert len(sim_golden) >= 150
    for rec in sim_golden:
        case = by_case[rec["case"]]
        if case.name not in loaded:
            loaded[case.name] = _load(product_lib, golden_plans, case)
        js, csv, mk = product_lib.simulate(*loaded[case.name], *rec["options"])
        assert (_sha(js), _sha(csv), mk.hex()) == (rec["json"], rec["csv"], rec["makespan"]), rec


def test_hp_simulate_batch_matches_reference(product_lib, golden_plans, sim_golden):
    # one launch per option set over every plan of one model (the cfg5 snapshots
    # share a model: a sweep's validation in one call)
    by_case = {c.name: c for c in cases.plan_cases()}
    groups = {}
    for rec in sim_golden:
        case = by_case[rec["case"]]
        groups.setdefault((case.model, tuple(rec["options"])), []).append((case, rec))
    checked = 0
    for (model, opt), items in groups.items():
        if len(items) < 2:
            continue
        loaded = [_load(product_lib, golden_plans, c) for c, _ in items]
        md = product_lib.model_parse(model)
        outs = product_lib.simulate_batch([x[0] for x in loaded], [x[1] for x in loaded], md,
                                          [x[3] for x in loaded], *opt)
        for (case, rec), (js, csv, mk) in zip(items, outs):
            assert (_sha(js), _sha(csv), mk.hex()) == (rec["json"], rec["csv"],
                                                        rec["makespan"]), rec
            checked += 1
    assert checked >= 100


def test_plan_validate_with_sim_matches_reference(product_lib, ref_lib, golden_plans):
    from paper_2512_20953_b200 import configs
    from paper_2512_20953_b200.capi import PlanOptions
    w = configs.cfg3()
    opts = PlanOptions(validate_with_sim=True)
    got = product_lib.plan_json(w.cluster_json(), w.model_json(), w.max_layers, opts)
    want = ref_lib.plan_json(w.cluster_json(), w.model_json(), w.max_layers, opts)
    assert got == want


def _static_order(p, P, K):
    """Stage p's tasks (forward?, microbatch) in the order of pipeline_sim.cpp:53-66."""
    warm = min(K, P - 1 - p)
    seq = [(True, m) for m in range(warm)]
    for m in range(warm, K):
        seq += [(True, m), (False, m - warm)]
    seq += [(False, m) for m in range(K - warm, K)]
    return seq


def test_pipeline_kernel_matches_reference_on_random_pipelines(engine):
    """hpk_pipeline_sim against the reference simulate_pipeline (probe) on 300
    random pipelines in one launch: makespan, busy, peak live microbatches and
    every task's start / end, bit for bit (durations drawn from a small set so
    that ties and zero-length tasks occur)."""
    import ctypes as C
    import random

    from oracle.binding import PROBE_LIB
    if not os.path.exists(PROBE_LIB):
        pytest.skip("reference probe not built")
    probe = C.CDLL(PROBE_LIB)
    rng = random.Random(1234)
    pipes = []
    for _ in range(300):
        P = rng.choice([1, 2, 3, 4, 7, 16, 33, 64, 70])
        K = rng.choice([1, 2, 3, 5, 8, 16, 40])
        vals = [0.0, 0.25, 0.5, 1.0, 1.5, 0.1, 0.3, 2.0 / 3.0]
        stages = [tuple(rng.choice(vals) for _ in range(4)) for _ in range(P)]
        pipes.append((K, stages))
    got = engine.pipeline_sim(pipes)
    D = lambda a: (C.c_double * len(a))(*a)  # noqa: E731
    for (K, stages), (mk, busy, peak, ts, te) in zip(pipes, got):
        P = len(stages)
        wmk = C.c_double()
        wbusy = (C.c_double * P)()
        wpeak = (C.c_int * P)()
        evi = (C.c_int * (3 * 2 * P * K))()
        evt = (C.c_double * (2 * 2 * P * K))()
        assert probe.ref_simulate_pipeline(P, K, D([s[0] for s in stages]),
                                           D([s[1] for s in stages]), D([s[2] for s in stages]),
                                           D([s[3] for s in stages]), C.byref(wmk), wbusy, wpeak,
                                           evi, evt) == 0
        assert mk == wmk.value and busy == list(wbusy) and peak == list(wpeak)
        want = {}
        for i in range(2 * P * K):
            want[(evi[3 * i], evi[3 * i + 1], evi[3 * i + 2])] = (evt[2 * i], evt[2 * i + 1])
        for p in range(P):
            for q, (fwd, m) in enumerate(_static_order(p, P, K)):
                key = (p, 0 if fwd else 1, m)
                assert (ts[p * 2 * K + q], te[p * 2 * K + q]) == want[key], (P, K, key)
