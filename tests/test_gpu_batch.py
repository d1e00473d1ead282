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


def test_batch_full_cfg5_sweep_plans_match_reference(product_lib):
    """All 1000 snapshots of the sweep in ONE hp_plan_compute_batch call: every
    plan JSON hashes to the reference planner's (tests/golden/cfg5_plans.json,
    tools/make_cfg5_plans.py, oracle/_ref/libhetplan.so at default options)."""
    import hashlib
    import os
    with open(os.path.join(os.path.dirname(__file__), "golden", "cfg5_plans.json")) as f:
        golden = json.load(f)
    snaps = configs.cfg5_snapshots(1000)
    got = _batch(product_lib, [s.cluster_json() for s in snaps], snaps[0].model_json(),
                 snaps[0].max_layers)
    assert len(got) == len(golden) == 1000
    bad = [g["snapshot"] for g, (st, out) in zip(golden, got)
           if (st, hashlib.sha256(out.encode()).hexdigest()) != (g["status"], g["sha256"])]
    assert not bad, (len(bad), bad[:10])


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


def test_full_cfg5_sweep_searches_match_golden(engine):
    """All 1167 grouping searches of the 1000-snapshot sweep in ONE wave-kernel
    launch (range pieces, pool compaction and the parallel queue step at full
    load): every search's visits, optimal flag, winner objective and RGS equal
    the pinned oracle's (tests/golden/cfg5_search.json, tools/make_cfg5_search.py)."""
    import math
    import os

    from paper_2512_20953_b200.configs import min_mem_for, units_for
    from paper_2512_20953_b200.engine import GroupingProblem
    with open(os.path.join(os.path.dirname(__file__), "golden", "cfg5_search.json")) as f:
        golden = json.load(f)
    probs = []
    for w in configs.cfg5_snapshots(1000):
        g = 0
        for nd in w.cluster["nodes"]:
            g = math.gcd(g, nd["count"])
        for tp in [t for t in range(1, g + 1) if g % t == 0]:
            P, M, T, N = units_for(w.cluster, tp)
            probs.append(GroupingProblem(P, M, w.model["n_microbatches"], min_mem_for(w.model),
                                         T, N))
    assert len(probs) == len(golden)
    res = engine.grouping_search(probs, max_seconds=120)
    bad = []
    for g, r in zip(golden, res):
        if r.status != g["status"]:
            bad.append(g)
            continue
        if g["status"] != 0:
            continue
        if (r.visited, r.optimal, r.objective[0].hex(), "".join(chr(48 + x) for x in r.rgs[0])) \
                != (g["visited"], g["optimal"], g["objective"], g["rgs"]):
            bad.append(g)
    assert not bad, (len(bad), bad[:3])


def _oracle_topk(args):
    from oracle.binding import Oracle
    P, M, K, MIN, T, N, k = args
    r = Oracle().solve_grouping(P, M, K, MIN, T, N, top_k=k)
    return (r.status, r.count, r.visited, r.optimal, [x.hex() for x in r.objective], r.rgs)


def test_cfg5_sweep_top_k_matches_oracle(engine):
    """top_k = 3 on 200 sweep snapshots in one launch (the top-k state at scale:
    range pieces, compaction, sequential queue scans with improvers)."""
    import math
    import os
    from multiprocessing import get_context

    from paper_2512_20953_b200.configs import min_mem_for, units_for
    from paper_2512_20953_b200.engine import GroupingProblem
    args, probs = [], []
    for w in configs.cfg5_snapshots(200):
        g = 0
        for nd in w.cluster["nodes"]:
            g = math.gcd(g, nd["count"])
        for tp in [t for t in range(1, g + 1) if g % t == 0]:
            P, M, T, N = units_for(w.cluster, tp)
            K, MIN = w.model["n_microbatches"], min_mem_for(w.model)
            probs.append(GroupingProblem(P, M, K, MIN, T, N, top_k=3))
            args.append((P, M, K, MIN, T, N, 3))
    res = engine.grouping_search(probs, max_seconds=120)
    with get_context("spawn").Pool(os.cpu_count()) as pool:
        want = pool.map(_oracle_topk, args, chunksize=2)
    got = [(r.status, r.count, r.visited, r.optimal, [x.hex() for x in r.objective], r.rgs)
           if r.status == 0 else (r.status,) for r in res]
    want = [w if w[0] == 0 else (w[0],) for w in want]
    bad = [i for i, (a, b) in enumerate(zip(got, want)) if a != b]
    assert not bad, (len(bad), [(got[i], want[i]) for i in bad[:2]])
