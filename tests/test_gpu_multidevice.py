"""Multi-GPU inside the drop-in API: hpk_grouping_search(device=HPK_ALL_DEVICES)
spreads a batch's searches over every visible GPU (longest-first to the
least-loaded device) and hp_plan_compute uses it. On one GPU this runs the
single-device branch; on N GPUs the split. Either way the results must equal
the single-device engine's and the reference's plans."""
import pytest

from paper_2512_20953_b200 import configs
from paper_2512_20953_b200.configs import min_mem_for, tp_dims_of, units_for
from paper_2512_20953_b200.engine import HPK_ALL_DEVICES, GroupingProblem

pytestmark = pytest.mark.gpu


def _problems(ws):
    out = []
    for w in ws:
        for tp in tp_dims_of(w.cluster):
            P, M, T, N = units_for(w.cluster, tp)
            out.append(GroupingProblem(P, M, w.model["n_microbatches"], min_mem_for(w.model),
                                       T, N))
    return out


def test_all_devices_equals_one_device(engine):
    probs = _problems([configs.cfg3()] + configs.cfg5_snapshots(40))
    one = engine.grouping_search(probs, device=0)
    t1 = engine.timing()
    engine.reset_timing()
    alln = engine.grouping_search(probs, device=HPK_ALL_DEVICES)
    tn = engine.timing()
    key = lambda r: (r.status, r.count, r.optimal, r.visited, r.objective, r.rgs)  # noqa: E731
    assert [key(r) for r in one] == [key(r) for r in alln]
    assert tn.devices_used == min(engine.device_count(), 16, len(probs)) and t1.devices_used == 1


def test_plan_uses_every_device_and_matches_reference(product_lib, golden_plans, engine):
    w = configs.cfg4()
    engine.reset_timing()
    got = product_lib.plan_json(w.cluster_json(), w.model_json(), w.max_layers)
    assert got == golden_plans["cfg4"]["json"]
    assert engine.timing().devices_used == min(engine.device_count(), 4)  # 4 TP dims


def test_concurrent_plan_calls_are_reentrant(product_lib, golden_plans):
    """The reference C ABI is reentrant (no static mutable state, thread-local
    error); the B200 library keeps that: per-device contexts with
    their own stream and lock, thread-local errors and timings. Four host
    threads planning at once (ctypes releases the GIL) get the reference's
    plans."""
    import threading
    names = ["cfg1", "cfg2", "cfg3", "cfg1", "cfg2", "cfg3", "cfg4", "cfg2"]
    out = [None] * len(names)

    def work(i):
        w = configs.get(names[i])
        out[i] = product_lib.plan_json(w.cluster_json(), w.model_json(), w.max_layers)

    threads = [threading.Thread(target=work, args=(i,)) for i in range(len(names))]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    for nm, js in zip(names, out):
        assert js == golden_plans[nm]["json"], nm
