"""The multi-GPU split inside the drop-in API, host side (no GPU needed):
hpk_grouping_search(device=HPK_ALL_DEVICES) sends each search to the device
chosen by hpk_assign_devices — longest-first to the least-loaded device — so a
plan's budget-truncated TP dimensions land on different GPUs and a sweep's
snapshots spread evenly. The GPU side (equal results on any device count) is
tests/test_gpu_multidevice.py."""
from paper_2512_20953_b200 import configs
from paper_2512_20953_b200.configs import min_mem_for, tp_dims_of, units_for
from paper_2512_20953_b200.engine import GroupingProblem


def _problems(w):
    out = []
    for tp in tp_dims_of(w.cluster):
        P, M, T, N = units_for(w.cluster, tp)
        out.append(GroupingProblem(P, M, w.model["n_microbatches"], min_mem_for(w.model), T, N))
    return out


def test_cfg4_tp_dimensions_longest_first(engine):
    probs = _problems(configs.cfg4())  # tp 1, 2, 4 budgeted (64/32/16 units), tp 8 exhaustive
    assert engine.assign_devices(probs, 1) == [0, 0, 0, 0]
    assert engine.assign_devices(probs, 2) == [0, 1, 1, 1]
    assert engine.assign_devices(probs, 4) == [0, 1, 2, 3]
    assert engine.assign_devices(probs, 8) == [0, 1, 2, 3]


def test_sweep_snapshots_balance(engine):
    probs = [pb for w in configs.cfg5_snapshots(200) for pb in _problems(w)]

    def cost(pb):  # search_cost (hpk_grouping.cu): visits x (n + 8)
        row, bell = [1.0], 1.0
        for _ in range(1, pb.n):
            nxt = [row[-1]]
            for x in row:
                nxt.append(nxt[-1] + x)
            row, bell = nxt, nxt[-1]
        visits = min(pb.node_budget, bell) if pb.n > pb.exact_threshold else bell
        return visits * (pb.n + 8)

    for nd in (2, 4, 8):
        dev = engine.assign_devices(probs, nd)
        load = [sum(cost(pb) for d, pb in zip(dev, probs) if d == k) for k in range(nd)]
        # LPT: the loads differ by at most one search's cost
        assert max(load) - min(load) <= max(cost(pb) for pb in probs)
        assert sorted(set(dev)) == list(range(nd))
