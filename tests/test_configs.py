"""Synthetic workload generators (configs.py): shapes of SURVEY.md 8(d), the
value contract (dyadic powers, integer bytes) and the cfg5 snapshot RNG."""
from paper_2512_20953_b200 import configs


def test_mt19937_64_matches_std():
    # std::mt19937_64 default-seeded (5489): the 10000th output is
    # 9981545732273789042 (C++ standard [rand.predef]).
    r = configs.MT19937_64(5489)
    v = None
    for _ in range(10000):
        v = r()
    assert v == 9981545732273789042


def test_config_shapes():
    assert configs.cfg1().n_gpus == 8
    assert configs.cfg2().n_gpus == 16
    assert configs.cfg3().n_gpus == 32
    assert configs.cfg4().n_gpus == 64
    assert configs.cfg4().model["n_layers"] == 96


def test_value_contract():
    for name in ("cfg1", "cfg2", "cfg3", "cfg4"):
        w = configs.get(name)
        for t in w.cluster["gpu_types"].values():
            assert (t["compute_power"] * 2) == int(t["compute_power"] * 2)
            assert t["memory_bytes"] == int(t["memory_bytes"])


def test_snapshots_deterministic():
    a = configs.cfg5_snapshots(50)
    b = configs.cfg5_snapshots(50)
    assert [x.cluster for x in a] == [x.cluster for x in b]
    assert len({x.cluster_json() for x in a}) > 10
