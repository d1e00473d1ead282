"""Synthetic cluster / model inputs for the five BASELINE.json configurations.

SURVEY.md section 8(d) fixes the shapes: GPU types are the reference's own
three-type fixture (P/tests/acceptance.cpp:449-451), bandwidths are the fixture
values (P/tests/fixtures/cluster_small.json:10-15), optimizer_multiplier = 3.0,
profiles come from ``hp_profile_synth(cluster, 0.05, max_layers)``
(P/src/profile.cpp:263-289), planner options are the reference defaults.
Every power is dyadic and every byte count an integer below 2**53, which is the
value contract under which plans are bit-exact.
"""
from __future__ import annotations

import json
from dataclasses import dataclass, field

A100 = {"compute_power": 1.0, "memory_bytes": 80e9}
A100_40G = {"compute_power": 1.0, "memory_bytes": 40e9}
H800 = {"compute_power": 2.0, "memory_bytes": 80e9}
H20 = {"compute_power": 1.5, "memory_bytes": 100e9}
BANDWIDTHS = {"intra_node": 600e9, "inter_node": 50e9, "cloud": 1200e6, "local_disk": 3500e6}


@dataclass
class Workload:
    name: str
    cluster: dict
    model: dict
    max_layers: int
    base_seconds: float = 0.05
    note: str = ""

    def cluster_json(self) -> str:
        return json.dumps(self.cluster)

    def model_json(self) -> str:
        return json.dumps(self.model)

    @property
    def n_gpus(self) -> int:
        return sum(n["count"] for n in self.cluster["nodes"])


def _cluster(types: dict, nodes: list[tuple[int, str]]) -> dict:
    return {
        "gpu_types": types,
        "nodes": [{"node_id": i, "count": c, "type": t} for i, (c, t) in enumerate(nodes)],
        "bandwidths": dict(BANDWIDTHS),
    }


def _model(L: int, ppb: float, pab: float, K: int) -> dict:
    return {
        "n_layers": L,
        "per_layer_param_bytes": ppb,
        "per_layer_activation_bytes": pab,
        "optimizer_multiplier": 3.0,
        "n_microbatches": K,
        "global_batch_tokens": 1048576,
    }


def cfg1() -> Workload:
    """GPT-3 1.3B-class, 8 GPUs of 2 types (4 A100 + 4 H800)."""
    return Workload("cfg1-gpt3-1.3b-8gpu-2type",
                    _cluster({"A100": A100, "H800": H800}, [(4, "A100"), (4, "H800")]),
                    _model(24, 1.0e8, 1.4e8, 16), 32)


def cfg2() -> Workload:
    """LLaMA-7B-class, 16 GPUs of 3 types; A100 capped at 40 GB."""
    return Workload("cfg2-llama7b-16gpu-3type",
                    _cluster({"A100": A100_40G, "H800": H800, "H20": H20},
                             [(8, "A100"), (4, "H800"), (4, "H20")]),
                    _model(32, 4.0e8, 2.8e8, 32), 32)


def cfg3() -> Workload:
    """GPT-3 13B-class, 32 GPUs of 3 types."""
    return Workload("cfg3-gpt3-13b-32gpu-3type",
                    _cluster({"A100": A100, "H800": H800, "H20": H20},
                             [(8, "A100"), (8, "A100"), (8, "H800"), (8, "H20")]),
                    _model(40, 6.3e8, 3.6e8, 32), 64)


def cfg4() -> Workload:
    """96-layer 175B-class, 64 GPUs of 3 types (largest candidate space)."""
    nodes = [(8, "A100")] * 3 + [(8, "H800")] * 3 + [(8, "H20")] * 2
    return Workload("cfg4-175b-96layer-64gpu-3type",
                    _cluster({"A100": A100, "H800": H800, "H20": H20}, nodes),
                    _model(96, 3.6e9, 8.6e8, 64), 64)


class MT19937_64:
    """std::mt19937_64 (the reference's test RNG engine), bit-exact."""

    def __init__(self, seed: int):
        self.mt = [0] * 312
        self.mt[0] = seed & 0xFFFFFFFFFFFFFFFF
        for i in range(1, 312):
            prev = self.mt[i - 1]
            self.mt[i] = (6364136223846793005 * (prev ^ (prev >> 62)) + i) & 0xFFFFFFFFFFFFFFFF
        self.idx = 312

    def _twist(self):
        mt = self.mt
        for i in range(312):
            x = (mt[i] & 0xFFFFFFFF80000000) | (mt[(i + 1) % 312] & 0x7FFFFFFF)
            xa = x >> 1
            if x & 1:
                xa ^= 0xB5026F5AA96619E9
            mt[i] = mt[(i + 156) % 312] ^ xa
        self.idx = 0

    def __call__(self) -> int:
        if self.idx >= 312:
            self._twist()
        y = self.mt[self.idx]
        self.idx += 1
        y ^= (y >> 29) & 0x5555555555555555
        y ^= (y << 17) & 0x71D67FFFEDA60000
        y ^= (y << 37) & 0xFFF7EEE000000000
        y ^= y >> 43
        return y & 0xFFFFFFFFFFFFFFFF


def cfg5_snapshots(count: int = 1000, seed: int = 2512) -> list[Workload]:
    """Spot-preemption replanning sweep over the cfg3 cluster.

    For each base node in order: count' = 8 - rng()%5 (dropped if <= 0); node ids
    renumbered densely. Then with probability 1/4 (rng()%4 == 0) a node of
    1 + rng()%8 GPUs of type rng()%3 in (A100, H800, H20) joins.
    """
    rng = MT19937_64(seed)
    base = cfg3()
    type_names = ["A100", "H800", "H20"]
    out = []
    for s in range(count):
        nodes = []
        for nd in base.cluster["nodes"]:
            c = 8 - rng() % 5
            if c > 0:
                nodes.append((c, nd["type"]))
        if rng() % 4 == 0:
            c = 1 + rng() % 8
            t = type_names[rng() % 3]
            nodes.append((c, t))
        out.append(Workload(f"cfg5-snapshot-{s:04d}",
                            _cluster({"A100": A100, "H800": H800, "H20": H20}, nodes),
                            dict(base.model), base.max_layers))
    return out


WORKLOADS = {"cfg1": cfg1, "cfg2": cfg2, "cfg3": cfg3, "cfg4": cfg4}


def get(name: str) -> Workload:
    return WORKLOADS[name]()


# ---- grouping inputs of a workload (the planner builds the same through the C
# ABI; these let bench.py and the tests drive the kernel C-ABI directly)

def units_for(cluster: dict, tp: int):
    """TP units of a JSON cluster whose nodes are single-type, as
    build_tp_units forms them (P/src/grouping.cpp:40-75): nodes by id, blocks of
    tp ranks, power and memory summed in rank order. Returns (power, memory,
    type_key, node_key) in unit order."""
    types = cluster["gpu_types"]
    names = sorted(types)
    P, M, T, N = [], [], [], []
    for nd in sorted(cluster["nodes"], key=lambda x: x["node_id"]):
        t = types[nd["type"]]
        for _ in range(0, nd["count"], tp):
            p = 0.0
            m = 0.0
            for _ in range(tp):
                p += float(t["compute_power"])
                m += float(t["memory_bytes"])
            P.append(p)
            M.append(m)
            T.append(names.index(nd["type"]))
            N.append(nd["node_id"])
    return P, M, T, N


def min_mem_for(model: dict) -> float:
    """MIN_mem, MemoryModel::required_group_memory (P/src/profile.cpp:217-224)."""
    L = model["n_layers"]
    return (L * model["per_layer_param_bytes"] * (1.0 + model["optimizer_multiplier"])
            + L * model["per_layer_activation_bytes"])


def tp_dims_of(cluster: dict) -> list:
    """enumerate_tp_dims (P/src/grouping.cpp:341-350): divisors of the gcd."""
    import math
    g = 0
    for nd in cluster["nodes"]:
        g = math.gcd(g, nd["count"])
    return [t for t in range(1, g + 1) if g % t == 0] or [1]
