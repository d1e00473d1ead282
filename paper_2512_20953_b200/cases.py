"""Parity case catalog shared by tests/, tools/make_golden.py and smoke().

Plan cases cover the BASELINE configurations, the reference's own test
fixtures (P/tests/fixtures/*.json, restated as data), the acceptance clusters
(P/tests/acceptance.cpp C6/C10/C11) and every planner option of
hp_plan_options (P/include/hetplan/c_api.h:76-87).
"""
from __future__ import annotations

import json
import random
from dataclasses import dataclass, field
from typing import Optional

from . import configs
from .capi import PlanOptions

BW = {"intra_node": 6e11, "inter_node": 5e10, "cloud": 1.2e9, "local_disk": 3.5e9}

# P/tests/fixtures/cluster_small.json, model_small.json, model_too_big.json
CLUSTER_SMALL = {
    "gpu_types": {"A100": {"compute_power": 1.0, "memory_bytes": 80e9},
                  "H800": {"compute_power": 2.0, "memory_bytes": 80e9}},
    "nodes": [{"node_id": 0, "count": 4, "type": "A100"},
              {"node_id": 1, "count": 2, "type": "H800"}],
    "bandwidths": {"intra_node": 600e9, "inter_node": 50e9, "cloud": 1200e6,
                   "local_disk": 3500e6},
}
MODEL_SMALL = {"n_layers": 24, "per_layer_param_bytes": 1e9, "per_layer_activation_bytes": 2e8,
               "optimizer_multiplier": 3.0, "n_microbatches": 8, "global_batch_tokens": 1048576}
MODEL_TOO_BIG = {"n_layers": 24, "per_layer_param_bytes": 2e11,
                 "per_layer_activation_bytes": 2e8, "optimizer_multiplier": 3.0,
                 "n_microbatches": 8}

# acceptance.cpp:449-451 (C10/C11): 3 types x 8 GPUs
CLUSTER_24 = {
    "gpu_types": {"A100": {"compute_power": 1.0, "memory_bytes": 80e9},
                  "H800": {"compute_power": 2.0, "memory_bytes": 80e9},
                  "H20": {"compute_power": 1.5, "memory_bytes": 100e9}},
    "nodes": [{"node_id": 0, "count": 8, "type": "A100"},
              {"node_id": 1, "count": 8, "type": "H800"},
              {"node_id": 2, "count": 8, "type": "H20"}],
    "bandwidths": dict(BW),
}
MODEL_24 = {"n_layers": 32, "per_layer_param_bytes": 2.0e9, "per_layer_activation_bytes": 2.0e8,
            "optimizer_multiplier": 3.0, "n_microbatches": 16}
CLUSTER_HOMOG = {"gpu_types": {"A100": {"compute_power": 1.0, "memory_bytes": 300e9}},
                 "nodes": [{"node_id": 0, "count": 8, "type": "A100"}],
                 "bandwidths": dict(BW)}
MODEL_HOMOG = dict(MODEL_24, n_layers=24)


@dataclass
class PlanCase:
    name: str
    cluster: str
    model: str
    max_layers: int
    options: Optional[PlanOptions] = None
    base_seconds: float = 0.05
    heavy: bool = False  # > 0.1 s on the CPU reference


def _case(name, cluster, model, max_layers, options=None, heavy=False):
    return PlanCase(name, json.dumps(cluster), json.dumps(model), max_layers, options,
                    heavy=heavy)


def plan_cases(include_heavy: bool = True, n_snapshots: int = 24) -> list[PlanCase]:
    out = []
    for name in ("cfg1", "cfg2", "cfg3", "cfg4"):
        w = configs.get(name)
        out.append(PlanCase(name, w.cluster_json(), w.model_json(), w.max_layers,
                            heavy=name != "cfg1"))
    out += [
        _case("fixture-small", CLUSTER_SMALL, MODEL_SMALL, 32),
        _case("fixture-too-big", CLUSTER_SMALL, MODEL_TOO_BIG, 32),
        _case("accept-c10-24gpu", CLUSTER_24, MODEL_24, 64),
        _case("accept-c10-homog", CLUSTER_HOMOG, MODEL_HOMOG, 32),
        _case("opt-tp2", CLUSTER_SMALL, MODEL_SMALL, 32, PlanOptions(tp_dims=[2])),
        _case("opt-tp-dup", CLUSTER_SMALL, MODEL_SMALL, 32, PlanOptions(tp_dims=[2, 1, 2, 4])),
        _case("opt-tp3-divisibility", CLUSTER_SMALL, MODEL_SMALL, 32, PlanOptions(tp_dims=[3])),
        _case("opt-minmem", CLUSTER_SMALL, MODEL_SMALL, 32, PlanOptions(min_mem_override=1.5e11)),
        _case("opt-budget50", CLUSTER_24, MODEL_24, 64,
              PlanOptions(exact_threshold=4, node_budget=50)),
        _case("opt-budget0", CLUSTER_24, MODEL_24, 64,
              PlanOptions(exact_threshold=0, node_budget=0)),
        _case("opt-budget777", CLUSTER_24, MODEL_24, 64,
              PlanOptions(exact_threshold=2, node_budget=777)),
        _case("opt-topk3", CLUSTER_24, MODEL_24, 64, PlanOptions(top_k=3)),
        _case("opt-sync-max", CLUSTER_24, MODEL_24, 64, PlanOptions(sync_overlap_max=True)),
        _case("opt-validate-sim", CLUSTER_SMALL, MODEL_SMALL, 32,
              PlanOptions(validate_with_sim=True)),
        _case("opt-derive-power", CLUSTER_SMALL, MODEL_SMALL, 32, PlanOptions(derive_power=True)),
        _case("opt-derive-power-ref", CLUSTER_24, MODEL_24, 64,
              PlanOptions(derive_power=True, power_reference="H800", exact_threshold=12)),
        _case("opt-exhaustive-12", CLUSTER_24, MODEL_24, 64, PlanOptions(exact_threshold=12)),
        _case("missing-profile", CLUSTER_SMALL, MODEL_SMALL, 4),
    ]
    # top_k > 1 on the budget-truncated configs (the wave engine's top-k state)
    for name, k in (("cfg2", 2), ("cfg3", 4), ("cfg4", 2), ("cfg4", 4), ("cfg4", 8)):
        w = configs.get(name)
        out.append(PlanCase(f"{name}-topk{k}", w.cluster_json(), w.model_json(), w.max_layers,
                            PlanOptions(top_k=k), heavy=True))
    for w in configs.cfg5_snapshots(n_snapshots):
        out.append(PlanCase(w.name, w.cluster_json(), w.model_json(), w.max_layers, heavy=True))
    if not include_heavy:
        out = [c for c in out if not c.heavy]
    return out


def grouping_cases(rng: random.Random, count: int) -> list[dict]:
    """Seeded random solve_grouping_topk instances (exhaustive, budgeted, top_k,
    ties, infeasible). Powers are dyadic, memories integers (the value contract)."""
    out = []
    for t in range(count):
        n = rng.randint(1, 11)
        kind = t % 4
        if kind == 0:  # ties: identical units
            P = [2.0] * n
            M = [8.0] * n
        else:
            P = [rng.choice([0.5, 1.0, 1.5, 2.0, 3.0, 4.0]) for _ in range(n)]
            M = [float(rng.randint(4, 24)) for _ in range(n)]
        T = [int(p * 2) for p in P]
        N = sorted(rng.randint(0, 4) for _ in range(n))
        K = rng.randint(1, 16)
        MIN = float(round(sum(M) * rng.uniform(0.05, 1.1) / rng.randint(1, 4)))
        thr = rng.choice([0, 4, 8, 100])
        B = rng.choice([0, 1, 7, 50, 300, 3000, 5_000_000])
        topk = rng.choice([1, 1, 1, 2, 3])
        out.append({"power": P, "memory": M, "type_key": T, "node_key": N, "K": K,
                    "min_mem": MIN, "exact_threshold": thr, "node_budget": B, "top_k": topk})
    return out


def partition_cases(rng: random.Random, count: int) -> list[dict]:
    """Seeded random balance_workload instances through the profile + memory
    model path (stage times dyadic, byte coefficients integers)."""
    out = []
    for _ in range(count):
        P = rng.randint(1, 6)
        L = P + rng.randint(0, 30)
        n_bits = max(1, L.bit_length())
        prof = []
        for _s in range(P):
            per = rng.choice([0.25, 0.5, 0.75, 1.0, 1.5])
            row = [per * (1 << b) * rng.choice([1.0, 1.0, 0.75, 1.25]) for b in range(n_bits)]
            prof.append(row)
        K = rng.randint(1, 8)
        ppb, pab, om = 1.0e9, 1.0e8, 3.0
        per_layer = ppb * (1 + om) + pab * K
        caps = [per_layer * rng.randint(1, L + 2) for _s in range(P)]
        out.append({"n_layers": L, "prof": prof, "mem_capacity": caps,
                    "stage_index": list(range(1, P + 1)), "tp": rng.choice([1, 2, 4]),
                    "ppb": ppb, "pab": pab, "opt_mult": om, "k_total": K})
    return out
