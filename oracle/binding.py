"""ctypes binding of the oracle (TEST INFRASTRUCTURE ONLY).

* ``Oracle``: the C restatement oracle/hetplan_oracle.c (oracle/_ref/libhpo.so).
* ``REF_LIB``: path of the reference library compiled from /root/reference
  sources by oracle/Makefile (exports the reference C ABI; used through
  paper_2512_20953_b200.capi.HetplanLib as the parity oracle for whole plans).
Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
arm may use this module.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass
from typing import List, Optional, Sequence

HERE = os.path.dirname(os.path.abspath(__file__))
HPO_LIB = os.path.join(HERE, "_ref", "libhpo.so")
REF_LIB = os.path.join(HERE, "_ref", "libhetplan.so")
PROBE_LIB = os.path.join(HERE, "_ref", "libhetplan_probe.so")


class hpo_grouping_stats(C.Structure):
    _fields_ = [(n, C.c_longlong) for n in ("visited", "internal", "leaves", "feasible",
                                             "bound_prunes", "deficit_prunes",
                                             "improvements")] + [("model_ops", C.c_double)]


@dataclass
class OracleGrouping:
    status: int
    count: int
    optimal: bool
    visited: int
    objective: List[float]
    z: List[float]
    rgs: List[List[int]]
    stats: hpo_grouping_stats


def _d(a):
    return (C.c_double * len(a))(*a)


def _i(a):
    return (C.c_int * len(a))(*a)


class Oracle:
    def __init__(self, path: str = HPO_LIB):
        self.lib = C.CDLL(path)
        L = self.lib
        L.hpo_seed_floor.restype = C.c_double
        L.hpo_stage_time.restype = C.c_double
        L.hpo_stage_memory.restype = C.c_double

    def solve_grouping(self, power: Sequence[float], memory: Sequence[float],
                       n_microbatches: int, min_mem: float,
                       type_key: Optional[Sequence[int]] = None,
                       node_key: Optional[Sequence[int]] = None, exact_threshold: int = 8,
                       node_budget: int = 5_000_000, top_k: int = 1) -> OracleGrouping:
        n = len(power)
        tk = type_key if type_key is not None else [0] * n
        nk = node_key if node_key is not None else list(range(n))
        k = max(1, top_k)
        cnt = C.c_int()
        rgs = (C.c_int * (n * k))()
        obj = (C.c_double * k)()
        z = (C.c_double * k)()
        opt = C.c_int()
        st = hpo_grouping_stats()
        rc = self.lib.hpo_solve_grouping(n, _d(power), _d(memory), _i(tk), _i(nk),
                                         n_microbatches, C.c_double(min_mem), exact_threshold,
                                         C.c_longlong(node_budget), top_k, C.byref(cnt), rgs,
                                         obj, z, C.byref(opt), C.byref(st))
        c = cnt.value if rc == 0 else 0
        return OracleGrouping(rc, c, bool(opt.value), st.visited, list(obj[:c]), list(z[:c]),
                              [[rgs[j * n + u] for u in range(n)] for j in range(c)], st)

    def balance_workload(self, n_layers, prof_rows, mem_capacity, stage_index, tp, ppb, pab,
                         opt_mult, k_total, allow_zero=False):
        P = len(prof_rows)
        n_bits = len(prof_rows[0]) if P else 0
        flat = [v for row in prof_rows for v in row]
        layers = (C.c_int * P)()
        times = (C.c_double * P)()
        bn = C.c_double()
        ms = C.c_int(-1)
        ml = C.c_int(-1)
        rc = self.lib.hpo_balance_workload(n_layers, P, n_bits, _d(flat), _d(mem_capacity),
                                           _i(stage_index), tp, C.c_double(ppb),
                                           C.c_double(pab), C.c_double(opt_mult), k_total,
                                           int(allow_zero), layers, times, C.byref(bn),
                                           C.byref(ms), C.byref(ml))
        return rc, list(layers), list(times), bn.value, ms.value, ml.value
