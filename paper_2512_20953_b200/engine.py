"""ctypes binding of the B200 kernel C-ABI (include/hetplan_b200.h, ``hpk_*``).

This is the layer planner_b200.cpp drives; tests and bench.py use it directly to
run batched grouping searches (the hot loop) and partition/cost batches on the
GPU. The library fails loudly (status 5, "no CUDA device visible") when no GPU
is present — there is no CPU fallback anywhere in it.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field
from typing import List, Optional, Sequence

HPK_MAX_UNITS = 64
HPK_MAX_TOPK = 16

PKG_DIR = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("HPK_LIB") or os.path.join(PKG_DIR, "libhetplan_b200.so")


class hpk_grouping_problem(C.Structure):
    _fields_ = [
        ("n", C.c_int),
        ("n_microbatches", C.c_int),
        ("min_mem", C.c_double),
        ("exact_threshold", C.c_int),
        ("node_budget", C.c_longlong),
        ("top_k", C.c_int),
        ("power", C.POINTER(C.c_double)),
        ("memory", C.POINTER(C.c_double)),
        ("type_key", C.POINTER(C.c_int)),
        ("node_key", C.POINTER(C.c_int)),
    ]


class hpk_grouping_result(C.Structure):
    _fields_ = [
        ("status", C.c_int),
        ("count", C.c_int),
        ("optimal", C.c_int),
        ("engine", C.c_int),
        ("visited", C.c_longlong),
        ("objective", C.c_double * HPK_MAX_TOPK),
        ("z", C.c_double * HPK_MAX_TOPK),
        ("rgs", C.POINTER(C.c_int)),
        ("waves", C.c_int),
        ("segment_runs", C.c_longlong),
        ("segment_visits", C.c_longlong),
        ("max_list", C.c_int),
        ("exact_checks", C.c_longlong),
    ]


class hpk_search_config(C.Structure):
    _fields_ = [
        ("device", C.c_int),
        ("segment_cap", C.c_longlong),
        ("max_list", C.c_int),
        ("force_serial", C.c_int),
        ("enumerate", C.c_int),
        ("max_waves", C.c_int),
        ("max_seconds", C.c_double),
    ]


class hpk_timing(C.Structure):
    _fields_ = [
        ("search_ms", C.c_double),
        ("serial_ms", C.c_double),
        ("partition_ms", C.c_double),
        ("h2d_ms", C.c_double),
        ("d2h_ms", C.c_double),
        ("h2d_bytes", C.c_longlong),
        ("d2h_bytes", C.c_longlong),
        ("kernel_launches", C.c_int),
    ]


@dataclass
class GroupingProblem:
    """Mirror of GroupingProblem (P/include/hetplan/grouping.hpp:49-59) over units."""

    power: Sequence[float]
    memory: Sequence[float]
    n_microbatches: int
    min_mem: float
    type_key: Optional[Sequence[int]] = None
    node_key: Optional[Sequence[int]] = None
    exact_threshold: int = 8
    node_budget: int = 5_000_000
    top_k: int = 1

    @property
    def n(self) -> int:
        return len(self.power)


@dataclass
class GroupingResult:
    status: int
    count: int
    optimal: bool
    engine: int
    visited: int
    objective: List[float]
    z: List[float]
    rgs: List[List[int]]
    waves: int
    segment_runs: int
    segment_visits: int
    max_list: int
    exact_checks: int = 0


class EngineError(RuntimeError):
    def __init__(self, code: int, message: str):
        super().__init__(f"hpk status {code}: {message}")
        self.code = code
        self.message = message


class Engine:
    def __init__(self, path: str = LIB_PATH):
        if not os.path.exists(path):
            raise FileNotFoundError(
                f"{path} missing: run __graft_entry__.build() (no CPU fallback exists)")
        self.lib = C.CDLL(path, mode=getattr(os, "RTLD_LOCAL", 0) | getattr(os, "RTLD_NOW", 2))
        L = self.lib
        L.hpk_version.restype = C.c_char_p
        L.hpk_last_error.restype = C.c_char_p
        L.hpk_device_count.restype = C.c_int
        L.hpk_search_config_init.argtypes = [C.POINTER(hpk_search_config)]
        L.hpk_grouping_search.argtypes = [C.POINTER(hpk_grouping_problem), C.c_int,
                                          C.POINTER(hpk_grouping_result),
                                          C.POINTER(hpk_search_config)]
        L.hpk_grouping_search.restype = C.c_int
        L.hpk_last_timing.argtypes = [C.POINTER(hpk_timing)]
        L.hpk_reset_timing.argtypes = []

    def version(self) -> str:
        return self.lib.hpk_version().decode()

    def device_count(self) -> int:
        return self.lib.hpk_device_count()

    def timing(self) -> hpk_timing:
        t = hpk_timing()
        self.lib.hpk_last_timing(C.byref(t))
        return t

    def reset_timing(self) -> None:
        self.lib.hpk_reset_timing()

    def grouping_search(self, problems: Sequence[GroupingProblem], *, device: int = -1,
                        segment_cap: int = 0, max_list: int = 0,
                        force_serial: bool = False, max_waves: int = 0,
                        max_seconds: float = 0.0, enumeration: bool = False) -> List[GroupingResult]:
        n = len(problems)
        arr = (hpk_grouping_problem * n)()
        res = (hpk_grouping_result * n)()
        keep = []
        for i, pb in enumerate(problems):
            m = pb.n
            pw = (C.c_double * m)(*pb.power)
            me = (C.c_double * m)(*pb.memory)
            tk = (C.c_int * m)(*(pb.type_key if pb.type_key is not None else [0] * m))
            nk = (C.c_int * m)(*(pb.node_key if pb.node_key is not None else list(range(m))))
            rg = (C.c_int * (max(1, pb.top_k) * m))()
            keep += [pw, me, tk, nk, rg]
            arr[i] = hpk_grouping_problem(m, pb.n_microbatches, pb.min_mem, pb.exact_threshold,
                                          pb.node_budget, pb.top_k, pw, me, tk, nk)
            res[i].rgs = rg
        cfg = hpk_search_config()
        self.lib.hpk_search_config_init(C.byref(cfg))
        cfg.device = device
        cfg.segment_cap = segment_cap
        cfg.max_list = max_list
        cfg.force_serial = int(force_serial)
        cfg.enumerate = int(enumeration)
        cfg.max_waves = max_waves
        cfg.max_seconds = max_seconds
        rc = self.lib.hpk_grouping_search(arr, n, res, C.byref(cfg))
        if rc != 0:
            raise EngineError(rc, self.lib.hpk_last_error().decode())
        out = []
        for i, pb in enumerate(problems):
            r = res[i]
            m = pb.n
            rgs = [[r.rgs[k * m + u] for u in range(m)] for k in range(r.count)]
            out.append(GroupingResult(r.status, r.count, bool(r.optimal), r.engine, r.visited,
                                      list(r.objective[:r.count]), list(r.z[:r.count]), rgs,
                                      r.waves, r.segment_runs, r.segment_visits, r.max_list,
                                      r.exact_checks))
        return out
