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

HPK_MAX_UNITS = 128
HPK_MAX_TOPK = 16
HPK_ALL_DEVICES = -2

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
        ("objective", C.POINTER(C.c_double)),
        ("z", C.POINTER(C.c_double)),
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
        ("max_ctas", C.c_int),
        ("cut_intervals", C.c_int),
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
        ("devices_used", C.c_int),
        ("affinity_ms", C.c_double),
        ("pipeline_ms", C.c_double),
    ]


class hpk_plan_candidate(C.Structure):
    _fields_ = [
        ("n_layers", C.c_int), ("tp", C.c_int), ("k_total", C.c_int), ("n_groups", C.c_int),
        ("ppb", C.c_double), ("pab", C.c_double), ("opt_mult", C.c_double),
        ("cost_ppb", C.c_double), ("cost_pab", C.c_double),
        ("intra_bw", C.c_double), ("inter_bw", C.c_double),
        ("sync_max", C.c_int), ("allow_zero", C.c_int),
        ("group_stage_off", C.POINTER(C.c_int)), ("microbatches", C.POINTER(C.c_int)),
        ("stage_type", C.POINTER(C.c_int)), ("stage_index", C.POINTER(C.c_int)),
        ("stage_mem_capacity", C.POINTER(C.c_double)), ("stage_node", C.POINTER(C.c_int)),
        ("stage_rank0", C.POINTER(C.c_int)),
        ("n_types", C.c_int), ("n_bits", C.c_int),
        ("prof", C.POINTER(C.c_double)),
    ]


class hpk_plan_result(C.Structure):
    _fields_ = [
        ("status", C.c_int), ("fail_group", C.c_int), ("fail_kind", C.c_int),
        ("missing_stage", C.c_int), ("missing_layers", C.c_int),
        ("stage_layers", C.POINTER(C.c_int)), ("stage_time", C.POINTER(C.c_double)),
        ("stage_mem", C.POINTER(C.c_double)), ("group_fill", C.POINTER(C.c_double)),
        ("group_steady", C.POINTER(C.c_double)), ("group_total", C.POINTER(C.c_double)),
        ("group_bubble", C.POINTER(C.c_double)),
        ("t_sync", C.c_double), ("t_star", C.c_double),
    ]


class hpk_affinity_problem(C.Structure):
    _fields_ = [
        ("n_groups", C.c_int), ("n_slots", C.c_int),
        ("group_off", C.POINTER(C.c_int)), ("slot_type", C.POINTER(C.c_int)),
        ("slot_node", C.POINTER(C.c_int)), ("slot_perm", C.POINTER(C.c_int)),
        ("swaps", C.c_int),
    ]


class hpk_pipeline(C.Structure):
    _fields_ = [
        ("n_stages", C.c_int), ("n_microbatches", C.c_int),
        ("forward", C.POINTER(C.c_double)), ("backward", C.POINTER(C.c_double)),
        ("send_forward", C.POINTER(C.c_double)), ("send_backward", C.POINTER(C.c_double)),
        ("makespan", C.c_double), ("busy", C.POINTER(C.c_double)),
        ("peak_in_flight", C.POINTER(C.c_int)), ("task_start", C.POINTER(C.c_double)),
        ("task_end", C.POINTER(C.c_double)),
    ]


HPK_PART_GMEM_TABLES = 1
HPK_PART_PER_L_MEMORY = 2


@dataclass
class PlanCandidate:
    """One candidate plan for hpk_partition_cost (include/hetplan_b200.h):
    groups of stages, each stage = (type row, stage_index, capacity, node, rank0)."""

    n_layers: int
    tp: int
    k_total: int
    groups: Sequence[Sequence[tuple]]
    microbatches: Sequence[int]
    prof: Sequence[Sequence[float]]  # [type][bit] seconds for 2**bit layers (<= 0: missing)
    ppb: float
    pab: float
    opt_mult: float = 3.0
    cost_ppb: Optional[float] = None
    cost_pab: Optional[float] = None
    intra_bw: float = 600e9
    inter_bw: float = 50e9
    sync_max: bool = False
    allow_zero: bool = False


@dataclass
class PlanResult:
    status: int
    fail_group: int
    fail_kind: int
    missing_stage: int
    missing_layers: int
    layers: List[int]
    stage_time: List[float]
    stage_mem: List[float]
    fill: List[float]
    steady: List[float]
    total: List[float]
    bubble: List[float]
    t_sync: float
    t_star: float


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
        L.hpk_partition_cost_ex.argtypes = [C.POINTER(hpk_plan_candidate), C.c_int,
                                            C.POINTER(hpk_plan_result), C.c_int, C.c_int]
        L.hpk_partition_cost_ex.restype = C.c_int
        L.hpk_pipeline_sim.argtypes = [C.POINTER(hpk_pipeline), C.c_int, C.c_int]
        L.hpk_pipeline_sim.restype = C.c_int
        L.hpk_stage_affinity.argtypes = [C.POINTER(hpk_affinity_problem), C.c_int, C.c_int]
        L.hpk_stage_affinity.restype = C.c_int
        L.hpk_assign_devices.argtypes = [C.POINTER(hpk_grouping_problem), C.c_int, C.c_int,
                                         C.POINTER(C.c_int)]
        L.hpk_assign_devices.restype = C.c_int
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
                        max_seconds: float = 0.0, enumeration: bool = False,
                        max_ctas: int = 0, cut_intervals: int = -1) -> List[GroupingResult]:
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
            ob = (C.c_double * max(1, pb.top_k))()
            zz = (C.c_double * max(1, pb.top_k))()
            keep += [pw, me, tk, nk, rg, ob, zz]
            arr[i] = hpk_grouping_problem(m, pb.n_microbatches, pb.min_mem, pb.exact_threshold,
                                          pb.node_budget, pb.top_k, pw, me, tk, nk)
            res[i].rgs = rg
            res[i].objective = ob
            res[i].z = zz
        cfg = hpk_search_config()
        self.lib.hpk_search_config_init(C.byref(cfg))
        cfg.device = device
        cfg.segment_cap = segment_cap
        cfg.max_list = max_list
        cfg.force_serial = int(force_serial)
        cfg.enumerate = int(enumeration)
        cfg.max_waves = max_waves
        cfg.max_seconds = max_seconds
        cfg.max_ctas = max_ctas
        cfg.cut_intervals = cut_intervals
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

    def partition_cost(self, cands: Sequence[PlanCandidate], *, device: int = -1,
                       flags: int = 0) -> List[PlanResult]:
        """hpk_partition_cost_ex: layer partition + Eq. (1) cost of every
        candidate in one launch (one CTA per candidate)."""
        n = len(cands)
        arr = (hpk_plan_candidate * n)()
        res = (hpk_plan_result * n)()
        keep = []
        shapes = []
        for i, c in enumerate(cands):
            goff = [0]
            st, si, cap, nd, rk = [], [], [], [], []
            for g in c.groups:
                for (ty, idx, cp, node, r0) in g:
                    st.append(ty)
                    si.append(idx)
                    cap.append(cp)
                    nd.append(node)
                    rk.append(r0)
                goff.append(len(st))
            S, G = len(st), len(c.groups)
            n_bits = len(c.prof[0]) if c.prof else 0
            flat = [v for row in c.prof for v in row]
            bufs = [(C.c_int * len(goff))(*goff), (C.c_int * G)(*c.microbatches),
                    (C.c_int * S)(*st), (C.c_int * S)(*si), (C.c_double * S)(*cap),
                    (C.c_int * S)(*nd), (C.c_int * S)(*rk), (C.c_double * max(1, len(flat)))(*flat)]
            outs = [(C.c_int * S)(), (C.c_double * S)(), (C.c_double * S)(), (C.c_double * G)(),
                    (C.c_double * G)(), (C.c_double * G)(), (C.c_double * G)()]
            keep += bufs + outs
            shapes.append((S, G, outs))
            arr[i] = hpk_plan_candidate(
                c.n_layers, c.tp, c.k_total, G, c.ppb, c.pab, c.opt_mult,
                c.ppb if c.cost_ppb is None else c.cost_ppb,
                c.pab if c.cost_pab is None else c.cost_pab, c.intra_bw, c.inter_bw,
                int(c.sync_max), int(c.allow_zero), bufs[0], bufs[1], bufs[2], bufs[3], bufs[4],
                bufs[5], bufs[6], len(c.prof), n_bits, bufs[7])
            r = res[i]
            (r.stage_layers, r.stage_time, r.stage_mem, r.group_fill, r.group_steady,
             r.group_total, r.group_bubble) = outs
        rc = self.lib.hpk_partition_cost_ex(arr, n, res, device, flags)
        if rc != 0:
            raise EngineError(rc, self.lib.hpk_last_error().decode())
        out = []
        for i in range(n):
            S, G, o = shapes[i]
            r = res[i]
            out.append(PlanResult(r.status, r.fail_group, r.fail_kind, r.missing_stage,
                                  r.missing_layers, list(o[0]), list(o[1]), list(o[2]),
                                  list(o[3]), list(o[4]), list(o[5]), list(o[6]), r.t_sync,
                                  r.t_star))
        return out

    def stage_affinity(self, problems: Sequence[tuple], *, device: int = -1):
        """hpk_stage_affinity: the stage mapper's DP-affinity pass for every
        problem (groups: list of [(type, node), ...] slots in stage order).
        Returns (perm, swaps) per problem: slot s now holds original slot perm[s]."""
        n = len(problems)
        arr = (hpk_affinity_problem * n)()
        keep, perms = [], []
        for i, groups in enumerate(problems):
            goff, ty, nd = [0], [], []
            for g in groups:
                for (t, v) in g:
                    ty.append(t)
                    nd.append(v)
                goff.append(len(ty))
            S = len(ty)
            b = [(C.c_int * len(goff))(*goff), (C.c_int * S)(*ty), (C.c_int * S)(*nd),
                 (C.c_int * S)()]
            keep += b
            perms.append(b[3])
            arr[i] = hpk_affinity_problem(len(groups), S, b[0], b[1], b[2], b[3], 0)
        rc = self.lib.hpk_stage_affinity(arr, n, device)
        if rc != 0:
            raise EngineError(rc, self.lib.hpk_last_error().decode())
        return [(list(perms[i]), arr[i].swaps) for i in range(n)]

    def pipeline_sim(self, pipes, *, device: int = -1):
        """hpk_pipeline_sim: pipes = [(K, [(fwd, bwd, send_f, send_b) per stage])].
        Returns [(makespan, busy, peak, starts, ends)] with each stage's tasks in
        its static 1F1B order (stage-major)."""
        n = len(pipes)
        arr = (hpk_pipeline * n)()
        keep, outs = [], []
        for i, (K, stages) in enumerate(pipes):
            P = len(stages)
            cols = [(C.c_double * P)(*[s[j] for s in stages]) for j in range(4)]
            o = [(C.c_double * P)(), (C.c_int * P)(), (C.c_double * (2 * P * K))(),
                 (C.c_double * (2 * P * K))()]
            keep += cols
            outs.append(o)
            arr[i] = hpk_pipeline(P, K, cols[0], cols[1], cols[2], cols[3], 0.0, o[0], o[1],
                                  o[2], o[3])
        rc = self.lib.hpk_pipeline_sim(arr, n, device)
        if rc != 0:
            raise EngineError(rc, self.lib.hpk_last_error().decode())
        return [(arr[i].makespan, list(outs[i][0]), list(outs[i][1]), list(outs[i][2]),
                 list(outs[i][3])) for i in range(n)]

    def assign_devices(self, problems: Sequence[GroupingProblem], n_devices: int) -> List[int]:
        """hpk_assign_devices: the device of each search under HPK_ALL_DEVICES
        (host-only; no GPU needed)."""
        n = len(problems)
        arr = (hpk_grouping_problem * n)()
        keep = []
        for i, pb in enumerate(problems):
            m = pb.n
            pw = (C.c_double * m)(*pb.power)
            me = (C.c_double * m)(*pb.memory)
            keep += [pw, me]
            arr[i] = hpk_grouping_problem(m, pb.n_microbatches, pb.min_mem, pb.exact_threshold,
                                          pb.node_budget, pb.top_k, pw, me, None, None)
        out = (C.c_int * max(1, n))()
        rc = self.lib.hpk_assign_devices(arr, n, n_devices, out)
        if rc != 0:
            raise EngineError(rc, "hpk_assign_devices: bad arguments")
        return list(out[:n])
