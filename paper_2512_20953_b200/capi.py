"""ctypes binding of the reference C ABI (P/include/hetplan/c_api.h).

The same binding drives both the product library (``libhetplan_b200.so``, the
drop-in) and the reference library compiled from its own sources
(``oracle/_ref/libhetplan.so``, test/baseline only) — they export the identical
ABI, which is the point of the drop-in boundary. Function names and error
behaviour follow the reference: every call returns an ``hp_status``
(c_api.h:41-48) and failures raise :class:`HetplanError` carrying the status and
``hp_last_error()`` text.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass
from typing import List, Optional, Sequence, Tuple

HP_OK = 0
HP_PARSE_ERROR = 2
HP_INFEASIBLE = 3
HP_UNRECOVERABLE = 4
HP_INTERNAL_ERROR = 5
HP_INVALID_ARGUMENT = 6

STATUS_NAMES = {
    HP_OK: "HP_OK",
    HP_PARSE_ERROR: "HP_PARSE_ERROR",
    HP_INFEASIBLE: "HP_INFEASIBLE",
    HP_UNRECOVERABLE: "HP_UNRECOVERABLE",
    HP_INTERNAL_ERROR: "HP_INTERNAL_ERROR",
    HP_INVALID_ARGUMENT: "HP_INVALID_ARGUMENT",
}


class HetplanError(RuntimeError):
    def __init__(self, status: int, message: str):
        super().__init__(f"{STATUS_NAMES.get(status, status)}: {message}")
        self.status = status
        self.message = message


class hp_plan_options(C.Structure):
    """c_api.h:76-87, field for field."""

    _fields_ = [
        ("tp_dims", C.POINTER(C.c_int)),
        ("n_tp_dims", C.c_int),
        ("min_mem_override", C.c_double),
        ("exact_threshold", C.c_int),
        ("node_budget", C.c_longlong),
        ("top_k", C.c_int),
        ("sync_overlap_max", C.c_int),
        ("validate_with_sim", C.c_int),
        ("derive_power", C.c_int),
        ("power_reference", C.c_char_p),
    ]


class hp_sim_options(C.Structure):
    """c_api.h:105-109."""

    _fields_ = [("combined_time", C.c_int), ("fb_ratio", C.c_double), ("zero_comm", C.c_int)]


@dataclass
class PlanOptions:
    tp_dims: Optional[Sequence[int]] = None
    min_mem_override: float = 0.0
    exact_threshold: int = 8
    node_budget: int = 5_000_000
    top_k: int = 1
    sync_overlap_max: bool = False
    validate_with_sim: bool = False
    derive_power: bool = False
    power_reference: Optional[str] = None


_VP = C.c_void_p


class HetplanLib:
    """One loaded C-ABI library (product or reference)."""

    def __init__(self, path: str):
        if not os.path.exists(path):
            raise FileNotFoundError(path)
        # RTLD_LOCAL (the ctypes default): product and reference export the same
        # symbols and must not interpose on each other.
        self.path = path
        self.lib = C.CDLL(path, mode=getattr(os, "RTLD_LOCAL", 0) | getattr(os, "RTLD_NOW", 2))
        L = self.lib
        L.hp_version.restype = C.c_char_p
        L.hp_last_error.restype = C.c_char_p
        L.hp_string_free.argtypes = [C.c_void_p]
        for name in ("hp_cluster_parse", "hp_model_parse", "hp_profile_parse",
                     "hp_cluster_load_file", "hp_model_load_file", "hp_profile_load_file",
                     "hp_plan_load_file"):
            getattr(L, name).argtypes = [C.c_char_p, C.POINTER(_VP)]
            getattr(L, name).restype = C.c_int
        L.hp_profile_synth.argtypes = [_VP, C.c_double, C.c_int, C.POINTER(_VP)]
        L.hp_profile_synth.restype = C.c_int
        L.hp_cluster_device_count.argtypes = [_VP]
        L.hp_cluster_device_count.restype = C.c_int
        L.hp_plan_options_init.argtypes = [C.POINTER(hp_plan_options)]
        L.hp_plan_compute.argtypes = [_VP, _VP, _VP, C.POINTER(hp_plan_options), C.POINTER(_VP)]
        L.hp_plan_compute.restype = C.c_int
        if hasattr(L, "hp_plan_compute_batch"):  # product library only
            L.hp_plan_compute_batch.argtypes = [C.c_int, C.POINTER(_VP), _VP, C.POINTER(_VP),
                                                C.POINTER(hp_plan_options), C.c_int,
                                                C.POINTER(_VP), C.POINTER(C.c_int),
                                                C.POINTER(C.c_void_p)]
            L.hp_plan_compute_batch.restype = C.c_int
        for name in ("hp_plan_to_json", "hp_plan_explain"):
            getattr(L, name).argtypes = [_VP, C.POINTER(C.c_void_p)]
            getattr(L, name).restype = C.c_int
        L.hp_estimate_to_json.argtypes = [_VP, _VP, _VP, _VP, C.POINTER(C.c_void_p)]
        L.hp_estimate_to_json.restype = C.c_int
        L.hp_profile_write_file.argtypes = [_VP, C.c_char_p]
        L.hp_profile_write_file.restype = C.c_int
        L.hp_plan_write_file.argtypes = [_VP, C.c_char_p]
        L.hp_plan_write_file.restype = C.c_int
        # 1F1B simulation (c_api.h:105-120)
        L.hp_sim_options_init.argtypes = [C.POINTER(hp_sim_options)]
        L.hp_simulate.argtypes = [_VP, _VP, _VP, _VP, C.POINTER(hp_sim_options), C.POINTER(_VP)]
        L.hp_simulate.restype = C.c_int
        L.hp_sim_makespan.argtypes = [_VP]
        L.hp_sim_makespan.restype = C.c_double
        for name in ("hp_sim_result_to_json", "hp_sim_timeline_csv"):
            getattr(L, name).argtypes = [_VP, C.POINTER(C.c_void_p)]
            getattr(L, name).restype = C.c_int
        L.hp_sim_result_free.argtypes = [_VP]
        L.hp_sim_result_free.restype = None
        if hasattr(L, "hp_simulate_batch"):  # product library only
            L.hp_simulate_batch.argtypes = [C.c_int, C.POINTER(_VP), C.POINTER(_VP), _VP,
                                            C.POINTER(_VP), C.POINTER(hp_sim_options),
                                            C.POINTER(_VP)]
            L.hp_simulate_batch.restype = C.c_int
            L.hpk_last_error.restype = C.c_char_p
        # checkpoint / recovery (c_api.h:123-136): the reference's own engines
        L.hp_checkpoint_save.argtypes = [_VP, C.c_char_p, C.c_ulonglong, C.c_int, C.c_ulonglong,
                                         C.c_int]
        L.hp_checkpoint_save.restype = C.c_int
        L.hp_recovery_compute.argtypes = [_VP, _VP, C.c_char_p, _VP, C.POINTER(_VP)]
        L.hp_recovery_compute.restype = C.c_int
        L.hp_recovery_to_json.argtypes = [_VP, C.POINTER(C.c_void_p)]
        L.hp_recovery_to_json.restype = C.c_int
        for name in ("hp_cluster_free", "hp_model_free", "hp_profile_free", "hp_plan_free",
                     "hp_recovery_free"):
            getattr(L, name).argtypes = [_VP]
            getattr(L, name).restype = None

    # -- helpers ---------------------------------------------------------
    def _check(self, status: int) -> None:
        if status != HP_OK:
            raise HetplanError(status, self.lib.hp_last_error().decode())

    def _take_string(self, ptr: C.c_void_p) -> str:
        s = C.cast(ptr, C.c_char_p).value.decode()
        self.lib.hp_string_free(ptr)
        return s

    def version(self) -> str:
        return self.lib.hp_version().decode()

    # -- handles ---------------------------------------------------------
    def cluster_parse(self, text: str) -> "Handle":
        h = _VP()
        self._check(self.lib.hp_cluster_parse(text.encode(), C.byref(h)))
        return Handle(self, h, "hp_cluster_free")

    def model_parse(self, text: str) -> "Handle":
        h = _VP()
        self._check(self.lib.hp_model_parse(text.encode(), C.byref(h)))
        return Handle(self, h, "hp_model_free")

    def profile_parse(self, text: str) -> "Handle":
        h = _VP()
        self._check(self.lib.hp_profile_parse(text.encode(), C.byref(h)))
        return Handle(self, h, "hp_profile_free")

    def profile_synth(self, cluster: "Handle", base_seconds: float, max_layers: int) -> "Handle":
        h = _VP()
        self._check(self.lib.hp_profile_synth(cluster.ptr, base_seconds, max_layers, C.byref(h)))
        return Handle(self, h, "hp_profile_free")

    def _options(self, options: Optional[PlanOptions], keep: list) -> hp_plan_options:
        o = hp_plan_options()
        self.lib.hp_plan_options_init(C.byref(o))
        if options is not None:
            if options.tp_dims is not None:
                arr = (C.c_int * len(options.tp_dims))(*options.tp_dims)
                keep.append(arr)
                o.tp_dims = C.cast(arr, C.POINTER(C.c_int))
                o.n_tp_dims = len(options.tp_dims)
            o.min_mem_override = options.min_mem_override
            o.exact_threshold = options.exact_threshold
            o.node_budget = options.node_budget
            o.top_k = options.top_k
            o.sync_overlap_max = int(options.sync_overlap_max)
            o.validate_with_sim = int(options.validate_with_sim)
            o.derive_power = int(options.derive_power)
            if options.power_reference is not None:
                b = options.power_reference.encode()
                keep.append(b)
                o.power_reference = b
        return o

    def plan_compute_batch(self, clusters: List["Handle"], model: "Handle",
                           profiles: List["Handle"], options: Optional[PlanOptions] = None,
                           host_threads: int = 0) -> List[Tuple[int, Optional["Handle"], str]]:
        """hp_plan_compute_batch: [(status, plan handle or None, error message)]."""
        n = len(clusters)
        keep: list = []
        o = self._options(options, keep)
        cl = (_VP * n)(*[c.ptr for c in clusters])
        pr = (_VP * n)(*[p.ptr for p in profiles])
        plans = (_VP * n)()
        status = (C.c_int * n)()
        errs = (C.c_void_p * n)()
        rc = self.lib.hp_plan_compute_batch(n, cl, model.ptr, pr, C.byref(o), host_threads,
                                            plans, status, errs)
        if rc != HP_OK:
            raise HetplanError(rc, "hp_plan_compute_batch: invalid arguments")
        out = []
        for i in range(n):
            msg = self._take_string(errs[i]) if errs[i] else ""
            h = Handle(self, _VP(plans[i]), "hp_plan_free") if plans[i] else None
            out.append((status[i], h, msg))
        return out

    def plan_compute(self, cluster: "Handle", model: "Handle", profile: "Handle",
                     options: Optional[PlanOptions] = None) -> "Handle":
        o = hp_plan_options()
        self.lib.hp_plan_options_init(C.byref(o))
        keep = []
        if options is not None:
            if options.tp_dims is not None:
                arr = (C.c_int * len(options.tp_dims))(*options.tp_dims)
                keep.append(arr)
                o.tp_dims = C.cast(arr, C.POINTER(C.c_int))
                o.n_tp_dims = len(options.tp_dims)
            o.min_mem_override = options.min_mem_override
            o.exact_threshold = options.exact_threshold
            o.node_budget = options.node_budget
            o.top_k = options.top_k
            o.sync_overlap_max = int(options.sync_overlap_max)
            o.validate_with_sim = int(options.validate_with_sim)
            o.derive_power = int(options.derive_power)
            if options.power_reference is not None:
                b = options.power_reference.encode()
                keep.append(b)
                o.power_reference = b
        h = _VP()
        self._check(self.lib.hp_plan_compute(cluster.ptr, model.ptr, profile.ptr, C.byref(o),
                                             C.byref(h)))
        return Handle(self, h, "hp_plan_free")

    def plan_to_json(self, plan: "Handle") -> str:
        p = C.c_void_p()
        self._check(self.lib.hp_plan_to_json(plan.ptr, C.byref(p)))
        return self._take_string(p)

    def plan_explain(self, plan: "Handle") -> str:
        p = C.c_void_p()
        self._check(self.lib.hp_plan_explain(plan.ptr, C.byref(p)))
        return self._take_string(p)

    def estimate_to_json(self, plan, cluster, model, profile) -> str:
        p = C.c_void_p()
        self._check(self.lib.hp_estimate_to_json(plan.ptr, cluster.ptr, model.ptr, profile.ptr,
                                                 C.byref(p)))
        return self._take_string(p)

    def checkpoint_save(self, plan: "Handle", root: str, step: int, hidden_dim: int = 8,
                        seed: int = 2512, zero_optimizer: bool = False) -> None:
        """hp_checkpoint_save (c_api.h:123-125): writes root/manifest.json,
        root/bitmap.json and the per-device layer shards."""
        self._check(self.lib.hp_checkpoint_save(plan.ptr, root.encode(), step, hidden_dim, seed,
                                                int(zero_optimizer)))

    def recovery_json(self, old_plan: "Handle", new_plan: "Handle", bitmap_path: str,
                      cluster: "Handle") -> str:
        """hp_recovery_compute + hp_recovery_to_json (c_api.h:127-132)."""
        out = C.c_void_p()
        self._check(self.lib.hp_recovery_compute(old_plan.ptr, new_plan.ptr, bitmap_path.encode(),
                                                 cluster.ptr, C.byref(out)))
        h = Handle(self, out, "hp_recovery_free")
        js = C.c_void_p()
        self._check(self.lib.hp_recovery_to_json(h.ptr, C.byref(js)))
        return self._take_string(js)

    def plan_load(self, path: str) -> "Handle":
        h = _VP()
        self._check(self.lib.hp_plan_load_file(path.encode(), C.byref(h)))
        return Handle(self, h, "hp_plan_free")

    def _sim_options(self, combined_time, fb_ratio, zero_comm):
        o = hp_sim_options()
        self.lib.hp_sim_options_init(C.byref(o))
        o.combined_time = int(combined_time)
        if fb_ratio is not None:
            o.fb_ratio = fb_ratio
        o.zero_comm = int(zero_comm)
        return o

    def _sim_outputs(self, h):
        js, csv = C.c_void_p(), C.c_void_p()
        self._check(self.lib.hp_sim_result_to_json(h, C.byref(js)))
        self._check(self.lib.hp_sim_timeline_csv(h, C.byref(csv)))
        out = (self._take_string(js), self._take_string(csv), self.lib.hp_sim_makespan(h))
        self.lib.hp_sim_result_free(h)
        return out

    def simulate(self, plan, cluster, model, profile, combined_time=False, fb_ratio=None,
                 zero_comm=False):
        """hp_simulate + hp_sim_result_to_json + hp_sim_timeline_csv:
        (json, csv, makespan)."""
        o = self._sim_options(combined_time, fb_ratio, zero_comm)
        h = _VP()
        self._check(self.lib.hp_simulate(plan.ptr, cluster.ptr, model.ptr, profile.ptr,
                                         C.byref(o), C.byref(h)))
        return self._sim_outputs(h)

    def simulate_batch(self, plans, clusters, model, profiles, combined_time=False,
                       fb_ratio=None, zero_comm=False):
        """hp_simulate_batch (product extension): every plan in one launch."""
        n = len(plans)
        o = self._sim_options(combined_time, fb_ratio, zero_comm)
        out = (_VP * n)()
        rc = self.lib.hp_simulate_batch(n, (_VP * n)(*[p.ptr for p in plans]),
                                        (_VP * n)(*[c.ptr for c in clusters]), model.ptr,
                                        (_VP * n)(*[p.ptr for p in profiles]), C.byref(o), out)
        if rc != HP_OK:
            raise HetplanError(rc, self.lib.hpk_last_error().decode())
        return [self._sim_outputs(_VP(out[i])) for i in range(n)]

    def plan_json(self, cluster_text: str, model_text: str, max_layers: int,
                  options: Optional[PlanOptions] = None, base_seconds: float = 0.05) -> str:
        """Convenience: parse, synthesize the profile, plan, serialize."""
        cl = self.cluster_parse(cluster_text)
        md = self.model_parse(model_text)
        pr = self.profile_synth(cl, base_seconds, max_layers)
        return self.plan_to_json(self.plan_compute(cl, md, pr, options))


class Handle:
    """Owns one opaque hp_* handle; freed with the matching hp_*_free."""

    def __init__(self, lib: HetplanLib, ptr: C.c_void_p, free_name: str):
        self.lib = lib
        self.ptr = ptr
        self._free = getattr(lib.lib, free_name)

    def close(self) -> None:
        if self.ptr:
            self._free(self.ptr)
            self.ptr = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
