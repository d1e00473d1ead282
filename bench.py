"""Benchmark: parallelism-plan search (AutoHet / hetplan) on the B200.

Metric (BASELINE.json): candidate plans evaluated/sec and plan-search latency
(ms). A "candidate" is one grouping-search visit — the reference's own counter
GroupingSolution::nodes_visited (P/include/hetplan/grouping.hpp:64) summed over
the TP dimensions of one plan search (profiles/workload_stats.json). A step is
one full default-option plan search of the workload through the product's
public C ABI, hp_plan_compute (grouping search, stage mapping, layer partition,
cost, selection), with host buffers.

  e2e    the headline: candidates / wall time of hp_plan_compute, the same
         call the reference arm times (host<->device copies, the device->host
         read of every kernel's results and every host phase inside the timed
         region)
  value  the same calls, device time only: the kernels' CUDA-event durations
         on their launching streams (grouping search = max over GPUs, + stage
         affinity + partition/cost), i.e. throughput with inputs resident

Multi-GPU: hp_plan_compute drives every visible GPU from one call (the TP-
dimension searches of a plan, or a sweep's snapshots, go longest-first to the
least-loaded device). Under torchrun rank 0 restricts CUDA_VISIBLE_DEVICES to
the job's N devices and plans; the other ranks hold their GPU and wait at the
barrier. Strong scaling: the workload is fixed as N grows.

workloads: cfg1-3 latency and the cfg5 1000-snapshot sweep
(hp_plan_compute_batch), each beside the reference planner on this host.

--impl reference times the reference planner (oracle/_ref/libhetplan.so, the
reference compiled from its own sources) on this host's CPU, same workload.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "candidate plans evaluated/sec and plan-search latency (ms) at 1/2/4/8 B200"
UNIT = "candidates/s"


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def stats():
    with open(os.path.join(ROOT, "profiles", "workload_stats.json")) as f:
        return json.load(f)


class ClockSampler:
    """nvidia-smi clocks + throttle reasons, sampled while the timed loop runs."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, indices):
        self.indices = ",".join(str(i) for i in indices)
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", self.indices, f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            threading.Thread(target=self._read, daemon=True).start()
            time.sleep(0.1)
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc:
            time.sleep(0.1)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for nm, v in zip(names, parts[4:8]):
                if v.lower() == "active":
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


def _cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    return ln.split(":", 1)[1].strip()
    except Exception:
        pass
    return None


# ------------------------------------------------------------ reference (CPU)

def _ref_lib():
    from oracle.binding import REF_LIB
    from paper_2512_20953_b200.capi import HetplanLib
    return HetplanLib(REF_LIB)


def ref_plan_times(w, steps, warmup=0, budget_s=None):
    """The reference planner (compiled from its own sources) on one host core:
    wall time of hp_plan_compute per plan search."""
    ref = _ref_lib()
    cl = ref.cluster_parse(w.cluster_json())
    md = ref.model_parse(w.model_json())
    pr = ref.profile_synth(cl, w.base_seconds, w.max_layers)
    times = []
    t_end = time.time() + budget_s if budget_s else None
    for i in range(warmup + steps):
        t0 = time.perf_counter()
        ref.plan_compute(cl, md, pr).close()
        dt = time.perf_counter() - t0
        if i >= warmup:
            times.append(dt)
        if t_end and time.time() > t_end and len(times) >= 3:
            break
    return times


def _ref_plan_snapshot(i):
    """Worker of the cfg5 reference leg: one snapshot through the reference C ABI."""
    from paper_2512_20953_b200 import configs
    w = configs.cfg5_snapshots(i + 1)[i]
    ref = _ref_lib()
    cl = ref.cluster_parse(w.cluster_json())
    md = ref.model_parse(w.model_json())
    pr = ref.profile_synth(cl, w.base_seconds, w.max_layers)
    t0 = time.perf_counter()
    ref.plan_compute(cl, md, pr).close()
    return time.perf_counter() - t0


def ref_cfg5_rate(sample):
    """Reference planner over snapshots 0..sample-1 as independent processes on
    ALL host cores (it is single-threaded and reentrant): candidates/s."""
    import multiprocessing as mp
    vis = stats()["cfg5"]["sample_visits"][:sample]
    cores = os.cpu_count() or 1
    with mp.get_context("spawn").Pool(cores) as pool:
        pool.map(_ref_plan_snapshot, range(min(cores, sample)))  # warm the workers
        t0 = time.perf_counter()
        pool.map(_ref_plan_snapshot, range(sample), chunksize=1)
        dt = time.perf_counter() - t0
    return sum(vis) / dt, dt, cores


def run_reference(args):
    if int(os.environ.get("RANK", "0")) != 0:
        return
    from paper_2512_20953_b200 import configs
    st = stats()
    if args.workload == "cfg5":
        sample = min(256, max(8 * (os.cpu_count() or 1), 32))
        rates = [ref_cfg5_rate(sample) for _ in range(max(1, args.steps // 5))]
        value = statistics.mean(r[0] for r in rates)
        cores = rates[0][2]
        ms = st["cfg5"]["visits"] / value * 1e3
        line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
                "n_gpus": args.gpus, "steps": len(rates), "warmup": 0, "ms_per_step": ms,
                "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
                "dtype": "f64", "data": "synthetic",
                "config": {"workload": "cfg5 replanning sweep, 1000 snapshots (projected from "
                           f"a {sample}-snapshot sample)", "parallelism": f"{cores} host processes"},
                "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores,
                                 "kind": "reference", "sample": f"snapshots 0..{sample - 1}"},
                "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0,
                        "d2h_bytes_per_step": 0}}
        print(json.dumps(line), flush=True)
        return
    w = configs.get(args.workload)
    visits = st[args.workload]["visits"]
    times = ref_plan_times(w, args.steps, args.warmup)
    ms = statistics.mean(times) * 1e3
    value = visits / (ms * 1e-3)
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": w.name, "parallelism": "single host thread (the reference "
                   "planner is single-threaded)", "options": "reference defaults"},
        "latency_ms": ms,
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": 1, "kind": "reference",
                         "sample": f"{args.steps} full {w.name} plan searches "
                                   f"(hp_plan_compute, oracle/_ref/libhetplan.so)"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------ product (B200)

class Product:
    def __init__(self):
        from paper_2512_20953_b200.capi import HetplanLib
        from paper_2512_20953_b200.engine import LIB_PATH, Engine
        self.eng = Engine()
        if self.eng.device_count() < 1:
            raise SystemExit("no CUDA device")
        self.lib = HetplanLib(LIB_PATH)

    def device_ms(self):
        t = self.eng.timing()
        return t.search_ms + t.serial_ms + t.affinity_ms + t.partition_ms, t


def _flushers(n):
    import torch
    return [torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=f"cuda:{d}")
            for d in range(n)]


def _flush(bufs):
    import torch
    for b in bufs:
        b.zero_()
    for d in range(len(bufs)):
        torch.cuda.synchronize(d)


def time_plans(prod, w, steps, warmup, flush):
    """steps x hp_plan_compute + plan JSON through the C ABI (L2 flushed on every
    GPU between steps). Returns per-step wall ms, device ms, and the counters."""
    lib = prod.lib
    cl = lib.cluster_parse(w.cluster_json())
    md = lib.model_parse(w.model_json())
    pr = lib.profile_synth(cl, w.base_seconds, w.max_layers)
    wall, dev, h2d, d2h, launches, ndev = [], [], 0, 0, 0, 0
    for i in range(warmup + steps):
        _flush(flush)
        prod.eng.reset_timing()
        t0 = time.perf_counter()
        plan = lib.plan_compute(cl, md, pr)  # the plan (device results read back) is on the host
        dt = time.perf_counter() - t0
        plan.close()
        ms, t = prod.device_ms()
        if i >= warmup:
            wall.append(dt * 1e3)
            dev.append(ms)
            h2d += t.h2d_bytes
            d2h += t.d2h_bytes
            launches += t.kernel_launches
            ndev = max(ndev, t.devices_used)
    return wall, dev, h2d, d2h, launches, ndev


def time_sweep(prod, snaps, steps, flush):
    """The cfg5 sweep through hp_plan_compute_batch (one call plans every snapshot)."""
    lib = prod.lib
    cl = [lib.cluster_parse(w.cluster_json()) for w in snaps]
    md = lib.model_parse(snaps[0].model_json())
    pr = [lib.profile_synth(c, w.base_seconds, w.max_layers) for c, w in zip(cl, snaps)]
    wall, dev, launches = [], [], 0
    for i in range(1 + steps):
        _flush(flush)
        prod.eng.reset_timing()
        t0 = time.perf_counter()
        out = lib.plan_compute_batch(cl, md, pr)
        dt = time.perf_counter() - t0
        ms, t = prod.device_ms()
        if any(st != 0 for st, _, _ in out):
            raise SystemExit("cfg5: a snapshot failed to plan")
        for _, h, _ in out:
            h.close()
        if i >= 1:
            wall.append(dt * 1e3)
            dev.append(ms)
            launches += t.kernel_launches
    return wall, dev, launches


def roofline(prod, name, dev_ms, st, n_dev):
    """fp64-issue roofline of the plan search: the reference's
    fp64-op model of the visits / device time, against the fp64 issue peak
    measured on this GPU (x devices used)."""
    import ctypes as C
    f64, i32 = C.c_double(), C.c_double()
    L = prod.eng.lib
    L.hpk_measure_issue_peaks.argtypes = [C.c_int, C.POINTER(C.c_double),
                                          C.POINTER(C.c_double)]
    L.hpk_measure_issue_peaks(0, C.byref(f64), C.byref(i32))
    ops = (st[name]["model_ops"] if name != "cfg5"
           else st["cfg5"]["visits"] * st["cfg5"]["model_ops_per_visit"])
    achieved = ops / (dev_ms * 1e-3) / 1e9
    peak = f64.value / 1e9 * max(1, n_dev)
    out = {"bound": "fp64-issue", "achieved": achieved, "peak": peak, "unit": "GFLOP/s",
           "frac": achieved / peak if peak else None, "traffic": None,
           "ops_per_step": ops, "int32_peak_gops": i32.value / 1e9,
           "peak_source": "measured on this GPU (hpk_measure_issue_peaks: DMUL+DADD chains) "
                          f"x {max(1, n_dev)} GPU(s); MEASURED_PEAKS.json has no fp64 entry",
           "note": "reference fp64-op model of the visits (SURVEY.md 8(d)), whole plan search"}
    try:
        with open(os.path.join(ROOT, "profiles", "roofline_evidence.json")) as f:
            ev = json.load(f)
        key = "cfg5" if name == "cfg5" else "cfg4"
        out["traffic"] = ev.get("traffic", {}).get(key)
        out["traffic_unit"] = "DRAM bytes per launch of the search kernel (ncu)"
        out["issue"] = ev.get("issue", {}).get(key)
    except Exception:
        pass
    return out


def run_b200(args):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    n = max(world, args.gpus)
    if rank == 0:  # this process drives the job's N GPUs through the library
        vis = os.environ.get("CUDA_VISIBLE_DEVICES")
        ids = vis.split(",") if vis else [str(i) for i in range(n)]
        os.environ["CUDA_VISIBLE_DEVICES"] = ",".join(ids[:n])
    import torch
    dist = None
    if world > 1:
        import torch.distributed as dist
        torch.cuda.set_device(0 if rank == 0 else local)
        dist.init_process_group("nccl", device_id=torch.device(
            "cuda", 0 if rank == 0 else local))
    if rank != 0:  # the library in rank 0 drives this rank's GPU
        dist.barrier()
        dist.destroy_process_group()
        return
    from paper_2512_20953_b200 import configs
    prod = Product()
    ndev = prod.eng.device_count()
    st = stats()
    flush = _flushers(ndev)
    name = args.workload

    if name == "cfg5":
        snaps = configs.cfg5_snapshots(1000)
        with ClockSampler(range(ndev)) as cs:
            wall, dev, launches = time_sweep(prod, snaps, args.steps, flush)
        visits = st["cfg5"]["visits"]
        e2e_ms, dev_ms = statistics.mean(wall), statistics.mean(dev)
        h2d = d2h = None
        ndev_used = ndev
        wname = "cfg5 replanning sweep: 1000 snapshots of the cfg3 cluster (seed 2512)"
    else:
        w = configs.get(name)
        with ClockSampler(range(ndev)) as cs:
            wall, dev, h2d, d2h, launches, ndev_used = time_plans(prod, w, args.steps,
                                                                  args.warmup, flush)
        visits = st[name]["visits"]
        e2e_ms, dev_ms = statistics.mean(wall), statistics.mean(dev)
        wname = w.name
    clocks = cs.summary()

    # cross-check the candidate count against the product's own exact counter
    if name != "cfg5":
        from paper_2512_20953_b200.configs import min_mem_for, tp_dims_of, units_for
        from paper_2512_20953_b200.engine import HPK_ALL_DEVICES, GroupingProblem
        probs = []
        for tp in tp_dims_of(w.cluster):
            P, M, T, N = units_for(w.cluster, tp)
            if sum(M) >= min_mem_for(w.model):
                probs.append(GroupingProblem(P, M, w.model["n_microbatches"],
                                             min_mem_for(w.model), T, N))
        counted = sum(r.visited for r in prod.eng.grouping_search(probs, device=HPK_ALL_DEVICES))
        if counted != visits:
            raise SystemExit(f"visit count mismatch: engine {counted} vs reference {visits}")

    rl = roofline(prod, name, dev_ms, st, ndev_used)
    line = {
        "metric": METRIC, "value": visits / (dev_ms * 1e-3), "unit": UNIT, "n_gpus": n,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": e2e_ms,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic",
        "config": {"workload": wname,
                   "parallelism": f"one hp_plan_compute call drives {ndev} GPU(s) "
                                  f"(TP-dimension searches / snapshots longest-first)",
                   "options": "reference defaults (exact_threshold 8, node_budget 5e6, top_k 1)",
                   "l2": "flushed on every GPU between steps (256 MB write each)"},
        "latency_ms": e2e_ms, "device_ms_per_step": dev_ms, "visits_per_step": visits,
        "devices_used": ndev_used,
        "e2e": {"value": visits / (e2e_ms * 1e-3), "unit": UNIT,
                "h2d_bytes_per_step": h2d // args.steps if h2d is not None else None,
                "d2h_bytes_per_step": d2h // args.steps if d2h is not None else None,
                "latency_ms": e2e_ms},
        "roofline": rl,
        "clocks": clocks,
        "gpu_launches": launches,
    }
    if not args.no_cpu:
        times = ref_plan_times(configs.get("cfg4") if name == "cfg5" else w, 50, 1,
                               budget_s=10.0)
        cms = statistics.median(times) * 1e3
        cv = st["cfg4" if name == "cfg5" else name]["visits"]
        line["cpu_baseline"] = {"value": cv / (cms * 1e-3), "unit": UNIT, "cores": 1,
                                "kind": "reference", "latency_ms": cms,
                                "sample": f"{len(times)} full "
                                          f"{'cfg4' if name == 'cfg5' else name} plan searches "
                                          "on 1 host core (oracle/_ref/libhetplan.so, median)",
                                "host_cpu": _cpu_model(), "host_cores": os.cpu_count()}
    if not args.no_workloads and name != "cfg5":
        line["workloads"] = secondary_workloads(prod, flush, st, args)
    print(json.dumps(line), flush=True)
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()


def secondary_workloads(prod, flush, st, args):
    """cfg1-3 plan latency and the cfg5 sweep, each beside the reference on this host."""
    from paper_2512_20953_b200 import configs
    out = {}
    for nm in ("cfg1", "cfg2", "cfg3"):
        w = configs.get(nm)
        wall, dev, _, _, _, nd = time_plans(prod, w, 5, 2, flush)
        ref = ref_plan_times(w, 5, 1, budget_s=3.0) if not args.no_cpu else None
        out[nm] = {"workload": w.name, "visits": st[nm]["visits"],
                   "e2e_ms": statistics.mean(wall), "device_ms": statistics.mean(dev),
                   "devices_used": nd,
                   "reference_1core_ms": statistics.median(ref) * 1e3 if ref else None}
        if ref:
            out[nm]["e2e_speedup_vs_reference"] = out[nm]["reference_1core_ms"] / out[nm]["e2e_ms"]
    snaps = configs.cfg5_snapshots(1000)
    wall, dev, _ = time_sweep(prod, snaps, 2, flush)
    v = st["cfg5"]["visits"]
    rec = {"workload": "cfg5 sweep, 1000 snapshots, one hp_plan_compute_batch call",
           "visits": v, "e2e_ms": statistics.mean(wall), "device_ms": statistics.mean(dev),
           "e2e_candidates_per_s": v / (statistics.mean(wall) * 1e-3)}
    if not args.no_cpu:
        sample = min(256, max(8 * (os.cpu_count() or 1), 32))
        rate, dt, cores = ref_cfg5_rate(sample)
        rec["reference"] = {"candidates_per_s": rate, "cores": cores,
                            "projected_sweep_s": v / rate,
                            "sample": f"snapshots 0..{sample - 1} on {cores} host processes "
                                      f"({dt:.1f} s)"}
        rec["e2e_speedup_vs_reference_all_cores"] = rec["e2e_candidates_per_s"] / rate
    out["cfg5"] = rec
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--workload", default="cfg4",
                    choices=["cfg1", "cfg2", "cfg3", "cfg4", "cfg5"])
    ap.add_argument("--no-workloads", action="store_true", help="skip the secondary workloads")
    ap.add_argument("--no-cpu", action="store_true", help="skip the reference CPU legs")
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "b200":
        log("warning: fewer than 3 warm-up steps")
    (run_reference if args.impl == "reference" else run_b200)(args)


if __name__ == "__main__":
    main()
