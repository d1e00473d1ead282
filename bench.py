"""Benchmark: parallelism-plan search (AutoHet / hetplan) on the B200.

Metric (BASELINE.json): candidate plans evaluated/sec and plan-search latency
(ms). A "candidate" is one grouping-search visit — the reference's own counter
GroupingSolution::nodes_visited (P/include/hetplan/grouping.hpp:64) summed
over the TP dimensions of one plan search. A step = one full default-option
plan search of the workload (all TP dimensions: grouping search, stage
mapping, layer partition, cost, selection).

  value  device-resident throughput: visits / (wave-engine + partition kernel
         time, CUDA events on the launching stream), inputs already in HBM
  e2e    the same metric through the public C ABI hp_plan_compute with host
         buffers (host<->device copies, host stage mapping, plan assembly all
         inside the timed region); ms_per_step is this latency

--impl reference times the reference planner (oracle/_ref/libhetplan.so, the
reference compiled from its own sources) on this host's CPU, same workload.

Multi-GPU (torchrun, one process per GPU): the TP-dimension searches of one
plan are sharded across ranks (strong scaling); each rank's results are
exchanged with an NCCL all_gather (torch.distributed) and every rank replays
the reference selection. Max-over-ranks device time.
"""
from __future__ import annotations

import argparse
import json
import math
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


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            threading.Thread(target=self._read, daemon=True).start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc:
            time.sleep(0.25)
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


def workload(name):
    from paper_2512_20953_b200 import configs
    return configs.get(name)


def tp_problems(w):
    """The grouping problems of one plan search (one per valid TP dimension)."""
    from paper_2512_20953_b200.configs import min_mem_for, units_for  # data prep only (no compute)
    from paper_2512_20953_b200.engine import GroupingProblem
    g = 0
    for nd in w.cluster["nodes"]:
        g = math.gcd(g, nd["count"])
    out = []
    for tp in [t for t in range(1, g + 1) if g % t == 0]:
        P, M, T, N = units_for(w.cluster, tp)
        out.append((tp, GroupingProblem(P, M, w.model["n_microbatches"], min_mem_for(w.model),
                                        T, N)))
    return out


def cpu_baseline(w, budget_s=10.0):
    """Reference planner (compiled from its own sources) on one host core."""
    from oracle.binding import REF_LIB
    from paper_2512_20953_b200.capi import HetplanLib
    if not os.path.exists(REF_LIB):
        return None
    ref = HetplanLib(REF_LIB)
    cl = ref.cluster_parse(w.cluster_json())
    md = ref.model_parse(w.model_json())
    pr = ref.profile_synth(cl, w.base_seconds, w.max_layers)
    times = []
    t_end = time.time() + budget_s
    while time.time() < t_end and len(times) < 50:
        t0 = time.perf_counter()
        plan = ref.plan_compute(cl, md, pr)
        times.append(time.perf_counter() - t0)
        plan.close()
    return times


def visits_of(w):
    """Reference visits per plan search (oracle restatement; workload constant)."""
    from oracle.binding import Oracle
    o = Oracle()
    tot = 0
    ops = 0.0
    for tp, pb in tp_problems(w):
        r = o.solve_grouping(pb.power, pb.memory, pb.n_microbatches, pb.min_mem, pb.type_key,
                             pb.node_key)
        tot += r.visited
        ops += r.stats.model_ops
    return tot, ops


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    w = workload(args.workload)
    visits, _ = visits_of(w)
    times = []
    from oracle.binding import REF_LIB
    from paper_2512_20953_b200.capi import HetplanLib
    ref = HetplanLib(REF_LIB)
    cl = ref.cluster_parse(w.cluster_json())
    md = ref.model_parse(w.model_json())
    pr = ref.profile_synth(cl, w.base_seconds, w.max_layers)
    for i in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        ref.plan_compute(cl, md, pr).close()
        dt = time.perf_counter() - t0
        if i >= args.warmup:
            times.append(dt)
    ms = statistics.mean(times) * 1e3
    value = visits / (ms * 1e-3)
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": w.name, "parallelism": "single host thread (reference planner "
                   "is single-threaded)", "options": "reference defaults"},
        "latency_ms": ms,
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": 1, "kind": "reference",
                         "sample": f"{args.steps} full {w.name} plan searches "
                                   f"(hp_plan_compute, oracle/_ref/libhetplan.so)"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def run_b200(args):
    import torch
    from paper_2512_20953_b200.capi import HetplanLib
    from paper_2512_20953_b200.engine import LIB_PATH, Engine

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    eng = Engine()
    if eng.device_count() < 1:
        raise SystemExit("no CUDA device")
    w = workload(args.workload)
    probs = tp_problems(w)
    # shard the TP-dimension problems over ranks (longest-first by estimated cost)
    from paper_2512_20953_b200.shard import search_cost, shard_indices, sharded_map
    costs = [search_cost(pb) for _, pb in probs]  # longest search on its own GPU first
    mine = [probs[i][1] for i in shard_indices(len(probs), rank, world, costs)]

    def barrier():
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()

    # L2 flush buffer (> 126 MB L2), written between timed iterations
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")

    # ---- device-resident leg: the kernels themselves (CUDA events inside the library)
    dev_ms, launches, visits_done = [], 0, 0
    for i in range(args.warmup + args.steps):
        flush.zero_()
        barrier()
        eng.reset_timing()
        res = eng.grouping_search(mine, device=local) if mine else []
        t = eng.timing()
        barrier()
        if i >= args.warmup:
            dev_ms.append(t.search_ms + t.serial_ms + t.partition_ms)
            launches += t.kernel_launches
            visits_done += sum(r.visited for r in res)
    # every rank ends with the full, problem-ordered result list (one all-gather)
    full = sharded_map([pb for _, pb in probs],
                       lambda b: [(r.visited, r.optimal, r.objective, r.rgs)
                                  for r in eng.grouping_search(b, device=local)], dist, costs)
    assert len(full) == len(probs)
    ms_local = statistics.mean(dev_ms) if dev_ms else 0.0
    ms_max = ms_local
    total_visits = visits_done / max(1, args.steps)
    if dist is not None:
        tt = torch.tensor([ms_local, total_visits], dtype=torch.float64, device="cuda")
        gathered = [torch.zeros_like(tt) for _ in range(world)]
        dist.all_gather(gathered, tt)
        ms_max = max(float(g[0]) for g in gathered)
        total_visits = sum(float(g[1]) for g in gathered)

    # ---- e2e leg: public C ABI, host buffers (rank 0 at N=1; every rank plans
    # the full workload at N>1 is not sharded through the ABI yet -> rank 0 only)
    e2e = None
    e2e_ms = None
    if rank == 0:
        lib = HetplanLib(LIB_PATH)
        cl = lib.cluster_parse(w.cluster_json())
        md = lib.model_parse(w.model_json())
        pr = lib.profile_synth(cl, w.base_seconds, w.max_layers)
        e2e_times, h2d, d2h, e2e_launches = [], 0, 0, 0
        for i in range(args.warmup + args.steps):
            flush.zero_()
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            plan = lib.plan_compute(cl, md, pr)
            js = lib.plan_to_json(plan)  # device->host result read is inside compute
            dt = time.perf_counter() - t0
            plan.close()
            t = eng.timing()
            if i >= args.warmup:
                e2e_times.append(dt)
                h2d += t.h2d_bytes
                d2h += t.d2h_bytes
                e2e_launches += t.kernel_launches
        e2e_ms = statistics.mean(e2e_times) * 1e3
        e2e_visits = sum(r.visited for r in eng.grouping_search([pb for _, pb in probs]))
        e2e = {"value": e2e_visits / (e2e_ms * 1e-3), "unit": UNIT,
               "h2d_bytes_per_step": h2d // args.steps, "d2h_bytes_per_step": d2h // args.steps,
               "latency_ms": e2e_ms}

    if rank != 0:
        if dist is not None:
            dist.barrier()
            dist.destroy_process_group()
        return

    # ---- clocks during a timed window of repeated searches
    with ClockSampler(local) as cs:
        t_end = time.time() + 1.0
        while time.time() < t_end:
            eng.grouping_search(mine, device=local)
    clocks = cs.summary()

    # ---- roofline: fp64-issue bound (measured peak on this GPU)
    import ctypes as C
    f64 = C.c_double()
    i32 = C.c_double()
    eng.lib.hpk_measure_issue_peaks.argtypes = [C.c_int, C.POINTER(C.c_double),
                                                C.POINTER(C.c_double)]
    eng.lib.hpk_measure_issue_peaks(local, C.byref(f64), C.byref(i32))
    ref_visits, model_ops = visits_of(w)
    achieved = model_ops / (ms_max * 1e-3) / 1e9 if ms_max > 0 else 0.0
    peak = f64.value / 1e9
    traffic = None
    try:  # dram read+write per launch of the dominant kernel, from the committed ncu capture
        with open(os.path.join(ROOT, "profiles", "r1_traffic.json")) as f:
            traffic = json.load(f)["hpk_wave_kernel"]["traffic_bytes_per_launch"]
    except Exception:
        pass
    roofline = {"bound": "fp64-issue", "achieved": achieved, "peak": peak, "unit": "GFLOP/s",
                "frac": achieved / peak if peak else None, "traffic": traffic,
                "traffic_unit": "bytes/launch (ncu dram__bytes_read+write, profiles/r1_traffic.json)",
                "ops_per_launch": model_ops, "int32_peak_gops": i32.value / 1e9,
                "peak_source": "measured (hpk_measure_issue_peaks: DMUL+DADD chains, this GPU)",
                "note": "fp64-op model of SURVEY.md 8(d) (reference ops), whole plan search",
                "issue": _issue_roofline("cfg4")}

    cpu = cpu_baseline(w)
    cpu_line = None
    if cpu:
        cms = statistics.median(cpu) * 1e3
        cpu_line = {"value": ref_visits / (cms * 1e-3), "unit": UNIT, "cores": 1,
                    "kind": "reference", "latency_ms": cms,
                    "sample": f"{len(cpu)} full {w.name} plan searches on 1 host core "
                              f"(oracle/_ref/libhetplan.so, median)",
                    "host_cpu": _cpu_model(), "host_cores": os.cpu_count()}

    value = total_visits / (ms_max * 1e-3) if ms_max > 0 else 0.0
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": e2e_ms if e2e_ms else ms_max,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic",
        "config": {"workload": w.name, "tp_dims": [tp for tp, _ in probs],
                   "parallelism": f"tp-dimension searches sharded over {world} GPU(s)",
                   "options": "reference defaults (exact_threshold 8, node_budget 5e6, top_k 1)",
                   "l2": "flushed between timed iterations (256 MB write)"},
        "device_ms_per_step": ms_max,
        "latency_ms": e2e_ms,
        "visits_per_step": total_visits,
        "e2e": e2e,
        "roofline": roofline,
        "cpu_baseline": cpu_line,
        "clocks": clocks,
        "gpu_launches": launches,
    }
    print(json.dumps(line), flush=True)
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()


def _snapshot_inputs(lib, snaps):
    cl = [lib.cluster_parse(w.cluster_json()) for w in snaps]
    md = lib.model_parse(snaps[0].model_json())
    pr = [lib.profile_synth(c, w.base_seconds, w.max_layers) for c, w in zip(cl, snaps)]
    return cl, md, pr


def _ref_plan_one(i):
    """Worker of the cfg5 reference arm: one snapshot through the reference C ABI."""
    from oracle.binding import REF_LIB
    from paper_2512_20953_b200 import configs
    from paper_2512_20953_b200.capi import HetplanLib
    w = configs.cfg5_snapshots(i + 1)[i]
    ref = HetplanLib(REF_LIB)
    cl = ref.cluster_parse(w.cluster_json())
    md = ref.model_parse(w.model_json())
    pr = ref.profile_synth(cl, w.base_seconds, w.max_layers)
    t0 = time.perf_counter()
    ref.plan_compute(cl, md, pr).close()
    return time.perf_counter() - t0


def _cfg5_sample_visits():
    with open(os.path.join(ROOT, "tests", "golden", "cfg5_visits.json")) as f:
        return [r["visits"] for r in json.load(f)]


def run_reference_cfg5(args):
    """Reference planner over a bounded sample of the sweep on ALL host cores
    (independent snapshots, one process each: the reference is single-threaded)."""
    if int(os.environ.get("RANK", "0")) != 0:
        return
    import multiprocessing as mp
    vis = _cfg5_sample_visits()
    cores = os.cpu_count() or 1
    sample = min(len(vis), max(cores, 2 * cores))
    times = []
    with mp.get_context("spawn").Pool(cores) as pool:
        for i in range(args.warmup + args.steps):
            t0 = time.perf_counter()
            pool.map(_ref_plan_one, range(sample))
            dt = time.perf_counter() - t0
            if i >= args.warmup:
                times.append(dt)
    ms = statistics.mean(times) * 1e3
    value = sum(vis[:sample]) / (ms * 1e-3)
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"cfg5 replanning sweep (sample of {sample} snapshots per step)",
                   "parallelism": f"{cores} host processes", "options": "reference defaults"},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "reference",
                         "sample": f"snapshots 0..{sample - 1} of the seed-2512 sweep per step"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def run_b200_cfg5(args):
    """The replanning sweep: every snapshot's plan search batched into one
    hp_plan_compute_batch call per rank (snapshots sharded round-robin over ranks)."""
    import torch
    from paper_2512_20953_b200 import configs
    from paper_2512_20953_b200.capi import HetplanLib
    from paper_2512_20953_b200.engine import LIB_PATH, Engine

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    eng = Engine()
    from paper_2512_20953_b200.shard import shard_indices
    snaps = configs.cfg5_snapshots(args.snapshots)
    mine = [snaps[i] for i in shard_indices(len(snaps), rank, world)]
    probs = [pb for w in mine for _, pb in tp_problems(w)]
    lib = HetplanLib(LIB_PATH)
    cl, md, pr = _snapshot_inputs(lib, mine)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")

    def barrier():
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()

    dev_ms, e2e_ms, launches, visits, h2d, d2h = [], [], 0, 0, 0, 0
    for i in range(args.warmup + args.steps):
        flush.zero_()
        barrier()
        eng.reset_timing()
        res = eng.grouping_search(probs, device=local)
        t = eng.timing()
        flush.zero_()
        barrier()
        t0 = time.perf_counter()
        out = lib.plan_compute_batch(cl, md, pr)
        dt = time.perf_counter() - t0
        te = eng.timing()
        bad = [st for st, _, _ in out if st != 0]
        if bad:
            raise SystemExit(f"cfg5: {len(bad)} snapshots failed to plan")
        barrier()
        if i >= args.warmup:
            dev_ms.append(t.search_ms + t.serial_ms)
            e2e_ms.append(dt * 1e3)
            launches += t.kernel_launches + te.kernel_launches
            visits = sum(r.visited for r in res)
            h2d += te.h2d_bytes
            d2h += te.d2h_bytes
    local_vals = [statistics.mean(dev_ms), statistics.mean(e2e_ms), float(visits)]
    vals = [local_vals]
    if dist is not None:
        tt = torch.tensor(local_vals, dtype=torch.float64, device="cuda")
        g = [torch.zeros_like(tt) for _ in range(world)]
        dist.all_gather(g, tt)
        vals = [[float(x) for x in v] for v in g]
    if rank != 0:
        dist.barrier()
        dist.destroy_process_group()
        return
    dev_max = max(v[0] for v in vals)
    e2e_max = max(v[1] for v in vals)
    total_visits = sum(v[2] for v in vals)
    with ClockSampler(local) as cs:
        t_end = time.time() + 1.0
        while time.time() < t_end:
            eng.grouping_search(probs[: max(1, len(probs) // 8)], device=local)
    # CPU baseline: the reference on 1 core over a small sample (scaled per visit)
    svis = _cfg5_sample_visits()
    k = min(4, len(svis))
    ct = [_ref_plan_one(i) for i in range(k)]
    cpu_value = sum(svis[:k]) / sum(ct)
    # roofline: fp64-op model ops per visit from the oracle on the sampled
    # snapshots, scaled to the sweep's visits; measured peak
    import ctypes as C
    f64, i32 = C.c_double(), C.c_double()
    eng.lib.hpk_measure_issue_peaks.argtypes = [C.c_int, C.POINTER(C.c_double),
                                                C.POINTER(C.c_double)]
    eng.lib.hpk_measure_issue_peaks(local, C.byref(f64), C.byref(i32))
    sv = so = 0.0
    for w in configs.cfg5_snapshots(k):
        v, o = visits_of(w)
        sv += v
        so += o
    ops = total_visits * (so / sv) if sv else 0.0
    achieved = ops / (dev_max * 1e-3) / 1e9 if dev_max > 0 else 0.0
    roofline = {"bound": "fp64-issue", "achieved": achieved, "peak": f64.value / 1e9,
                "unit": "GFLOP/s", "frac": achieved * 1e9 / f64.value if f64.value else None,
                "traffic": None, "ops_per_launch": ops,
                "peak_source": "measured (hpk_measure_issue_peaks: DMUL+DADD chains, this GPU)",
                "note": f"fp64-op model of SURVEY.md 8(d), ops per visit sampled on snapshots "
                        f"0..{k - 1} ({so / sv if sv else 0:.2f})",
                "issue": _issue_roofline("cfg5")}
    line = {
        "metric": METRIC, "value": total_visits / (dev_max * 1e-3), "unit": UNIT,
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": e2e_max,
        "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"cfg5 replanning sweep: {args.snapshots} snapshots of the cfg3 "
                   "cluster (seed 2512)", "parallelism": f"snapshots sharded over {world} GPU(s)",
                   "options": "reference defaults", "l2": "flushed between timed iterations"},
        "device_ms_per_step": dev_max,
        "visits_per_step": total_visits,
        "e2e": {"value": total_visits / (e2e_max * 1e-3), "unit": UNIT,
                "h2d_bytes_per_step": h2d // args.steps, "d2h_bytes_per_step": d2h // args.steps,
                "latency_ms": e2e_max},
        "cpu_baseline": {"value": cpu_value, "unit": UNIT, "cores": 1, "kind": "reference",
                         "sample": f"snapshots 0..{k - 1}, hp_plan_compute on 1 host core",
                         "host_cores": os.cpu_count()},
        "roofline": roofline,
        "clocks": cs.summary(),
        "gpu_launches": launches,
    }
    print(json.dumps(line), flush=True)
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()


def _issue_roofline(workload):
    """The instruction-issue roofline of the search kernel (the bound that applies
    to this control-heavy tree search): ncu's issue-slot utilization of the same
    workload, from the committed capture (profiles/r1_issue.json)."""
    try:
        with open(os.path.join(ROOT, "profiles", "r1_issue.json")) as f:
            rec = json.load(f)["hpk_wave_kernel"][workload]
        return {"bound": "instruction-issue", "frac": rec["issue_active_pct"] / 100.0,
                "fp64_pipe_frac": rec["fp64_pipe_pct"] / 100.0, "source": rec["source"]}
    except Exception:
        return None


def _cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    return ln.split(":", 1)[1].strip()
    except Exception:
        pass
    return None


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--workload", default="cfg4",
                    choices=["cfg1", "cfg2", "cfg3", "cfg4", "cfg5"])
    ap.add_argument("--snapshots", type=int, default=1000, help="cfg5 sweep size")
    args = ap.parse_args()
    if args.workload == "cfg5":
        (run_reference_cfg5 if args.impl == "reference" else run_b200_cfg5)(args)
    elif args.impl == "reference":
        run_reference(args)
    else:
        run_b200(args)


if __name__ == "__main__":
    main()
