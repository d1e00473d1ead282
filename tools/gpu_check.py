"""GPU bring-up check: parity of the B200 engine against the oracle and the
reference library, printed step by step (run under gpurun with a timeout)."""
import json
import os
import random
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from oracle.binding import REF_LIB, Oracle
from paper_2512_20953_b200.configs import min_mem_for, units_for  # noqa: E402
from paper_2512_20953_b200 import configs  # noqa: E402
from paper_2512_20953_b200.capi import HetplanLib  # noqa: E402
from paper_2512_20953_b200.engine import Engine, GroupingProblem  # noqa: E402


def log(*a):
    print(*a, flush=True)


def main():
    which = sys.argv[1:] or ["small", "random", "plans"]
    eng = Engine()
    log("engine", eng.version(), "devices", eng.device_count())
    orc = Oracle()
    if "small" in which:
        pb = GroupingProblem([1.0, 1.0, 2.0], [10.0, 10.0, 10.0], 8, 5.0, [0, 0, 1], [0, 0, 1])
        for fs in (False, True):
            r = eng.grouping_search([pb], force_serial=fs)[0]
            o = orc.solve_grouping(pb.power, pb.memory, 8, 5.0, pb.type_key, pb.node_key)
            log("small serial=%d" % fs, r.status, r.rgs, r.objective, r.visited, r.optimal,
                "| oracle", o.rgs, o.objective, o.visited, o.optimal)
    if "random" in which or any(a.startswith("cap:") for a in which):
        rng = random.Random(7)
        probs = []
        for trial in range(int(os.environ.get("NRAND", "300"))):
            n = rng.randint(1, 12)
            P = [rng.choice([0.5, 1.0, 1.5, 2.0, 3.0]) for _ in range(n)]
            M = [float(rng.randint(4, 20)) for _ in range(n)]
            T = [int(p * 2) for p in P]
            N = sorted(rng.randint(0, 3) for _ in range(n))
            K = rng.randint(1, 16)
            MIN = sum(M) * rng.uniform(0.1, 0.9) / rng.randint(1, 4)
            if rng.random() < 0.5:
                MIN = float(round(MIN))
            thr = rng.choice([0, 8, 100])
            B = rng.randint(1, 3000)
            probs.append(GroupingProblem(P, M, K, MIN, T, N, thr, B))
        caps = [int(a.split(":")[1]) for a in which if a.startswith("cap:")] or [2, 5, 64, 2048]
        for cap in caps:
            t = time.time()
            if cap < 16:  # tiny caps only on small trees (progress is ~1 split per wave)
                sub = [p for p in probs if p.n <= 8 or p.exact_threshold < p.n and p.node_budget <= 300]
            else:
                sub = probs
            res = eng.grouping_search(sub, segment_cap=cap, max_seconds=30)
            probs_run = sub
            bad = 0
            for pb, r in zip(probs_run, res):
                o = orc.solve_grouping(pb.power, pb.memory, pb.n_microbatches, pb.min_mem,
                                       pb.type_key, pb.node_key, pb.exact_threshold,
                                       pb.node_budget)
                if o.status != 0:
                    ok = r.status == o.status
                else:
                    ok = (r.status == 0 and r.rgs[0] == o.rgs[0] and r.objective[0] == o.objective[0]
                          and r.z[0] == o.z[0] and r.visited == o.visited and r.optimal == o.optimal)
                if not ok:
                    bad += 1
                    if bad <= 3:
                        log("  MISMATCH", pb, "\n   gpu", r, "\n   orc", o.status, o.rgs, o.objective,
                            o.visited, o.optimal)
            log("random cap=%d: %d problems, %d mismatches, %.2fs" % (cap, len(probs_run), bad,
                                                                     time.time() - t))
        if "serial" not in which:
            probs = []
        res = eng.grouping_search(probs, force_serial=True) if probs else []
        bad = 0
        for pb, r in zip(probs, res):
            o = orc.solve_grouping(pb.power, pb.memory, pb.n_microbatches, pb.min_mem,
                                   pb.type_key, pb.node_key, pb.exact_threshold, pb.node_budget)
            ok = (r.status == o.status) if o.status else (
                r.rgs[0] == o.rgs[0] and r.objective[0] == o.objective[0]
                and r.visited == o.visited and r.optimal == o.optimal)
            bad += 0 if ok else 1
        log("random serial engine: %d mismatches" % bad)
    if "cfg" in which or "plans" in which:
        for name in ("cfg1", "cfg2", "cfg3", "cfg4"):
            w = configs.get(name)
            import math
            g = 0
            for nd in w.cluster["nodes"]:
                g = math.gcd(g, nd["count"])
            probs = []
            for tp in [t for t in range(1, g + 1) if g % t == 0]:
                P, M, T, N = units_for(w.cluster, tp)
                probs.append(GroupingProblem(P, M, w.model["n_microbatches"], min_mem_for(w.model),
                                             T, N))
            t = time.time()
            res = eng.grouping_search(probs)
            dt = time.time() - t
            tm = eng.timing()
            for pb, r in zip(probs, res):
                o = orc.solve_grouping(pb.power, pb.memory, pb.n_microbatches, pb.min_mem,
                                       pb.type_key, pb.node_key)
                same = (r.rgs[0] == o.rgs[0] and r.objective[0] == o.objective[0]
                        and r.visited == o.visited and r.optimal == o.optimal)
                log(" %s n=%d %s visited=%d waves=%d runs=%d run_visits=%d max_list=%d" % (
                    name, pb.n, "OK" if same else "DIFF", r.visited, r.waves, r.segment_runs,
                    r.segment_visits, r.max_list))
            log("%s search: wall %.2f ms, kernel %.2f ms" % (name, dt * 1e3, tm.search_ms))
    if "plans" in which:
        prod = HetplanLib(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                       "paper_2512_20953_b200", "libhetplan_b200.so"))
        ref = HetplanLib(REF_LIB)
        for name in ("cfg1", "cfg2", "cfg3", "cfg4"):
            w = configs.get(name)
            t = time.time()
            a = prod.plan_json(w.cluster_json(), w.model_json(), w.max_layers)
            ta = time.time() - t
            t = time.time()
            b = ref.plan_json(w.cluster_json(), w.model_json(), w.max_layers)
            tb = time.time() - t
            log("plan %s: %s  b200 %.1f ms  ref %.1f ms" % (name, "BYTE-IDENTICAL" if a == b else "DIFF",
                                                        ta * 1e3, tb * 1e3))
            if a != b:
                import difflib
                for line in list(difflib.unified_diff(b.splitlines(), a.splitlines(), lineterm=""))[:40]:
                    log("   ", line)


if __name__ == "__main__":
    main()
