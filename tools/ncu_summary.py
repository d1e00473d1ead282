"""Print the key metrics of an ncu report (raw page) and a launch-list share table.
usage: python tools/ncu_summary.py REPORT.ncu-rep [launches.csv]"""
import csv
import io
import subprocess
import sys
from collections import defaultdict

WANT = ["gpu__time_duration.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "sm__inst_executed.sum",
        "smsp__warps_eligible.avg.per_cycle_active", "smsp__thread_inst_executed_per_inst_executed.ratio",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "smsp__average_warp_latency_per_inst_issued.ratio", "dram__bytes_read.sum",
        "dram__bytes_write.sum", "lts__t_sector_hit_rate.pct", "l1tex__t_sector_hit_rate.pct",
        "launch__registers_per_thread", "launch__shared_mem_per_block_dynamic", "launch__grid_size"]

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr, units, vals = rows[0], rows[1], rows[2]
for w in WANT:
    if w in hdr:
        i = hdr.index(w)
        print(f"| {w} | {vals[i]} {units[i]} |")
if len(sys.argv) > 2:
    rows = list(csv.reader(open(sys.argv[2])))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hi]
    ki, mi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    agg = defaultdict(list)
    for r in rows[hi + 1:]:
        if len(r) > mi:
            v = float(r[mi].replace(",", ""))
            v *= {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3,
                  "msecond": 1e3}.get(r[ui], 1.0)
            agg[r[ki].split("(")[0]].append(v)
    tot = sum(sum(v) for v in agg.values())
    for k, v in sorted(agg.items(), key=lambda x: -sum(x[1])):
        print(f"| {k} | {len(v)} | {sum(v) / len(v):.1f} us | {100 * sum(v) / tot:.1f} % |")
