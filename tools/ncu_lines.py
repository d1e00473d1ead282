"""Per-source-line warp-stall attribution of an ncu report (SASS page + nvdisasm -g line map).

usage: python tools/ncu_lines.py report.ncu-rep cubin kernel_mangled_substring source.cu [top]
"""
import collections
import csv
import io
import re
import subprocess
import sys

rep, cubin, kname, srcfile = sys.argv[1:5]
top = int(sys.argv[5]) if len(sys.argv) > 5 else 40
dis = subprocess.run(["nvdisasm", "-g", "-c", cubin], capture_output=True, text=True).stdout.split("\n")
start = [i for i, l in enumerate(dis) if kname in l and "section" in l and ".text." in l][0]
end = start + 1
while end < len(dis) and not dis[end].startswith("//--------------------- .text."):
    end += 1
cur = None
off2line = {}
for l in dis[start:end]:
    m = re.search(r'//## File "(.*?)", line (\d+)', l)
    if m:
        cur = int(m.group(2)) if m.group(1).endswith(srcfile.split("/")[-1]) else -2
        continue
    m = re.search(r"/\*([0-9a-f]{4,})\*/", l)
    if m and cur is not None:
        off2line[int(m.group(1), 16)] = cur
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[1]
data = rows[2:]
i_s = hdr.index("Warp Stall Sampling (All Samples)")
i_e = hdr.index("Instructions Executed")
reasons = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
i_r = [hdr.index(h) for h in reasons]
base = int(data[0][0], 16)
agg = collections.Counter()
agge = collections.Counter()
aggr = collections.defaultdict(collections.Counter)
tot = 0
totr = collections.Counter()
for r in data:
    a = int(r[0], 16) - base
    v = float(r[i_s] or 0)
    tot += v
    ln = off2line.get(a, -1)
    agg[ln] += v
    agge[ln] += float(r[i_e] or 0)
    for h, ix in zip(reasons, i_r):
        x = float(r[ix] or 0)
        aggr[ln][h] += x
        totr[h] += x
src = open(srcfile).read().split("\n")
print("total samples", tot)
print("by reason:", ", ".join(f"{k[6:]} {100*v/tot:.1f}%" for k, v in totr.most_common(8)))
for ln, v in agg.most_common(top):
    rs = ", ".join(f"{k[6:]} {100*x/v:.0f}%" for k, x in aggr[ln].most_common(3) if v)
    print("%5d %5.1f%% exec=%10d  %-70s | %s" % (ln, 100 * v / tot, agge[ln],
                                               src[ln - 1].strip()[:70] if ln > 0 else "?", rs))
