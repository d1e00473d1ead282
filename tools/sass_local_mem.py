"""Local-memory (LDL/STL) instructions of a kernel per source line, from the
SASS with line info (nvdisasm -g on the cubin inside the object file). Used to
show that the DFS hot loop (run_segment) has no local-memory traffic.
usage: python tools/sass_local_mem.py OBJ KERNEL_MANGLED [first_line last_line]"""
import collections
import os
import re
import subprocess
import sys
import tempfile

obj, kern = sys.argv[1], sys.argv[2]
lo, hi = (int(sys.argv[3]), int(sys.argv[4])) if len(sys.argv) > 4 else (0, 1 << 30)
with tempfile.TemporaryDirectory() as d:
    subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(obj)], cwd=d, check=True,
                   capture_output=True)
    cub = [f for f in os.listdir(d) if f.endswith(".cubin")][0]
    sass = subprocess.run(["nvdisasm", "-g", "-c", os.path.join(d, cub)],
                          capture_output=True, text=True).stdout
cur, cnt, total, inside = None, collections.Counter(), 0, False
for ln in sass.splitlines():
    if ln.lstrip().startswith(".section") or ln.startswith(".text."):
        inside = (".text." + kern) in ln
        continue
    if not inside:
        continue
    m = re.search(r'//## File "([^"]+)", line (\d+)', ln)
    if m:
        cur = (os.path.basename(m.group(1)), int(m.group(2)))
        continue
    if re.search(r"\b(LDL|STL)\b", ln):
        total += 1
        if cur and lo <= cur[1] <= hi:
            cnt[(cur, "LDL" if "LDL" in ln else "STL")] += 1
print(f"{kern}: {total} LDL/STL instructions in the kernel; {sum(cnt.values())} in lines "
      f"{lo}-{hi}")
for (where, op), v in sorted(cnt.items(), key=lambda x: (x[0][0] or ("", 0))[1]):
    print(f"  {where[0]}:{where[1]} {op} x{v}")
