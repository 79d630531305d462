"""Tuning aid: map an ncu report's top-stalled SASS instructions to source lines.
usage: python scripts/ncu_lines.py <report.ncu-rep> <object.o> <kernel-substring> [n]"""
import csv
import re
import subprocess
import sys

rep, obj, kname = sys.argv[1], sys.argv[2], sys.argv[3]
n = int(sys.argv[4]) if len(sys.argv) > 4 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout.splitlines()
rows = list(csv.reader(out))
h = rows[1]
data = rows[2:]
i_s = h.index("Warp Stall Sampling (All Samples)")
base = min(int(r[0], 16) for r in data)
tot = sum(float(r[i_s] or 0) for r in data) or 1.0
# line info from cuobjdump (SASS with //## File ... line annotations)
import glob
import os
import tempfile
tmp = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(obj)], cwd=tmp, capture_output=True)
cubin = glob.glob(os.path.join(tmp, "*.cubin"))[0]
cub = subprocess.run(["nvdisasm", "-g", "-c", cubin], capture_output=True, text=True).stdout
cur_fn, line, off2line = None, None, {}
for l in cub.splitlines():
    m = re.match(r"^\.text\.(\S+):", l)
    if m:
        cur_fn = m.group(1)
        continue
    m = re.search(r"line (\d+)", l)
    if "//##" in l and m:
        line = int(m.group(1))
        continue
    m = re.match(r"\s*/\*([0-9a-f]{4,})\*/", l)
    if m and cur_fn and kname in cur_fn and line is not None:
        off2line[(cur_fn, int(m.group(1), 16))] = line
fns = sorted({f for f, _ in off2line})
by_line = {}
for r in data:
    off = int(r[0], 16) - base
    v = float(r[i_s] or 0)
    for f in fns:
        if (f, off) in off2line:
            ln = off2line[(f, off)]
            by_line[ln] = by_line.get(ln, 0) + v
            break
src = open(sys.argv[5]).read().splitlines() if len(sys.argv) > 5 else None
for ln, v in sorted(by_line.items(), key=lambda x: -x[1])[:n]:
    print(f"line {ln:5d} {v / tot * 100:5.1f}%", src[ln - 1].strip()[:90] if src else "")
