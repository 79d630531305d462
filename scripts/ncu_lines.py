#!/usr/bin/env python
"""Tuning aid: top CUDA source lines by warp-stall samples from an ncu report
(`ncu -i <rep> --page source --csv --print-source cuda,sass`), with the dominant stall reasons.
usage: python scripts/ncu_lines.py <report.ncu-rep> [file-substring] [top]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
sub = sys.argv[2] if len(sys.argv) > 2 else ""
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows, fname, hdr = [], None, None
for line in out.splitlines():
    r = next(csv.reader(io.StringIO(line)))
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or not r[0] or (sub and sub not in (fname or "")) or len(r) != len(hdr):
        continue
    try:
        s = int(r[4] or 0)
    except ValueError:
        continue
    if s:
        stalls = {hdr[k]: int(v) for k, v in enumerate(r) if hdr[k].startswith("stall_") and "Not Issued" not in hdr[k]
                  and v.isdigit() and int(v)}
        rows.append((s, fname.split("/")[-1], r[0], r[1].strip()[:80], stalls))
tot = sum(x[0] for x in rows)
rows.sort(key=lambda x: -x[0])
print(f"total samples {tot}")
for s, f, ln, src, st in rows[:top]:
    best = sorted(st.items(), key=lambda kv: -kv[1])[:3]
    print(f"{100*s/tot:5.1f}% {f}:{ln:>4} {src:80s} {' '.join(f'{k[6:]}={v}' for k, v in best)}")
