"""Tuning aid: top warp-stall SASS instructions and key pipe metrics of an ncu report."""
import csv
import subprocess
import sys

rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout.splitlines()
rows = list(csv.reader(out))
hi = next(i for i, r in enumerate(rows) if "Warp Stall Sampling (All Samples)" in r)
h = rows[hi]
data = [r for r in rows[hi + 1:] if len(r) == len(h)]
i_s = h.index("Warp Stall Sampling (All Samples)")
tot = sum(float(r[i_s] or 0) for r in data) or 1.0
stall_cols = [i for i, c in enumerate(h) if c.startswith("stall_") and "Not Issued" not in c]
for r in sorted(data, key=lambda r: -float(r[i_s] or 0))[:n]:
    st = sorted(((float(r[i] or 0), h[i]) for i in stall_cols), reverse=True)[:2]
    print(r[0][-5:], f"{float(r[i_s]) / tot * 100:5.1f}%", r[1][:70], [(nm[6:], int(v)) for v, nm in st])
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout.splitlines()
rr = list(csv.reader(raw))
want = ["gpu__time_duration.sum", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
        "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum"]
for k in want:
    if k in rr[0]:
        print(k, rr[2][rr[0].index(k)] if len(rr) > 2 else rr[1][rr[0].index(k)])
