#!/usr/bin/env python
"""Summarise ncu captures for profiles/: per-kernel key counters from
`ncu --page raw --csv` dumps, the launch-list time shares, and
profiles/traffic.json (dram bytes per launch of each bench kernel, read by
bench.py's roofline "traffic").

usage: python scripts/ncu_summary.py <round tag, e.g. r01>
  reads profiles/<tag>_<kernel>_raw.csv and profiles/<tag>_launches.csv
  writes profiles/<tag>_summary.md and updates profiles/traffic.json
"""
import collections
import csv
import glob
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
P = os.path.join(ROOT, "profiles")
KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "dram read"),
    ("dram__bytes_write.sum", "dram write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram % peak"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor pipe % active"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM % peak"),
    ("lts__t_bytes.sum", "L2 bytes"),
    ("launch__registers_per_thread", "regs/thread"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}


def raw(path):
    rows = list(csv.reader(open(path)))
    hdr, units = rows[0], rows[1]
    out = []
    for r in rows[2:]:
        d = {"name": r[hdr.index("Kernel Name")].split("(")[0]}
        for k, lab in KEYS:
            if k in hdr:
                i = hdr.index(k)
                d[k] = (r[i], units[i])
        out.append(d)
    return out


def to_bytes(v):
    val, unit = v
    return float(val.replace(",", "")) * SCALE.get(unit, 1)


def launches(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    hdr = rows[hi]
    ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    agg, cnt = collections.OrderedDict(), collections.Counter()
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        name = r[ki].split("(")[0].replace("void ", "").replace("(anonymous namespace)::", "")
        v = float(r[vi].replace(",", ""))
        v = {"ns": v / 1e3, "us": v, "ms": v * 1e3, "s": v * 1e6}.get(r[ui], v)
        agg[name] = agg.get(name, 0.0) + v
        cnt[name] += 1
    return agg, cnt


def main():
    tag = sys.argv[1] if len(sys.argv) > 1 else "r01"
    lines = [f"# ncu summary {tag}", ""]
    tj = os.path.join(P, "traffic.json")
    traffic = json.load(open(tj)) if os.path.exists(tj) else {}
    for f in sorted(glob.glob(os.path.join(P, f"{tag}_*_raw.csv"))):
        kern = os.path.basename(f)[len(tag) + 1:-len("_raw.csv")]
        for d in raw(f):
            lines.append(f"## {kern}: `{d['name']}`")
            for k, lab in KEYS:
                if k in d:
                    lines.append(f"- {lab} (`{k}`): {d[k][0]} {d[k][1]}")
            if "dram__bytes_read.sum" in d:
                traffic[kern] = int(to_bytes(d["dram__bytes_read.sum"]) + to_bytes(d["dram__bytes_write.sum"]))
                lines.append(f"- traffic (read+write): {traffic[kern] / 1e9:.3f} GB per launch")
            lines.append("")
    lf = os.path.join(P, f"{tag}_launches.csv")
    if os.path.exists(lf):
        agg, cnt = launches(lf)
        tot = sum(agg.values())
        lines += ["## launch list (ncu gpu__time_duration, cold + serialised: compare shares)", "",
                  "| kernel | launches | total us | share |", "|---|---|---|---|"]
        for k, v in sorted(agg.items(), key=lambda x: -x[1]):
            lines.append(f"| `{k}` | {cnt[k]} | {v:.1f} | {100 * v / tot:.1f}% |")
        lines.append("")
    open(os.path.join(P, f"{tag}_summary.md"), "w").write("\n".join(lines) + "\n")
    json.dump(traffic, open(tj, "w"), indent=1, sort_keys=True)
    print("\n".join(lines))


if __name__ == "__main__":
    main()
