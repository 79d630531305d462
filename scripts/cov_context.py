"""Tuning aid: the fused cov kernel's phase stamps and effective SM clock (PB_GRAM_TIMING=1)
in three contexts — alone, right after syr2k 8192 (tensor-bound, power-capped), and right
after gesummv 32768 (HBM-bound) — plus graph-replay call times against an empty graph.

usage: PB_GRAM_TIMING=1 python scripts/cov_context.py
"""
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2312_13170_b200 as pb  # noqa: E402
import pbgen  # noqa: E402

dev = torch.device("cuda", 0)


def g(r, c, s):
    t = torch.empty(r, c, device=dev)
    pbgen.gen_device(t, s)
    return t


n = 2048
data, out = g(n, n, 5), torch.empty(n, n, device=dev)
ws = pb.workspace("covariance", (n, n), dev)
SY = 8192
A, B, C = g(SY, SY, 1), g(SY, SY, 2), g(SY, SY, 3)
wsy = pb.workspace("syr2k", (SY, SY), dev)
MV = 32768
Am, Bm = g(MV, MV, 1), g(MV, MV, 2)
x, y, t = g(1, MV, 6).view(-1), torch.empty(MV, device=dev), torch.empty(MV, device=dev)
fl = torch.empty(256 << 20, dtype=torch.uint8, device=dev)


def cov():
    pb.pb_covariance(n, n, float(n), data, out, None, ws=ws)


def syr2k():
    pb.pb_syr2k(SY, SY, 1.5, 1.2, C, A, B, ws=wsy)


def gesummv():
    pb.pb_gesummv(MV, 1.5, 1.2, Am, Bm, t, x, y)


for name, pre in (("alone", None), ("after syr2k", syr2k), ("after gesummv", gesummv)):
    for it in range(2):
        if pre:
            pre()
        fl.fill_(1)
        print(f"== cov {name} call {it}", file=sys.stderr, flush=True)
        cov()  # the timing path synchronises and prints the stamps
        torch.cuda.synchronize()

if not os.environ.get("PB_GRAM_TIMING"):
    def replay(fn, reps=30):
        st = torch.cuda.Stream()
        fn()
        torch.cuda.synchronize()
        gr = torch.cuda.CUDAGraph()
        with torch.cuda.graph(gr, stream=st):
            fn()
        ts = []
        for _ in range(reps):
            fl.fill_(1)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            gr.replay()
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1) * 1e3)
        return statistics.median(ts)

    z = torch.zeros(4, device=dev)
    print(f"graph replay: empty-ish op {replay(lambda: z.add_(1)):.1f} us, cov {replay(cov):.1f} us", flush=True)

if not os.environ.get("PB_GRAM_TIMING"):
    # L2 flush variants before each replay: a 256 MiB write leaves ~126 MB of dirty lines
    # that the next kernel's misses must write back; a read pass after it leaves clean lines
    fr = torch.empty(64 << 20, device=dev)  # 256 MiB of fp32

    def replay2(fn, mode, reps=30):
        st = torch.cuda.Stream()
        gr = torch.cuda.CUDAGraph()
        with torch.cuda.graph(gr, stream=st):
            fn()
        ts = []
        for _ in range(reps):
            if mode >= 1:
                fl.fill_(1)
            if mode == 2:
                fr.sum()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            gr.replay()
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1) * 1e3)
        return statistics.median(ts)

    def corr():
        pb.pb_correlation(n, n, float(n), 0.1, data, out, None, None, ws=ws)

    for name, fn in (("cov", cov), ("corr", corr)):
        print(name, {m: round(replay2(fn, i), 1) for i, m in enumerate(("no flush", "write flush", "write+read flush"))},
              flush=True)
