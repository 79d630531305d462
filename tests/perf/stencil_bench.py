#!/usr/bin/env python
"""Timing of the SYCL-Bench stencils (readings R19-R21)
on one B200 through the C ABI: each call captured in a CUDA graph and replayed,
CUDA events on the replay stream, L2 flushed (256 MiB write) before every replay,
median / min of `reps`. Sizes: the paper's (2D Convolution 4096,
3D Convolution and FDTD2D 1024) plus HBM-bound sizes (conv2d 16384^2). Each
configuration is first checked against the oracle on sampled rows / planes.

Roofline: conv2d/conv3d are HBM-bound, algorithmic bytes = A read
once + B's interior written once (8 B per interior point, + 4 B per border point
read... the border is not touched: 4 B per point read + 4 B per interior point
written); peak = MEASURED_PEAKS.json hbm_gbs (copy bandwidth). fdtd_2d at 1024^2
keeps its 24 MiB (state + ping-pong copy) in L2; its algorithmic traffic per step
is 3 fields read + 3 written (24 B per point); reported as us per step and GB/s
per step, against the copy bandwidth as well (an L2-resident step may exceed it).

usage: python scripts/stencil_bench.py [out.json]
"""
import json
import os
import statistics
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402  (test infrastructure: sampled parity)
import paper_2312_13170_b200 as pb  # noqa: E402
import pbgen  # noqa: E402

dev = torch.device("cuda", 0)
PEAK = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
S = pbgen.STREAM


def timed(fn, reps=20, flush=True):
    fn()
    torch.cuda.synchronize()
    st = torch.cuda.Stream()
    gr = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gr, stream=st):
        fn()
    fl = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    ts = []
    for _ in range(reps):
        if flush:
            fl.fill_(1)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        gr.replay()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return statistics.median(ts), min(ts)


def gen(shape, stream):
    t = torch.empty(*shape, device=dev)
    pbgen.gen_device(t.view(-1, shape[-1]), stream)
    return t


def conv2d(n, reps):
    A, B = gen((n, n), S["A"]), gen((n, n), S["B"])
    w = pbgen.CONV2D_W
    fn = lambda: pb.pb_conv2d(n, n, w, A, B)  # noqa: E731
    med, mn = timed(fn, reps)
    # sampled parity (rows 1, n/2, n-2)
    err = 0.0
    for i in (1, n // 2, n - 2):
        Ah = A[i - 1:i + 2].cpu().numpy()
        Bin = np.zeros_like(Ah)
        r = oracle.conv2d(w, Ah, Bin, rows=(1, 2))[0]
        s = oracle.conv2d(w, Ah, Bin, rows=(1, 2), absmode=True)[0]
        g = B[i].cpu().numpy()
        err = max(err, float(np.max(np.abs(g[1:-1] - r[1:-1]) / s[1:-1])))
    nbytes = 4 * n * n + 4 * (n - 2) * (n - 2)
    return dict(kernel="conv2d", n=n, ms=med, ms_min=mn, gbs=nbytes / med / 1e6, frac=nbytes / med / 1e6 / PEAK,
                bytes=nbytes, sampled_err=err, launches=pb.last_launch_count())


def conv3d(n, reps):
    A, B = gen((n, n, n), S["A"]), gen((n, n, n), S["B"])
    w = pbgen.conv3d_w27()
    fn = lambda: pb.pb_conv3d(n, n, n, w, A, B)  # noqa: E731
    med, mn = timed(fn, reps)
    err = 0.0
    for p in (1, n // 2, n - 2):
        Ah = A[p - 1:p + 2].cpu().numpy()
        Bin = np.zeros_like(Ah)
        r = oracle.conv3d(w, Ah, Bin, planes=(1, 2))[0]
        s = oracle.conv3d(w, Ah, Bin, planes=(1, 2), absmode=True)[0]
        g = B[p].cpu().numpy()
        err = max(err, float(np.max(np.abs(g[1:-1, 1:-1] - r[1:-1, 1:-1]) / s[1:-1, 1:-1])))
    nbytes = 4 * n ** 3 + 4 * (n - 2) ** 3
    return dict(kernel="conv3d", n=n, ms=med, ms_min=mn, gbs=nbytes / med / 1e6, frac=nbytes / med / 1e6 / PEAK,
                bytes=nbytes, sampled_err=err, launches=pb.last_launch_count())


def fdtd(n, tmax, reps):
    ex, ey, hz = gen((n, n), S["ex"]), gen((n, n), S["ey"]), gen((n, n), S["hz"])
    f = gen((1, tmax), S["fict"]).view(-1)
    ws = pb.workspace("fdtd_2d", (n, n), dev)
    keep = [t.clone() for t in (ex, ey, hz)]
    fn = lambda: pb.pb_fdtd_2d(tmax, n, n, ex, ey, hz, f, ws)  # noqa: E731
    med, mn = timed(fn, reps)
    # parity on a fresh run from the initial state: bitwise vs the fp32 oracle
    for t, k in zip((ex, ey, hz), keep):
        t.copy_(k)
    fn()
    torch.cuda.synchronize()
    r32 = oracle.fdtd2d(tmax, *(k.cpu().numpy() for k in keep), f.cpu().numpy(), f32=True)
    bitwise = all(np.array_equal(t.cpu().numpy().view(np.uint32), r.view(np.uint32)) for t, r in zip((ex, ey, hz), r32))
    step_bytes = 24 * n * n
    return dict(kernel="fdtd_2d", n=n, tmax=tmax, ms=med, ms_min=mn, us_per_step=1000 * med / tmax,
                gbs_per_step=step_bytes * tmax / med / 1e6, frac=step_bytes * tmax / med / 1e6 / PEAK,
                bitwise_f32=bitwise, launches=pb.last_launch_count())


def gramschmidt(n, reps):
    A0 = gen((n, n), S["A"])
    A = A0.clone()
    R = torch.zeros(n, n, device=dev)
    Q = torch.zeros(n, n, device=dev)
    ws = pb.workspace("gramschmidt", (n, n), dev)

    def fn():
        A.copy_(A0)  # in/out: restored inside the graph (a 4 MiB D2D copy, ~2 us)
        pb.pb_gramschmidt(n, n, A, R, Q, ws)
    med, mn = timed(fn, reps)
    flops = 2.0 * n * n * n  # sum_k (n-k-1) * 4m + 3m  ~ 2 m n^2
    return dict(kernel="gramschmidt", n=n, ms=med, ms_min=mn, us_per_step=1000 * med / n,
                gflops=flops / med / 1e6, launches=pb.last_launch_count())


def ablation():
    """The paper's question for the stencils (loop internalization did
    not apply to them): the SYCL-Bench kernel shape (variant 0: one thread per point,
    every tap a global load) against the staged march kernel, and FDTD's per-step
    launches against the persistent temporally blocked kernel (PB_FDTD_STEPS is read
    once per process, so that pair is timed by scripts/fdtd_h.py in two processes)."""
    out = []
    for n in (4096, 16384):
        A, B = gen((n, n), S["A"]), gen((n, n), S["B"])
        t0, _ = timed(lambda: pb.pb_conv2d_variant(0, n, n, pbgen.CONV2D_W, A, B), 10)
        t1, _ = timed(lambda: pb.pb_conv2d_variant(1, n, n, pbgen.CONV2D_W, A, B), 10)
        out.append(dict(kernel="conv2d", n=n, naive_ms=t0, staged_ms=t1, speedup=t0 / t1))
        del A, B
    for n in (512, 1024):
        A, B = gen((n, n, n), S["A"]), gen((n, n, n), S["B"])
        t0, _ = timed(lambda: pb.pb_conv3d_variant(0, n, n, n, pbgen.conv3d_w27(), A, B), 5)
        t1, _ = timed(lambda: pb.pb_conv3d_variant(1, n, n, n, pbgen.conv3d_w27(), A, B), 5)
        out.append(dict(kernel="conv3d", n=n, naive_ms=t0, staged_ms=t1, speedup=t0 / t1))
        del A, B
    for n in (512, 1024):
        A0 = gen((n, n), S["A"])
        A = A0.clone()
        R, Q = torch.zeros(n, n, device=dev), torch.zeros(n, n, device=dev)
        ws = pb.workspace("gramschmidt", (n, n), dev)
        res = []
        for v in (0, 1):
            def fn(v=v):
                A.copy_(A0)
                pb.pb_gramschmidt_variant(v, n, n, A, R, Q, ws)
            res.append(timed(fn, 5)[0])
        out.append(dict(kernel="gramschmidt", n=n, naive_ms=res[0], staged_ms=res[1], speedup=res[0] / res[1],
                        naive_launches=3 * n + 3))
    return out


def main():
    out = sys.argv[1] if len(sys.argv) > 1 else None
    torch.cuda.set_device(0)
    if len(sys.argv) > 2 and sys.argv[2] == "ablation":
        res = ablation()
        for r in res:
            print(json.dumps(r))
        json.dump({"ablation": res}, open(out, "w"), indent=1)
        return
    res = [conv2d(4096, 30), conv2d(16384, 20), conv3d(1024, 10), conv3d(512, 20), fdtd(1024, 500, 10),
           gramschmidt(1024, 10), gramschmidt(2048, 5)]
    for r in res:
        print(json.dumps(r))
    if out:
        json.dump({"peak_hbm_gbs": PEAK, "results": res}, open(out, "w"), indent=1)


if __name__ == "__main__":
    main()
