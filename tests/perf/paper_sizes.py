#!/usr/bin/env python
"""Secondary context sweep: every kernel at the paper's own
problem sizes (PAPER.md:524 — 1024 for gemm/2mm/3mm/syrk/syr2k/covariance/
correlation, 4096 for atax, 16384 for bicg/mvt/gesummv), one GPU, timed as a
CUDA-graph replay with CUDA events (median of 20, L2 flushed before each
replay) and checked against the oracle on sampled outputs. Not gated: context
for the paper's Intel-GPU speedups (other hardware).

usage: python scripts/paper_sizes.py [out.json]
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

A1, B1 = 1.5, 1.2
dev = torch.device("cuda", 0)


def g(r, c, s):
    t = torch.empty(r, c, device=dev)
    pbgen.gen_device(t, s)
    return t


def h(r, c, s):
    return pbgen.gen_host(r, c, s)


def timed(fn, reps=20):
    fn()
    torch.cuda.synchronize()
    st = torch.cuda.Stream()
    gr = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gr, stream=st):
        fn()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    ts = []
    for _ in range(reps):
        flush.fill_(1)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        gr.replay()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return statistics.median(ts)


def rel(got, ref):
    return float(np.max(np.abs(got - ref) / np.maximum(np.abs(ref), 1e-30)))


def main():
    out = []
    n = 1024
    Ah, Bh, Ch, Dh = h(n, n, 1), h(n, n, 2), h(n, n, 3), h(n, n, 4)
    # gemm
    A, B, C = g(n, n, 1), g(n, n, 2), g(n, n, 3)
    C0 = C.clone()
    ws = pb.workspace("gemm", (n, n, n), dev)
    ms = timed(lambda: pb.pb_gemm(n, n, n, A1, B1, C, A, B, ws=ws))
    C.copy_(C0)
    pb.pb_gemm(n, n, n, A1, B1, C, A, B, ws=ws)
    out.append(("gemm", n, ms, 2 * n ** 3, rel(C.cpu().numpy(), oracle.gemm(A1, B1, Ch, Ah, Bh))))
    # 2mm / 3mm
    Dm = g(n, n, 4)
    tmp = torch.empty(n, n, device=dev)
    D0 = Dm.clone()
    ws = pb.workspace("2mm", (n,) * 4, dev)
    ms = timed(lambda: pb.pb_2mm(n, n, n, n, A1, B1, tmp, A, B, C0, Dm, ws=ws))
    Dm.copy_(D0)
    pb.pb_2mm(n, n, n, n, A1, B1, tmp, A, B, C0, Dm, ws=ws)
    out.append(("2mm", n, ms, 4 * n ** 3, rel(Dm.cpu().numpy(), oracle.mm2(A1, B1, Ah, Bh, Ch, Dh)[1])))
    E, F, G = (torch.empty(n, n, device=dev) for _ in range(3))
    ws = pb.workspace("3mm", (n,) * 5, dev)
    ms = timed(lambda: pb.pb_3mm(n, n, n, n, n, E, A, B, F, C0, D0, G, ws=ws))
    out.append(("3mm", n, ms, 6 * n ** 3, rel(G.cpu().numpy(), oracle.mm3(Ah, Bh, Ch, Dh)[2])))
    # syrk / syr2k (lower triangle)
    Csh = pbgen.gen_host(n, n, 3, mode=pbgen.U01 | pbgen.SYM)
    Cs = torch.from_numpy(Csh).to(dev)
    Cs0 = Cs.clone()
    ws = pb.workspace("syr2k", (n, n), dev)
    lo = np.tril(np.ones((n, n), bool))
    for name, two in (("syrk", False), ("syr2k", True)):
        f = (lambda: pb.pb_syr2k(n, n, A1, B1, Cs, A, B, ws=ws)) if two else \
            (lambda: pb.pb_syrk(n, n, A1, B1, Cs, A, ws=ws))
        ms = timed(f)
        Cs.copy_(Cs0)
        f()
        ref = oracle.syr2k(A1, B1, Csh, Ah, Bh) if two else oracle.syrk(A1, B1, Csh, Ah)
        out.append((name, n, ms, (2 if two else 1) * n * (n + 1) * n, rel(Cs.cpu().numpy()[lo], ref[lo])))
    # covariance / correlation
    data = g(n, n, 5)
    cov = torch.empty(n, n, device=dev)
    ws = pb.workspace("correlation", (n, n), dev)
    dh = h(n, n, 5)
    for name in ("covariance", "correlation"):
        if name == "covariance":
            f = lambda: pb.pb_covariance(n, n, float(n), data, cov, None, ws=ws)  # noqa: E731
            r, sc = oracle.covariance(float(n), dh)[0], oracle.covariance(float(n), dh, absmode=True)[0]
        else:
            f = lambda: pb.pb_correlation(n, n, float(n), 0.1, data, cov, None, None, ws=ws)  # noqa: E731
            r, sc = oracle.correlation(float(n), 0.1, dh)[0], oracle.correlation(float(n), 0.1, dh, absmode=True)[0]
        ms = timed(f)
        f()
        got = cov.cpu().numpy()
        out.append((name, n, ms, n * n * (n + 1), float(np.max(np.abs(got - r) / sc))))
    # matvec family
    for name, nv in (("atax", 4096), ("bicg", 16384), ("mvt", 16384), ("gesummv", 16384)):
        Av = g(nv, nv, 1)
        x, r_, y = g(1, nv, 6).view(-1), g(1, nv, 7).view(-1), torch.empty(nv, device=dev)
        q = torch.empty(nv, device=dev)
        Ah, xh, rh = h(nv, nv, 1), h(1, nv, 6)[0], h(1, nv, 7)[0]
        if name == "atax":
            ws = pb.workspace("atax", (nv, nv), dev)
            f = lambda: pb.pb_atax(nv, nv, Av, x, y, None, ws=ws)  # noqa: E731
            ref, got = oracle.atax(Ah, xh)[0], lambda: y  # noqa: E731
            byt = 4 * nv * nv
        elif name == "bicg":
            ws = pb.workspace("bicg", (nv, nv), dev)
            f = lambda: pb.pb_bicg(nv, nv, Av, y, q, x, r_, ws=ws)  # noqa: E731
            ref, got = oracle.bicg(Ah, xh, rh)[0], lambda: y  # noqa: E731
            byt = 4 * nv * nv
        elif name == "mvt":
            x1, x2 = g(1, nv, 8).view(-1), g(1, nv, 9).view(-1)
            x20 = x2.clone()
            ws = pb.workspace("mvt", (nv,), dev)
            f = lambda: pb.pb_mvt(nv, x1, x2, x, r_, Av, ws=ws)  # noqa: E731
            byt = 4 * nv * nv
        else:
            Bv = g(nv, nv, 2)
            ws = pb.workspace("gesummv", (nv,), dev)
            f = lambda: pb.pb_gesummv(nv, A1, B1, Av, Bv, None, x, y, ws=ws)  # noqa: E731
            ref, got = oracle.gesummv(A1, B1, Ah, h(nv, nv, 2), xh)[1], lambda: y  # noqa: E731
            byt = 8 * nv * nv
        ms = timed(f)
        if name == "mvt":
            x2.copy_(x20)
            pb.pb_mvt(nv, x1, x2, x, r_, Av, ws=ws)
            ref = oracle.mvt(h(1, nv, 8)[0], h(1, nv, 9)[0], xh, rh, Ah)[1]
            e = rel(x2.cpu().numpy(), ref)
        else:
            f()
            e = rel(got().cpu().numpy(), ref)
        out.append((name, nv, ms, byt, e))
    rows_out = []
    for name, size, ms, work, err in out:
        d = {"kernel": name, "n": size, "us": round(ms * 1e3, 1), "max_rel_err": err}
        if name in ("atax", "bicg", "mvt", "gesummv"):
            d["GB_s"] = round(work / ms / 1e6, 1)
        else:
            d["TFLOP_s"] = round(work / ms / 1e9, 2)
        rows_out.append(d)
        print(json.dumps(d), flush=True)
    if len(sys.argv) > 1:
        json.dump({"device": torch.cuda.get_device_name(0), "note": "paper sizes (PAPER.md:524); L2 flushed",
                   "rows": rows_out}, open(sys.argv[1], "w"), indent=1)


if __name__ == "__main__":
    main()
