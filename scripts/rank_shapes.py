#!/usr/bin/env python
"""Per-rank compute at G = 1/2/4/8: on one GPU, time the local
work of the slowest rank of each sharded kernel at BASELINE sizes — the same
row blocks and C-ABI calls the pb_<k>_dist entry points make, without the
exchange — and report the compute-only speedup T(1)/T(G). A proxy for strong
scaling while only one GPU is available (collectives: DESIGN.md §9).

usage: python scripts/rank_shapes.py [out.json]
"""
import json
import os
import statistics
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2312_13170_b200 as pb  # noqa: E402
import pbgen  # noqa: E402

dev = torch.device("cuda", 0)
MM, SY, MV, ST = 4096, 8192, 32768, 2048


def g(r, c, s):
    t = torch.empty(r, c, device=dev)
    pbgen.gen_device(t, s)
    return t


def timed(fn, reps=10):
    fn()
    torch.cuda.synchronize()
    st = torch.cuda.Stream()
    gr = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gr, stream=st):
        fn()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        gr.replay()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return statistics.median(ts)


def main():
    only_syrk = "--only-syrk" in sys.argv  # partition tuning: syrk / syr2k rows only
    if only_syrk:
        sys.argv.remove("--only-syrk")
    out = {}
    Amm, Bmm, Cmm, Dmm = g(MM, MM, 1), g(MM, MM, 2), g(MM, MM, 3), g(MM, MM, 4)
    Asy, Bsy = g(SY, SY, 1), g(SY, SY, 2)
    Amv = g(MV, MV, 1)
    Bmv = g(MV // 2, MV, 2)  # gesummv's B block (the largest block needed is half)
    x = g(1, MV, 6).view(-1)
    data = g(ST, ST, 5)
    for G in (1, 2, 4, 8):
        res = {}
        if only_syrk:
            for k in ("syrk", "syr2k"):
                worst = 0.0
                for gr in range(G):
                    b, e = pb.pb_row_partition(SY, G, gr, 2, 256)
                    if e <= b:
                        continue
                    Cb = torch.empty(e - b, SY, device=dev)
                    wsy = pb.workspace(k + "_rows", (SY, SY, b, e), dev)
                    if k == "syrk":
                        f = lambda: pb.pb_syrk_rows(SY, SY, b, e, 1.5, 1.2, Cb, Asy, ws=wsy)  # noqa: E731
                    else:
                        f = lambda: pb.pb_syr2k_rows(SY, SY, b, e, 1.5, 1.2, Cb, Asy, Bsy, ws=wsy)  # noqa: E731
                    worst = max(worst, timed(f, 5))
                    del Cb
                res[k] = worst
            out[G] = {k: round(v * 1e3, 1) for k, v in res.items()}
            print(G, out[G], flush=True)
            continue
        # covariance / correlation: G = 1 is the single-GPU call (banded, triangle + mirror);
        # G > 1 a rank's row band of the replicated-data path (pb_<k>_rows)
        cov, mean, sd = torch.empty(ST, ST, device=dev), torch.empty(ST, device=dev), torch.empty(ST, device=dev)
        if G == 1:
            wss = pb.workspace("covariance", (ST, ST), dev)
            res["covariance"] = timed(lambda: pb.pb_covariance(ST, ST, float(ST), data, cov, mean, ws=wss))
            res["correlation"] = timed(lambda: pb.pb_correlation(ST, ST, float(ST), 0.1, data, cov, mean, sd, ws=wss))
        else:
            # observations split (pb_<k>_dist, bench's N > 1 path): the rank's Gram of its
            # observation block, m x m full square over K = n / G (pb_syrk_full on the centred
            # transpose); the column-sum / centring / scaling kernels (~5 us) and the two
            # collectives (8 KB all-gather, 16 MiB reduce-scatter) are not included
            o0, o1 = pb.pb_row_partition(ST, G, 0, 0, 32)
            nl = (o1 - o0 + 3) // 4 * 4
            Yt = g(ST, nl, 5)
            P_ = torch.empty(ST, ST, device=dev)
            wso = pb.workspace("syrk_full", (ST, nl), dev)
            res["covariance_obs_gram"] = timed(lambda: pb.pb_syrk_full(ST, nl, 1.0, 0.0, P_, Yt, ws=wso))
            del Yt, P_
            b, e = pb.pb_row_partition(ST, G, 0, 0, 128)
            wsr = pb.workspace("covariance_rows", (ST, ST, b, e), dev)
            res["covariance"] = timed(lambda: pb.pb_covariance_rows(ST, ST, float(ST), b, e, data, cov[:e - b], mean,
                                                                    ws=wsr))
            res["correlation"] = timed(lambda: pb.pb_correlation_rows(ST, ST, float(ST), 0.1, b, e, data, cov[:e - b],
                                                                      mean, sd, ws=wsr))
        r0, r1 = pb.pb_row_partition(MM, G, 0, 0, 128)  # uniform blocks: rank 0 is representative
        rows = r1 - r0
        tmp, D2 = torch.empty(rows, MM, device=dev), Dmm[:rows].clone()
        ws = pb.workspace("2mm", (rows, MM, MM, MM), dev)
        res["2mm"] = timed(lambda: pb.pb_2mm(rows, MM, MM, MM, 1.5, 1.2, tmp, Amm[:rows], Bmm, Cmm, D2, ws=ws))
        E, F, Gm = torch.empty(rows, MM, device=dev), torch.empty(MM, MM, device=dev), torch.empty(rows, MM, device=dev)
        wsg = pb.workspace("gemm", (rows, MM, MM), dev)

        def mm3():
            pb.pb_gemm(rows, MM, MM, 1.0, 0.0, F[:rows], Cmm[:rows], Dmm, ws=wsg)  # F rows
            pb.pb_gemm(rows, MM, MM, 1.0, 0.0, E, Amm[:rows], Bmm, ws=wsg)         # E rows
            pb.pb_gemm(rows, MM, MM, 1.0, 0.0, Gm, E, F, ws=wsg)                   # G rows
        res["3mm"] = timed(mm3)
        for k in ("syrk", "syr2k"):
            worst = 0.0
            for gr in range(G):
                b, e = pb.pb_row_partition(SY, G, gr, 2, 256)
                if e <= b:
                    continue
                Cb = torch.empty(e - b, SY, device=dev)
                wsy = pb.workspace(k + "_rows", (SY, SY, b, e), dev)
                if k == "syrk":
                    f = lambda: pb.pb_syrk_rows(SY, SY, b, e, 1.5, 1.2, Cb, Asy, ws=wsy)  # noqa: E731
                else:
                    f = lambda: pb.pb_syr2k_rows(SY, SY, b, e, 1.5, 1.2, Cb, Asy, Bsy, ws=wsy)  # noqa: E731
                worst = max(worst, timed(f, 5))
                del Cb
            res[k] = worst
        b, e = pb.pb_row_partition(MV, G, 0, 0, 4)
        rows = e - b
        y, t, q = torch.empty(MV, device=dev), torch.empty(rows, device=dev), torch.empty(rows, device=dev)
        wsa = pb.workspace("atax", (rows, MV), dev)
        res["atax"] = timed(lambda: pb.pb_atax(rows, MV, Amv[:rows], x, y, t, ws=wsa))
        wsb = pb.workspace("bicg", (MV, rows), dev)
        res["bicg"] = timed(lambda: pb.pb_bicg(MV, rows, Amv[:rows], y, q, x, x[:rows], ws=wsb))
        wsm = pb.workspace("matvec_partial", (rows, MV), dev)
        res["mvt"] = timed(lambda: pb.pb_matvec_partial(rows, MV, Amv[:rows], x, q, q, x[:rows], None, y, ws=wsm))
        if rows <= Bmv.shape[0]:
            res["gesummv"] = timed(lambda: pb.pb_gesummv_rows(rows, MV, 1.5, 1.2, Amv[:rows], Bmv[:rows], None, x, t))
        out[G] = {k: round(v * 1e3, 1) for k, v in res.items()}  # us
        print(G, out[G], flush=True)
    sp = {G: {k: round(out[1][k] / v, 2) for k, v in out[G].items() if k in out[1]} for G in out if G > 1}
    print("compute-only speedup T(1)/T(G):", sp)
    if len(sys.argv) > 1:
        json.dump({"per_rank_us": out, "speedup": sp,
                   "note": "slowest rank's local calls at BASELINE sizes, no exchange; 1 B200; graph replay, warm"},
                  open(sys.argv[1], "w"), indent=1)


if __name__ == "__main__":
    main()
