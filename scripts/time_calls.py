#!/usr/bin/env python
"""Quick device timing of single C-ABI calls (tuning aid; not the bench).

usage: python scripts/time_calls.py <kernel> [n] [reps]
Prints the median CUDA-event time of the call (captured into a CUDA graph so
host overhead is excluded). Env PB_UMMA_TILE / PB_UMMA_KSPLIT steer the GEMM
plan; PB_FLUSH=1 writes a 256 MB buffer before each replay (cold L2).
"""
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2312_13170_b200 as pb  # noqa: E402
import pbgen  # noqa: E402


def main():
    k = sys.argv[1]
    shape = sys.argv[2] if len(sys.argv) > 2 else "2048"
    dims = [int(v) for v in shape.split("x")]  # gemm/2mm also take MxNxK (2mm: rows x n)
    n = dims[0] if len(dims) == 1 else dims[-1]
    reps = int(sys.argv[3]) if len(sys.argv) > 3 else 20
    dev = torch.device("cuda", 0)

    def g(r, c, s):
        t = torch.empty(r, c, device=dev)
        pbgen.gen_device(t, s)
        return t

    if k in ("covariance", "correlation"):
        data, out = g(n, n, 5), torch.empty(n, n, device=dev)
        ws = pb.workspace(k, (n, n), dev)
        f = (lambda: pb.pb_covariance(n, n, float(n), data, out, None, ws=ws)) if k == "covariance" else \
            (lambda: pb.pb_correlation(n, n, float(n), 0.1, data, out, None, None, ws=ws))
        flops = n * n * (n + 1)
    elif k == "gemm":
        M, N, K = dims if len(dims) == 3 else (n, n, n)
        A, B, C = g(M, K, 1), g(K, N, 2), g(M, N, 3)
        ws = pb.workspace("gemm", (M, N, K), dev)
        f = lambda: pb.pb_gemm(M, N, K, 1.5, 1.2, C, A, B, ws=ws)  # noqa: E731
        flops = 2 * M * N * K
    elif k == "2mm":
        r = dims[0] if len(dims) == 2 else n  # 2mm on a row block: rows x n
        A, B, C, Dm, tmp = g(r, n, 1), g(n, n, 2), g(n, n, 3), g(r, n, 4), torch.empty(r, n, device=dev)
        ws = pb.workspace("2mm", (r, n, n, n), dev)
        f = lambda: pb.pb_2mm(r, n, n, n, 1.5, 1.2, tmp, A, B, C, Dm, ws=ws)  # noqa: E731
        flops = 4 * r * n * n
    elif k == "3mm":
        A, B, C, Dm = g(n, n, 1), g(n, n, 2), g(n, n, 3), g(n, n, 4)
        E, F, Gm = (torch.empty(n, n, device=dev) for _ in range(3))
        ws = pb.workspace("3mm", (n, n, n, n, n), dev)
        f = lambda: pb.pb_3mm(n, n, n, n, n, E, A, B, F, C, Dm, Gm, ws=ws)  # noqa: E731
        flops = 6 * n * n * n
    elif k == "syrk":
        A, C = g(n, n, 1), g(n, n, 3)
        ws = pb.workspace("syrk", (n, n), dev)
        f = lambda: pb.pb_syrk(n, n, 1.5, 1.2, C, A, ws=ws)  # noqa: E731
        flops = n * (n + 1) * n
    elif k == "syr2k":
        A, B, C = g(n, n, 1), g(n, n, 2), g(n, n, 3)
        ws = pb.workspace("syr2k", (n, n), dev)
        f = lambda: pb.pb_syr2k(n, n, 1.5, 1.2, C, A, B, ws=ws)  # noqa: E731
        flops = 2 * n * (n + 1) * n
    elif k == "atax":
        A, x, y = g(n, n, 1), g(1, n, 6).view(-1), torch.empty(n, device=dev)
        ws = pb.workspace("atax", (n, n), dev)
        f = lambda: pb.pb_atax(n, n, A, x, y, None, ws=ws)  # noqa: E731
        flops = 4 * n * n  # prints "TFLOP/s" = 1e3 GB/s of A (4 bytes per element)
    else:
        raise SystemExit(f"unknown kernel {k}")
    for _ in range(3):
        f()
    torch.cuda.synchronize()
    s = torch.cuda.Stream()
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph, stream=s):
        f()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev) if os.environ.get("PB_FLUSH") else None
    flush_rd = torch.zeros(64 << 20, device=dev) if flush is not None else None
    ts = []
    for _ in range(reps):
        if flush is not None:
            flush.fill_(1)  # evict the inputs from the 126 MB L2 (cold-input timing) ...
            flush_rd.sum()  # ... and leave it clean (the dirty lines are written back here)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        graph.replay()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ms = statistics.median(ts)
    print(f"{k} n={n} tile={os.environ.get('PB_UMMA_TILE', '-')} ks={os.environ.get('PB_UMMA_KSPLIT', '-')}: "
          f"{ms * 1e3:.1f} us  {flops / ms / 1e9:.1f} TFLOP/s useful")


if __name__ == "__main__":
    main()
