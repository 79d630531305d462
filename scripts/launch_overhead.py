#!/usr/bin/env python
"""Event-timed cost of one covariance / gemm-128 call: graph replay vs eager call.

usage: python scripts/launch_overhead.py [reps]
Before each timed call the stream is kept busy (256 MiB L2 flush, then a spin of
`torch.cuda._sleep`) so the host has queued the call before the start event fires:
the times below are device-side (launch latency included, host overhead excluded).
"""
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2312_13170_b200 as pb  # noqa: E402
import pbgen  # noqa: E402


def main():
    reps = int(sys.argv[1]) if len(sys.argv) > 1 else 30
    dev = torch.device("cuda", 0)

    def g(r, c, s):
        t = torch.empty(r, c, device=dev)
        pbgen.gen_device(t, s)
        return t

    n = 2048
    data, out = g(n, n, 5), torch.empty(n, n, device=dev)
    wsc = pb.workspace("covariance", (n, n), dev)
    A, B, C = g(128, 128, 1), g(128, 128, 2), g(128, 128, 3)
    wsg = pb.workspace("gemm", (128, 128, 128), dev)
    calls = {
        "covariance": lambda: pb.pb_covariance(n, n, float(n), data, out, None, ws=wsc),
        "gemm128": lambda: pb.pb_gemm(128, 128, 128, 1.5, 1.2, C, A, B, ws=wsg),
        "empty": lambda: None,
    }
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    s = torch.cuda.current_stream()
    res = {}
    for name, f in calls.items():
        for _ in range(3):
            f()
        torch.cuda.synchronize()
        cap = torch.cuda.Stream()
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph, stream=cap):
            f()
            if name == "empty":
                flush[:1].fill_(0)  # one tiny kernel: the floor of a graph replay
        for mode in ("graph", "eager"):
            if name == "empty" and mode == "eager":
                continue
            ts = []
            for _ in range(reps):
                flush.fill_(1)
                torch.cuda._sleep(200000)
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(s)
                graph.replay() if mode == "graph" else f()
                e1.record(s)
                torch.cuda.synchronize()
                ts.append(e0.elapsed_time(e1) * 1e3)
            res[f"{name}/{mode}"] = (statistics.median(ts), min(ts))
    for k, (med, mn) in res.items():
        print(f"{k:22s} median {med:7.1f} us  min {mn:7.1f} us")


if __name__ == "__main__":
    main()
