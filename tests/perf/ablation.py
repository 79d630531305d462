#!/usr/bin/env python
"""Paper ablation on B200: the GEMM of PAPER.md
Listing 8 (one work-item per C[i][j], k-loop over global memory, C updated in
global memory every iteration), its loop-internalised form Listing 9 (M x M
local tiles, two barriers per tile step), Listing 9 + detect-reduction
(register accumulator, Listing 5), and the production 3xTF32 tcgen05 path —
all through pb_gemm_variant at the paper's GEMM size (1024) and
larger. Every variant is checked against the CPU oracle on sampled entries.

usage: python scripts/ablation.py [out.json]
"""
import json
import os
import statistics
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402  (test infrastructure: parity of each variant)
import paper_2312_13170_b200 as pb  # noqa: E402
import pbgen  # noqa: E402

NAMES = {0: "Listing 8 (global k-loop, C in memory)", 1: "Listing 9 (loop internalization, 16x16 tiles)",
         2: "Listing 9 + detect reduction", 3: "3xTF32 tcgen05 (production)"}


def run(n, variant, reps):
    dev = torch.device("cuda", 0)
    A, B = torch.empty(n, n, device=dev), torch.empty(n, n, device=dev)
    C0 = torch.empty(n, n, device=dev)
    pbgen.gen_device(A, 1)
    pbgen.gen_device(B, 2)
    pbgen.gen_device(C0, 3)
    C = C0.clone()
    ws = pb.workspace("gemm", (n, n, n), dev)
    pb.pb_gemm_variant(variant, n, n, n, 1.5, 1.2, C, A, B, ws=ws)
    torch.cuda.synchronize()
    rng = np.random.default_rng(n + variant)
    rows, cols = rng.integers(0, n, 256), rng.integers(0, n, 256)
    Ah, Bh, Ch = (pbgen.gen_host(n, n, s) for s in (1, 2, 3))
    r = oracle.gemm_at(1.5, 1.2, Ch, Ah, Bh, rows, cols)
    g = C.cpu().numpy()[rows, cols]
    err = float(np.max(np.abs(g - r) / np.abs(r)))
    ts = []
    for _ in range(reps):
        C.copy_(C0)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        pb.pb_gemm_variant(variant, n, n, n, 1.5, 1.2, C, A, B, ws=ws)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ms = statistics.median(ts)
    return {"n": n, "variant": variant, "name": NAMES[variant], "ms": round(ms, 4),
            "gflops": round(2 * n ** 3 / ms / 1e6, 1), "max_rel_err": err}


def main():
    out = sys.argv[1] if len(sys.argv) > 1 else None
    rows = []
    for n in (1024, 2048, 4096):
        for v in (0, 1, 2, 3):
            if v == 0 and n > 2048:
                continue  # Listing 8 at 4096 takes seconds per call
            reps = 3 if v == 0 else 10
            r = run(n, v, reps)
            rows.append(r)
            print(json.dumps(r), flush=True)
    base = {r["n"]: r["ms"] for r in rows if r["variant"] == 1}
    for r in rows:
        r["speedup_vs_listing9"] = round(base[r["n"]] / r["ms"], 2) if r["n"] in base else None
    if out:
        json.dump({"device": torch.cuda.get_device_name(0), "rows": rows}, open(out, "w"), indent=1)


if __name__ == "__main__":
    main()
