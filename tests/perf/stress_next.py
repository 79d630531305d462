#!/usr/bin/env python
"""Repeat the persistent / flag-synchronised NEXT-3 kernels many times on varied shapes and
check every run bitwise against the first (races in the release/acquire hand-offs would
show up as run-to-run differences or hangs)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2312_13170_b200 as pb  # noqa: E402
from tests import parity as P  # noqa: E402

torch.cuda.set_device(0)
reps = int(sys.argv[1]) if len(sys.argv) > 1 else 20
bad = 0
for (nx, ny, T) in ((1024, 1024, 37), (257, 516, 19), (130, 132, 9)):
    ex, ey, hz, f = P.fdtd_inputs(nx, ny, T)
    ref = None
    for r in range(reps):
        d = [P.dev(a) for a in (ex, ey, hz)]
        pb.pb_fdtd_2d(T, nx, ny, d[0], d[1], d[2], P.dev(f))
        out = [P.host(t).view(np.uint32) for t in d]
        if ref is None:
            ref = out
        elif not all(np.array_equal(a, b) for a, b in zip(out, ref)):
            bad += 1
    print("fdtd", nx, ny, T, "ok" if bad == 0 else f"MISMATCH {bad}", flush=True)
for (m, n) in ((1024, 1024), (300, 149), (2048, 2048)):
    A = P.H(m, n, 1)
    ref = None
    for r in range(max(3, reps // 4)):
        dA, dR, dQ = P.dev(A), torch.zeros(n, n, device="cuda"), torch.zeros(m, n, device="cuda")
        pb.pb_gramschmidt(m, n, dA, dR, dQ)
        out = [P.host(t).view(np.uint32) for t in (dA, dR, dQ)]
        if ref is None:
            ref = out
        elif not all(np.array_equal(a, b) for a, b in zip(out, ref)):
            bad += 1
    print("gramschmidt", m, n, "ok" if bad == 0 else f"MISMATCH {bad}", flush=True)
import pbgen  # noqa: E402
for (ni, nj, nk) in ((1024, 1024, 1024), (257, 65, 516), (9, 130, 136)):
    A = torch.empty(ni * nj, nk, device="cuda")
    pbgen.gen_device(A, 1)
    ref = None
    for r in range(max(3, reps // 4)):
        B = torch.zeros(ni * nj, nk, device="cuda")
        pb.pb_conv3d(ni, nj, nk, pbgen.conv3d_w27(), A, B)
        torch.cuda.synchronize()
        h = torch.sum(B.view(torch.int32).to(torch.int64) * torch.arange(1, B.numel() + 1, device="cuda").view_as(B) % 1000003).item()
        if ref is None:
            ref = h
        elif h != ref:
            bad += 1
    print("conv3d", ni, nj, nk, "ok" if bad == 0 else f"MISMATCH {bad}", flush=True)
print("STRESS", "PASS" if bad == 0 else "FAIL")
