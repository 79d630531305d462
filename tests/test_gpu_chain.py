"""NEXT-4 chain fusion (§VII-B, kernel fusion as the way
to remove launch overhead and the global-memory dataflow between kernels): 2mm's two GEMMs,
and 3mm's F, E and G, run as ONE persistent tcgen05 launch in which a GEMM's tiles of row
panel i start as soon as the GEMM it reads has published panel i (k_umma.cu `Chain`), and
the later phases' operand splits are done inside the launch by the epilogue warps.
The chained path is opt-in (PB_CHAIN=1: measured slower than separate launches, DESIGN.md
§8), so these checks run in a subprocess with it set: parity against the CPU oracle on
shapes that take the chained path (2-CTA 256x256 tiles, >= 74 tiles so the split-K remainder
units are exercised, ragged edges, K not a multiple of 256), the launch count, bitwise
run-to-run determinism, and the 4096 BASELINE size on sampled rows."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CODE = r'''
import sys
import numpy as np
import torch
sys.path.insert(0, ROOT)
import oracle
import paper_2312_13170_b200 as pb
from tests import parity as P

for dims in [(2560, 2304, 1024, 2080), (2048, 2048, 1024, 2048)]:
    r = P.check_2mm(*dims)
    assert pb.last_launch_count() == 3, ("2mm launches", pb.last_launch_count())  # A, B^T splits + the chain
    assert r["ok"], ("2mm", dims, r)
for dims in [(2560, 2304, 520, 2080, 260)]:
    r = P.check_3mm(*dims)
    assert pb.last_launch_count() == 3, ("3mm launches", pb.last_launch_count())  # C, D^T splits + the chain
    assert r["ok"], ("3mm", dims, r)
ni, nj, nk, nl = 2560, 2304, 1024, 2080
A, B, C, D = (P.dev(P.H(*sh, s)) for sh, s in (((ni, nk), 1), ((nk, nj), 2), ((nj, nl), 3), ((ni, nl), 4)))
outs = []
for _ in range(2):
    d = D.clone()
    pb.pb_2mm(ni, nj, nk, nl, 1.5, 1.2, None, A, B, C, d)
    outs.append(P.host(d))
assert np.array_equal(outs[0].view(np.uint32), outs[1].view(np.uint32)), "chain not deterministic"
# BASELINE size (4096): sampled rows of G against the oracle's rows
n = 4096
Ah, Bh, Ch, Dh = (P.H(n, n, s) for s in (1, 2, 3, 4))
E, F, G = (torch.empty(n, n, device="cuda") for _ in range(3))
pb.pb_3mm(n, n, n, n, n, E, P.dev(Ah), P.dev(Bh), F, P.dev(Ch), P.dev(Dh), G)
rows = np.random.default_rng(7).choice(n, 8, replace=False)
Fr = Ch.astype(np.float64) @ Dh.astype(np.float64)
Er = Ah[rows].astype(np.float64) @ Bh.astype(np.float64)
Gr = Er @ Fr
Gs = np.abs(Er) @ np.abs(Fr)
err = np.max(np.abs(P.host(G)[rows] - Gr) / Gs)
assert err <= P.TOL, ("3mm 4096 rows", err)
print("chain ok")
'''.replace("ROOT", repr(ROOT))


def test_chain_fusion_parity_launches_determinism():
    pytest.importorskip("torch")
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    r = subprocess.run([sys.executable, "-c", CODE], cwd=ROOT, env=dict(os.environ, PB_CHAIN="1", PYTHONPATH=ROOT),
                       capture_output=True, text=True, timeout=900)
    assert r.returncode == 0 and "chain ok" in r.stdout, r.stdout[-3000:] + r.stderr[-3000:]
