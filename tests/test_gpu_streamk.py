"""Stream-K schedule of the tcgen05 GEMM engine (k_umma.cu `UnitIter`, opt-in with
PB_STREAMK=1; measured slower than the data-parallel plan on B200): shapes with
at most two partial waves of 256 x 256 tiles (a rank's block of 2mm at 8 GPUs, narrow row
bands of syr2k, small GEMMs) give every SM pair an equal share of the (tile, k-block)
iterations; a tile shared by several pairs is summed by the last arriver in segment order.
Run in a subprocess with PB_STREAMK=1: parity against the CPU oracle (ragged edges, segments
that start mid-tile and cross tile boundaries, syr2k's two operand pairs along K), bitwise
run-to-run determinism; and the default (data-parallel) plan agrees within 1e-5."""
import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CODE = r'''
import sys
import numpy as np
sys.path.insert(0, ROOT)
import paper_2312_13170_b200 as pb
from tests import parity as P
for dims in [(512, 4096, 4096), (700, 1000, 2000), (256, 2304, 3000), (1028, 1540, 1200)]:
    r = P.check_gemm(*dims)
    assert r["ok"], ("gemm", dims, r["err"])
for dims in [(512, 4096, 4096, 4096), (600, 1028, 2000, 1540)]:
    r = P.check_2mm(*dims)
    assert r["ok"], ("2mm", dims, r)
for n, m in [(1100, 3000), (760, 2052)]:
    r = P.check_syr2k(n, m)
    assert r["ok"], ("syr2k", n, m, r)
ni, nj, nk = 512, 4096, 4096
A, B, C = P.H(ni, nk, 1), P.H(nk, nj, 2), P.H(ni, nj, 3)
outs = []
for _ in range(2):
    dC = P.dev(C)
    pb.pb_gemm(ni, nj, nk, 1.5, 1.2, dC, P.dev(A), P.dev(B))
    outs.append(P.host(dC))
assert np.array_equal(outs[0].view(np.uint32), outs[1].view(np.uint32)), "stream-K not deterministic"
np.save(sys.argv[1], outs[0])
print("streamk ok")
'''.replace("ROOT", repr(ROOT))


def test_streamk_parity_determinism_and_default_plan_agree():
    pytest.importorskip("torch")
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    path = f"/tmp/pb_sk_{os.getpid()}.npy"
    r = subprocess.run([sys.executable, "-c", CODE, path], cwd=ROOT, env=dict(os.environ, PB_STREAMK="1"),
                       capture_output=True, text=True, timeout=900)
    assert r.returncode == 0 and "streamk ok" in r.stdout, r.stdout[-3000:] + r.stderr[-3000:]
    sk = np.load(path)
    os.unlink(path)
    sys.path.insert(0, ROOT)
    import paper_2312_13170_b200 as pb
    from tests import parity as P
    ni, nj, nk = 512, 4096, 4096
    A, B, C = P.H(ni, nk, 1), P.H(nk, nj, 2), P.H(ni, nj, 3)
    dC = P.dev(C)
    pb.pb_gemm(ni, nj, nk, 1.5, 1.2, dC, P.dev(A), P.dev(B))
    dp = P.host(dC)
    assert np.max(np.abs(dp - sk) / np.abs(dp)) <= 1e-5
