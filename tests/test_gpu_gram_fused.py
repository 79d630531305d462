"""The one-launch covariance / correlation path (csrc/k_gram.cu: band statistics +
centred split + 3xTF32 Gram + split-K exchange + epilogue in a single persistent
kernel; DESIGN.md §8 "cov/corr"). Parity against the CPU oracle on shapes that
exercise each split-K factor (S = 1, 2, 4), ragged variable counts (partial tiles,
a missing last slab), ragged observation counts (short last band), the diagonal and
off-diagonal (TMA-store) epilogues, plus launch count and run-to-run determinism.
The three-launch path (PB_GRAM_FUSED=0) is run in a subprocess on the same inputs
and must agree within the parity tolerance."""
import os
import subprocess
import sys

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2312_13170_b200 as pb  # noqa: E402
from tests import parity as P  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

# (m, n): T = tiles of 256 in the lower triangle; S = split-K chosen for <= 74 SM pairs
SHAPES = [
    (132, 137),    # T = 1, n < 256 (S = 1)
    (256, 2048),   # T = 1, 8 bands (S = 4)
    (1024, 1024),  # T = 10 (S = 4)
    (1028, 1000),  # T = 15, ragged m and n (S = 4)
    (1540, 777),   # T = 21 (S = 2), ragged
    (2048, 2048),  # T = 36 (S = 2): the BASELINE config
    (1800, 256),   # T = 28, one band, last CTA row slab beyond m
]


@pytest.mark.parametrize("m,n", SHAPES)
def test_fused_covariance(m, n):
    r = P.check_covariance(m, n)
    assert r["ok"], r


@pytest.mark.parametrize("m,n", SHAPES)
def test_fused_correlation(m, n):
    r = P.check_correlation(m, n)
    assert r["ok"], r


def test_fused_is_one_launch_and_deterministic():
    m = n = 2048
    data = P.dev(P.structured_data(n, m))
    outs = []
    for _ in range(2):
        c = torch.empty(m, m, device="cuda")
        pb.pb_correlation(m, n, float(n), 0.1, data, c, None, None)
        assert pb.last_launch_count() == 2  # flag zeroing + the fused kernel
        outs.append(P.host(c))
        c2 = torch.empty(m, m, device="cuda")
        pb.pb_covariance(m, n, float(n), data, c2, None)
        assert pb.last_launch_count() == 2  # flag zeroing + the fused kernel
        outs.append(P.host(c2))
    assert np.array_equal(outs[0].view(np.uint32), outs[2].view(np.uint32))
    assert np.array_equal(outs[1].view(np.uint32), outs[3].view(np.uint32))


def test_fused_matches_three_launch_path():
    """Same inputs through PB_GRAM_FUSED=0 (band prep + Gram + combine kernels)."""
    m, n = 1028, 1000
    code = ("import sys, json, numpy as np, torch; sys.path.insert(0, %r);"
            "import paper_2312_13170_b200 as pb; from tests import parity as P;"
            "d = P.dev(P.structured_data(%d, %d)); c = torch.empty(%d, %d, device='cuda');"
            "k = torch.empty(%d, %d, device='cuda');"
            "pb.pb_covariance(%d, %d, float(%d), d, c, None); pb.pb_correlation(%d, %d, float(%d), 0.1, d, k, None, None);"
            "L = pb.last_launch_count(); np.save(sys.argv[1], np.stack([P.host(c), P.host(k)])); print(L)"
            % (ROOT, n, m, m, m, m, m, m, n, n, m, n, n))
    outs, launches = [], []
    for fused in ("1", "0"):
        path = f"/tmp/pb_gram_{fused}_{os.getpid()}.npy"
        env = dict(os.environ, PB_GRAM_FUSED=fused, PYTHONPATH=ROOT)
        r = subprocess.run([sys.executable, "-c", code, path], env=env, capture_output=True, text=True, cwd=ROOT,
                           timeout=300)
        assert r.returncode == 0, r.stderr[-2000:]
        launches.append(int(r.stdout.strip().splitlines()[-1]))
        outs.append(np.load(path))
        os.unlink(path)
    assert launches[0] == 2 and launches[1] == 3, launches
    a, b = outs
    scale = np.maximum(np.abs(b), 1e-3)
    assert np.max(np.abs(a - b) / scale) <= 2e-4


@pytest.mark.parametrize("offset", [1000.0, -3.5e4])
def test_fused_large_offset(offset):
    """Columns whose mean dwarfs their spread (x = offset + U[0,1)): the band shifts (R18)
    keep the Gram operand centred, so the componentwise gate still holds."""
    import oracle
    m, n = 516, 1000
    data = P.H(n, m, P.S["data"], offset=offset)
    fn = float(n)
    d = P.dev(data)
    cov, corr = torch.empty(m, m, device="cuda"), torch.empty(m, m, device="cuda")
    mean, sd = torch.empty(m, device="cuda"), torch.empty(m, device="cuda")
    pb.pb_covariance(m, n, fn, d, cov, mean)
    assert pb.last_launch_count() == 2  # flag zeroing + the fused kernel
    pb.pb_correlation(m, n, fn, 0.1, d, corr, None, sd)
    c_r, mean_r = oracle.covariance(fn, data)
    c_s, mean_s = oracle.covariance(fn, data, absmode=True)
    k_r, _, sd_r = oracle.correlation(fn, 0.1, data)
    k_s, _, _ = oracle.correlation(fn, 0.1, data, absmode=True)
    errs = dict(cov=P.cerr(P.host(cov), c_r, c_s), mean=P.cerr(P.host(mean), mean_r, mean_s),
                corr=P.cerr(P.host(corr), k_r, k_s), sd=P.cerr(P.host(sd), sd_r, sd_r))
    assert max(errs.values()) <= P.TOL, errs
