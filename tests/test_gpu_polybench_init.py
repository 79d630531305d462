"""GPU parity on PolyBench/C 4.2 `init_array` inputs (the
suite's own data instead of U[0,1); `pbgen.polybench_init`). Same componentwise
tolerance as the synthetic parity (R8). The covariance / correlation data have
column means up to n (the centring / cancellation case), the gramschmidt matrix is
PolyBench's (m prime keeps it full rank), FDTD is bitwise against the fp32
statements. Sizes span several tiles with ragged tails."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import oracle  # noqa: E402
import paper_2312_13170_b200 as pb  # noqa: E402
import pbgen  # noqa: E402
from tests import parity as P  # noqa: E402

TOL = P.TOL


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    torch.cuda.set_device(0)


def test_gemm_2mm_3mm():
    d = pbgen.polybench_init("gemm", 260, 132, 200)
    dC = P.dev(d["C"])
    pb.pb_gemm(260, 132, 200, d["alpha"], d["beta"], dC, P.dev(d["A"]), P.dev(d["B"]))
    r, s = (oracle.gemm(d["alpha"], d["beta"], d["C"], d["A"], d["B"], absmode=a) for a in (False, True))
    assert P.cerr(P.host(dC), r, s) <= TOL
    d = pbgen.polybench_init("2mm", 132, 200, 260, 136)
    dt, dD = torch.empty(132, 200, device="cuda"), P.dev(d["D"])
    pb.pb_2mm(132, 200, 260, 136, d["alpha"], d["beta"], dt, P.dev(d["A"]), P.dev(d["B"]), P.dev(d["C"]), dD)
    (tr, Dr), (ts, Ds) = (oracle.mm2(d["alpha"], d["beta"], d["A"], d["B"], d["C"], d["D"], absmode=a)
                          for a in (False, True))
    assert P.cerr(P.host(dD), Dr, Ds) <= TOL and P.cerr(P.host(dt), tr, ts) <= TOL
    d = pbgen.polybench_init("3mm", 132, 136, 200, 140, 260)
    dE, dF, dG = (torch.empty(*sh, device="cuda") for sh in ((132, 136), (136, 140), (132, 140)))
    pb.pb_3mm(132, 136, 200, 140, 260, dE, P.dev(d["A"]), P.dev(d["B"]), dF, P.dev(d["C"]), P.dev(d["D"]), dG)
    rr, ss = (oracle.mm3(d["A"], d["B"], d["C"], d["D"], absmode=a) for a in (False, True))
    for g, r, s in zip((dE, dF, dG), rr, ss):
        assert P.cerr(P.host(g), r, s) <= TOL


@pytest.mark.parametrize("two", [False, True])
def test_syrk_syr2k(two):
    n, m = 260, 132
    d = pbgen.polybench_init("syr2k" if two else "syrk", n, m)
    dC = P.dev(d["C"])
    if two:
        pb.pb_syr2k(n, m, d["alpha"], d["beta"], dC, P.dev(d["A"]), P.dev(d["B"]))
        r, s = (oracle.syr2k(d["alpha"], d["beta"], d["C"], d["A"], d["B"], absmode=a) for a in (False, True))
    else:
        pb.pb_syrk(n, m, d["alpha"], d["beta"], dC, P.dev(d["A"]))
        r, s = (oracle.syrk(d["alpha"], d["beta"], d["C"], d["A"], absmode=a) for a in (False, True))
    assert P.cerr(P.host(dC), r, s) <= TOL


@pytest.mark.parametrize("m,n", [(132, 260), (260, 2048), (2048, 2048), (128, 3000)])
def test_covariance_correlation(m, n):
    d = pbgen.polybench_init("covariance", m, n)
    cov, mean = torch.empty(m, m, device="cuda"), torch.empty(m, device="cuda")
    pb.pb_covariance(m, n, d["float_n"], P.dev(d["data"]), cov, mean)
    (r, rm), (s, _) = (oracle.covariance(d["float_n"], d["data"], absmode=a) for a in (False, True))
    assert P.cerr(P.host(cov), r, s) <= TOL
    d = pbgen.polybench_init("correlation", m, n)
    corr = torch.empty(m, m, device="cuda")
    pb.pb_correlation(m, n, d["float_n"], 0.1, P.dev(d["data"]), corr)
    out = oracle.correlation(d["float_n"], 0.1, d["data"])
    sc = oracle.correlation(d["float_n"], 0.1, d["data"], absmode=True)
    assert P.cerr(P.host(corr), out[0], sc[0]) <= TOL


def test_matvec_family():
    m, n = 300, 516
    d = pbgen.polybench_init("atax", m, n)
    y, t = torch.empty(n, device="cuda"), torch.empty(m, device="cuda")
    pb.pb_atax(m, n, P.dev(d["A"]), P.dev(d["x"]), y, t)
    (yr, tr), (ys, tsc) = (oracle.atax(d["A"], d["x"], absmode=a) for a in (False, True))
    assert P.cerr(P.host(y), yr, ys) <= TOL and P.cerr(P.host(t), tr, tsc) <= TOL
    d = pbgen.polybench_init("bicg", 516, 300)
    s_, q = torch.empty(516, device="cuda"), torch.empty(300, device="cuda")
    pb.pb_bicg(516, 300, P.dev(d["A"]), s_, q, P.dev(d["p"]), P.dev(d["r"]))
    (sr, qr), (ss, qs) = (oracle.bicg(d["A"], d["p"], d["r"], absmode=a) for a in (False, True))
    assert P.cerr(P.host(s_), sr, ss) <= TOL and P.cerr(P.host(q), qr, qs) <= TOL
    n = 516
    d = pbgen.polybench_init("mvt", n)
    x1, x2 = P.dev(d["x1"]), P.dev(d["x2"])
    pb.pb_mvt(n, x1, x2, P.dev(d["y_1"]), P.dev(d["y_2"]), P.dev(d["A"]))
    (r1, r2), (s1, s2) = (oracle.mvt(d["x1"], d["x2"], d["y_1"], d["y_2"], d["A"], absmode=a) for a in (False, True))
    assert P.cerr(P.host(x1), r1, s1) <= TOL and P.cerr(P.host(x2), r2, s2) <= TOL
    d = pbgen.polybench_init("gesummv", n)
    tmp, y = torch.empty(n, device="cuda"), torch.empty(n, device="cuda")
    pb.pb_gesummv(n, d["alpha"], d["beta"], P.dev(d["A"]), P.dev(d["B"]), tmp, P.dev(d["x"]), y)
    (tr, yr), (tsc, ys) = (oracle.gesummv(d["alpha"], d["beta"], d["A"], d["B"], d["x"], absmode=a)
                           for a in (False, True))
    assert P.cerr(P.host(y), yr, ys) <= TOL and P.cerr(P.host(tmp), tr, tsc) <= TOL


def test_fdtd2d_bitwise():
    T, nx, ny = 20, 130, 132
    d = pbgen.polybench_init("fdtd_2d", T, nx, ny)
    g = [P.dev(d[k]) for k in ("ex", "ey", "hz")]
    pb.pb_fdtd_2d(T, nx, ny, g[0], g[1], g[2], P.dev(d["fict"]))
    r32 = oracle.fdtd2d(T, d["ex"], d["ey"], d["hz"], d["fict"], f32=True)
    for a, b in zip(g, r32):
        assert np.array_equal(P.host(a).view(np.uint32), b.view(np.uint32))


def test_gramschmidt_polybench_matrix():
    m = n = 131  # prime: the PolyBench matrix ((i*j % m)/m)*100 + 10 is then of full rank
    d = pbgen.polybench_init("gramschmidt", m, n)
    dA, dR, dQ = P.dev(d["A"]), torch.zeros(n, n, device="cuda"), torch.zeros(m, n, device="cuda")
    pb.pb_gramschmidt(m, n, dA, dR, dQ)
    rA, rR, rQ = oracle.gramschmidt(d["A"])
    gA, gR, gQ = P.host(dA), P.host(dR), P.host(dQ)
    cn = np.sqrt((d["A"].astype(np.float64) ** 2).sum(0))
    up = np.triu(np.ones((n, n), bool))
    assert (np.abs(gQ - rQ) / np.abs(rQ).max(0)).max() <= TOL
    assert (np.abs(gA - rA) / np.abs(rA).max(0)).max() <= TOL
    assert (np.abs(gR - rR) / cn[None, :])[up].max() <= TOL


# PolyBench-GPU / SYCL-Bench constants (readings R4/R5): a fixed
# FLOAT_N = 3214212.01 that is not the observation count (so the "mean" is not the
# mean and nothing cancels) and eps = 0.005.
@pytest.mark.parametrize("m,n", [(132, 260), (2048, 2048), (128, 3000)])
@pytest.mark.parametrize("float_n", [3214212.01, None])
def test_polybench_gpu_constants(m, n, float_n):
    r = P.check_covariance(m, n, float_n=float_n)
    assert r["ok"], r
    r = P.check_correlation(m, n, eps=0.005, float_n=float_n)
    assert r["ok"], r


@pytest.mark.parametrize("m,n", [(132, 260), (256, 2048), (128, 3000)])
@pytest.mark.parametrize("eps", [0.0, 10.0])
def test_correlation_eps_extremes(m, n, eps):
    """eps = 0: only the constant column (sd = 0 <= eps) is replaced; eps = 10: every
    column's sd is replaced by 1 (reading R5), on the banded and the long-column paths."""
    r = P.check_correlation(m, n, eps=eps)
    assert r["ok"], r
