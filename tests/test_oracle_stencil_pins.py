"""Pins for the stencil oracles (2DConvolution, 3DConvolution,
FDTD2D — PAPER.md:524 §VIII lists them; readings R19-R21 in DESIGN.md).

Each oracle function is pinned to something other than itself:
  * conv2d / conv3d: scipy's correlate (textbook library routine), exact shift /
    delta / constant closed forms, border preservation, hand-worked golden values
    (tests/golden/conv2d_3x4.json, conv3d_3x3x3.json — the latter built from the
    PolyBench-GPU 15-term source list, so the 27-tap reading R20 is pinned too).
  * gramschmidt (R22): LAPACK Householder QR via numpy (sign-normalised), Q^T Q = I,
    Q R = A, the final A = Q diag(R), and exact closed forms (upper-triangular input
    -> Q = I, R = A; orthogonal columns -> signed permutation / |D|).
  * fdtd2d: hand-worked single steps (tests/golden/fdtd2d_impulse.json), exact
    telescoping sums of each sweep, the light cone of an impulse (a wrong index
    moves the support), exact linearity under scaling by 2, and the fp32 twin
    against the fp64 state.
"""
import json
import os

import numpy as np
import pytest
from scipy import ndimage, signal

import oracle

HERE = os.path.dirname(os.path.abspath(__file__))
RNG = np.random.default_rng(2312)

PB_GPU_W2 = np.array([[0.2, 0.5, -0.8], [-0.3, 0.6, -0.9], [0.4, 0.7, 0.1]])


def _rand(*shape, lo=0.0, hi=1.0):
    return RNG.uniform(lo, hi, size=shape).astype(np.float32)


# ------------------------------------------------------------------ conv2d
def test_conv2d_golden_hand_worked():
    g = json.load(open(os.path.join(HERE, "golden", "conv2d_3x4.json")))
    A = np.array(g["A"], np.float32)
    out = oracle.conv2d(g["w"], A, np.zeros_like(A))
    np.testing.assert_allclose(out[1:-1, 1:-1], g["interior_expected"], rtol=0, atol=1e-12)
    assert np.all(out[0] == 0) and np.all(out[-1] == 0) and np.all(out[:, 0] == 0) and np.all(out[:, -1] == 0)


@pytest.mark.parametrize("shape", [(3, 3), (7, 12), (33, 65)])
def test_conv2d_matches_scipy_correlate2d(shape):
    A = _rand(*shape, lo=-1, hi=1)
    B = _rand(*shape)
    w = RNG.normal(size=(3, 3))
    out = oracle.conv2d(w, A, B)
    ref = signal.correlate2d(A.astype(np.float64), w, mode="valid")
    np.testing.assert_allclose(out[1:-1, 1:-1], ref, rtol=1e-13, atol=1e-13)
    # borders keep B_in bitwise
    m = np.ones(shape, bool)
    m[1:-1, 1:-1] = False
    assert np.array_equal(out[m], B.astype(np.float64)[m])
    # absmode = the same correlation of |A| with |w|
    s = oracle.conv2d(w, A, B, absmode=True)
    np.testing.assert_allclose(s[1:-1, 1:-1], signal.correlate2d(np.abs(A.astype(np.float64)), np.abs(w), mode="valid"),
                               rtol=1e-13)


@pytest.mark.parametrize("di,dj", [(-1, -1), (-1, 1), (0, 1), (1, 0), (1, -1)])
def test_conv2d_shift_exact(di, dj):
    A = _rand(9, 10)
    w = np.zeros((3, 3))
    w[di + 1, dj + 1] = 1.0
    out = oracle.conv2d(w, A, np.zeros_like(A))
    assert np.array_equal(out[1:-1, 1:-1], A[1 + di:9 - 1 + di, 1 + dj:10 - 1 + dj].astype(np.float64))


def test_conv2d_constant_and_row_range():
    A = np.full((6, 8), 0.75, np.float32)
    out = oracle.conv2d(PB_GPU_W2, A, np.zeros_like(A))
    np.testing.assert_allclose(out[1:-1, 1:-1], 0.75 * PB_GPU_W2.sum(), rtol=1e-15)
    A = _rand(17, 12)
    B = _rand(17, 12)
    full = oracle.conv2d(PB_GPU_W2, A, B)
    assert np.array_equal(oracle.conv2d(PB_GPU_W2, A, B, rows=(5, 11)), full[5:11])


# ------------------------------------------------------------------ conv3d
def _pbgpu_w27(terms):
    w = np.zeros((3, 3, 3))
    for c, di, dj, dk in terms:
        w[di + 1, dj + 1, dk + 1] += c
    return w


def test_conv3d_golden_polybench_gpu_terms():
    g = json.load(open(os.path.join(HERE, "golden", "conv3d_3x3x3.json")))
    i, j, k = np.meshgrid(np.arange(3), np.arange(3), np.arange(3), indexing="ij")
    A = (9 * i + 3 * j + k).astype(np.float32)
    out = oracle.conv3d(_pbgpu_w27(g["terms"]), A, np.zeros_like(A))
    assert out[1, 1, 1] == g["expected_center"]
    out[1, 1, 1] = 0
    assert np.all(out == 0)


@pytest.mark.parametrize("shape", [(3, 3, 3), (5, 7, 9), (12, 10, 16)])
def test_conv3d_matches_scipy(shape):
    A = _rand(*shape, lo=-1, hi=1)
    B = _rand(*shape)
    w = RNG.normal(size=(3, 3, 3))
    out = oracle.conv3d(w, A, B)
    ref = signal.correlate(A.astype(np.float64), w, mode="valid")
    np.testing.assert_allclose(out[1:-1, 1:-1, 1:-1], ref, rtol=1e-12, atol=1e-13)
    # and scipy.ndimage (a second, independent routine) on the interior
    ref2 = ndimage.correlate(A.astype(np.float64), w, mode="constant")[1:-1, 1:-1, 1:-1]
    np.testing.assert_allclose(out[1:-1, 1:-1, 1:-1], ref2, rtol=1e-12, atol=1e-13)
    m = np.ones(shape, bool)
    m[1:-1, 1:-1, 1:-1] = False
    assert np.array_equal(out[m], B.astype(np.float64)[m])
    part = oracle.conv3d(w, A, B, planes=(1, shape[0] - 1))
    assert np.array_equal(part, out[1:-1])


def test_conv3d_shift_and_constant():
    A = _rand(6, 7, 8)
    for d in [(-1, 0, 1), (1, 1, -1), (0, -1, 0)]:
        w = np.zeros((3, 3, 3))
        w[d[0] + 1, d[1] + 1, d[2] + 1] = 1
        out = oracle.conv3d(w, A, np.zeros_like(A))
        ref = A[1 + d[0]:5 + d[0], 1 + d[1]:6 + d[1], 1 + d[2]:7 + d[2]]
        assert np.array_equal(out[1:-1, 1:-1, 1:-1], ref.astype(np.float64))
    C = np.full((4, 5, 6), 0.5, np.float32)
    w = RNG.integers(-8, 9, size=(3, 3, 3)).astype(np.float64)
    out = oracle.conv3d(w, C, np.zeros_like(C))
    assert np.all(out[1:-1, 1:-1, 1:-1] == 0.5 * w.sum())


# ------------------------------------------------------------------ fdtd2d
def test_fdtd2d_golden_impulse_and_source():
    g = json.load(open(os.path.join(HERE, "golden", "fdtd2d_impulse.json")))
    c = g["impulse"]
    z = np.zeros((c["nx"], c["ny"]), np.float32)
    hz = z.copy()
    hz[tuple(c["hz_at"])] = 1.0
    for f32 in (False, True):
        ex, ey, h = oracle.fdtd2d(1, z, z, hz, np.array(c["fict"], np.float32), f32=f32)
        for arr, key in ((ey, "ey_nonzero"), (ex, "ex_nonzero"), (h, "hz_nonzero")):
            ref = np.zeros_like(arr, dtype=np.float64)
            for i, j, v in c[key]:
                ref[i, j] = v
            np.testing.assert_allclose(arr, ref, rtol=0, atol=1e-7 if f32 else 1e-15)
    c = g["source_case"]
    z = np.zeros((c["nx"], c["ny"]), np.float32)
    ex, ey, h = oracle.fdtd2d(1, z, z, z, np.array(c["fict"], np.float32))
    np.testing.assert_allclose(ey[0], c["ey_row0"], atol=1e-15)
    np.testing.assert_allclose(h[0], c["hz_row0"], atol=1e-15)
    assert np.all(ex == 0) and np.all(ey[1:] == 0) and np.all(h[1:] == 0)


def test_fdtd2d_zero_steps_and_linearity():
    ex, ey, hz = _rand(9, 11), _rand(9, 11), _rand(9, 11)
    f = _rand(6)
    r0 = oracle.fdtd2d(0, ex, ey, hz, f)
    for a, b in zip(r0, (ex, ey, hz)):
        assert np.array_equal(a, b.astype(np.float64))
    r1 = oracle.fdtd2d(6, ex, ey, hz, f)
    r2 = oracle.fdtd2d(6, 2 * ex, 2 * ey, 2 * hz, 2 * f)  # scaling by 2 is exact in fp64
    for a, b in zip(r1, r2):
        assert np.array_equal(2 * a, b)


def test_fdtd2d_telescoping_sums_one_step():
    """One step, each sweep's change sums (exactly, in rationals) to boundary terms:
    sum_{i>=1} dey[i][j] = -0.5 (hz[nx-1][j] - hz[0][j]) for every column j;
    sum_{j>=1} dex[i][j] = -0.5 (hz[i][ny-1] - hz[i][0]) for every row i;
    sum_{i<nx-1, j<ny-1} dhz = -0.7 (sum_i (ex'[i][ny-1]-ex'[i][0]) + sum_j (ey'[nx-1][j]-ey'[0][j]))
    (the last two sums over i < nx-1, j < ny-1)."""
    nx, ny = 13, 10
    ex, ey, hz = _rand(nx, ny, lo=-1, hi=1), _rand(nx, ny, lo=-1, hi=1), _rand(nx, ny, lo=-1, hi=1)
    f = np.array([0.25], np.float32)
    ex1, ey1, hz1 = oracle.fdtd2d(1, ex, ey, hz, f)
    E, Y, Hh = (a.astype(np.float64) for a in (ex, ey, hz))
    np.testing.assert_allclose((ey1[1:] - Y[1:]).sum(0), -0.5 * (Hh[nx - 1] - Hh[0]), atol=1e-13)
    np.testing.assert_allclose(ey1[0], 0.25, rtol=0, atol=0)
    np.testing.assert_allclose((ex1[:, 1:] - E[:, 1:]).sum(1), -0.5 * (Hh[:, ny - 1] - Hh[:, 0]), atol=1e-13)
    dh = (hz1 - Hh)[: nx - 1, : ny - 1].sum()
    rhs = -0.7 * ((ex1[: nx - 1, ny - 1] - ex1[: nx - 1, 0]).sum() + (ey1[nx - 1, : ny - 1] - ey1[0, : ny - 1]).sum())
    assert abs(dh - rhs) < 1e-12
    # entries outside the hz sweep are untouched
    assert np.array_equal(hz1[nx - 1], Hh[nx - 1]) and np.array_equal(hz1[:, ny - 1], Hh[:, ny - 1])
    assert np.array_equal(ex1[:, 0], E[:, 0])


@pytest.mark.parametrize("t", [1, 2, 5])
def test_fdtd2d_light_cone(t):
    """An hz impulse at (c, c) reaches hz only within L1 distance t after t steps
    (each hz update reads hz at (i,j), (i+-1,j), (i,j+-1) through ex/ey)."""
    n = 25
    c = 12
    z = np.zeros((n, n), np.float32)
    hz = z.copy()
    hz[c, c] = 1.0
    _, _, h = oracle.fdtd2d(t, z, z, hz, np.zeros(t, np.float32))
    ii, jj = np.nonzero(h)
    d = np.abs(ii - c) + np.abs(jj - c)
    assert d.max() == t  # reaches exactly distance t (no cancellation at the front)


def test_fdtd2d_f32_twin_close_to_f64():
    nx, ny, T = 40, 36, 20
    ex, ey, hz = _rand(nx, ny), _rand(nx, ny), _rand(nx, ny)
    f = _rand(T)
    r64 = oracle.fdtd2d(T, ex, ey, hz, f)
    r32 = oracle.fdtd2d(T, ex, ey, hz, f, f32=True)
    scale = max(np.abs(a).max() for a in r64)
    for a, b in zip(r64, r32):
        assert np.abs(a - b).max() <= 1e-5 * scale


# ------------------------------------------------------------------ gramschmidt (R22)
def _qr_pos(A):
    """numpy (LAPACK Householder) QR with the sign convention diag(R) > 0."""
    Qn, Rn = np.linalg.qr(A.astype(np.float64))
    d = np.sign(np.diag(Rn))
    return Qn * d, Rn * d[:, None]


@pytest.mark.parametrize("m,n", [(4, 4), (9, 5), (33, 33), (64, 40)])
def test_gramschmidt_matches_lapack_qr(m, n):
    A = _rand(m, n, lo=-1, hi=1)
    Ao, R, Q = oracle.gramschmidt(A)
    Qn, Rn = _qr_pos(A)
    np.testing.assert_allclose(Q, Qn, atol=1e-9)
    np.testing.assert_allclose(R, Rn, atol=1e-9 * np.abs(A).max() * m)
    assert np.all(np.tril(R, -1) == 0)
    np.testing.assert_allclose(Q.T @ Q, np.eye(n), atol=1e-10)
    np.testing.assert_allclose(Q @ R, A.astype(np.float64), atol=1e-12)
    # after the sweep, column j of A holds the vector Q[:, j] was normalised from
    np.testing.assert_allclose(Ao, Q * np.diag(R)[None, :], atol=1e-12)


def test_gramschmidt_upper_triangular_is_exact():
    """QR of an upper-triangular matrix with positive diagonal is Q = I, R = A (uniqueness);
    MGS reaches it exactly (each projection removes one entry exactly)."""
    n = 12
    A = np.triu(_rand(n, n, lo=0.5, hi=2.0))
    Ao, R, Q = oracle.gramschmidt(A)
    assert np.array_equal(Q, np.eye(n))
    assert np.array_equal(R, A.astype(np.float64))


def test_gramschmidt_orthogonal_columns_closed_form():
    """Columns already orthogonal: a scaled signed permutation P D -> Q = P sign(D), R = |D|."""
    n = 10
    perm = RNG.permutation(n)
    d = RNG.choice([-4.0, -0.5, 0.25, 2.0, 8.0], size=n)
    A = np.zeros((n, n), np.float32)
    A[perm, np.arange(n)] = d
    Ao, R, Q = oracle.gramschmidt(A)
    Qe = np.zeros((n, n))
    Qe[perm, np.arange(n)] = np.sign(d)
    assert np.array_equal(Q, Qe)
    assert np.array_equal(R, np.diag(np.abs(d)))


# ------------------------------------------------------------------ PolyBench init data (NEXT-2)
def test_polybench_init_correlation_closed_form():
    """PolyBench's correlation data i*j/M + i = i (1 + j/M): every column is a positive
    multiple of i, so every correlation is 1 (up to the fp32 rounding of the data)."""
    import pbgen
    d = pbgen.polybench_init("correlation", 24, 40)
    corr, mean, sd = oracle.correlation(d["float_n"], 0.1, d["data"])
    assert np.abs(corr - 1.0).max() < 1e-6
    # and the mean of column j is mean(i) (1 + j/M) = (n-1)/2 (1 + j/M)
    np.testing.assert_allclose(mean, 19.5 * (1 + np.arange(24) / 24), rtol=1e-6)


def test_polybench_init_covariance_closed_form():
    """PolyBench's covariance data i*j/M: cov[a][b] = (a/M)(b/M) var(i), var(i) = n(n+1)/12
    (ddof 1); column 0 is constant 0, so row and column 0 vanish exactly."""
    import pbgen
    m, n = 16, 64  # i*j/M exact in fp32 (M a power of two)
    d = pbgen.polybench_init("covariance", m, n)
    cov, mean = oracle.covariance(d["float_n"], d["data"])
    a = np.arange(m) / m
    np.testing.assert_allclose(cov, np.outer(a, a) * n * (n + 1) / 12.0, rtol=1e-12, atol=1e-12)
    assert np.all(cov[0] == 0) and np.all(cov[:, 0] == 0)


# ------------------------------------------------------------------ the pins bite
def _fdtd_np(T, ex, ey, hz, f, mut=None):
    """A numpy FDTD with optional plausible mistakes, to show the pins above reject them."""
    ex, ey, hz = (a.astype(np.float64).copy() for a in (ex, ey, hz))
    ce, ch = (0.7, 0.5) if mut == "swap_coef" else (0.5, 0.7)
    for t in range(T):
        if mut != "no_source":
            ey[0, :] = f[t]
        if mut == "hz_first":
            hz[:-1, :-1] -= ch * (ex[:-1, 1:] - ex[:-1, :-1] + ey[1:, :-1] - ey[:-1, :-1])
        ey[1:, :] -= ce * (hz[1:, :] - hz[:-1, :]) if mut != "ey_sign" else -ce * (hz[1:, :] - hz[:-1, :])
        if mut == "ex_rows":
            ex[1:, :] -= ce * (hz[1:, :] - hz[:-1, :])
        else:
            ex[:, 1:] -= ce * (hz[:, 1:] - hz[:, :-1])
        if mut != "hz_first":
            hz[:-1, :-1] -= ch * (ex[:-1, 1:] - ex[:-1, :-1] + ey[1:, :-1] - ey[:-1, :-1])
    return ex, ey, hz


def test_fdtd_pins_reject_mutants():
    g = json.load(open(os.path.join(HERE, "golden", "fdtd2d_impulse.json")))
    c = g["impulse"]
    z = np.zeros((c["nx"], c["ny"]), np.float32)
    hz = z.copy()
    hz[tuple(c["hz_at"])] = 1.0
    f = np.array(c["fict"], np.float32)

    def golden_ok(res):
        for arr, key in zip(res, ("ex_nonzero", "ey_nonzero", "hz_nonzero")):
            ref = np.zeros_like(arr)
            for i, j, v in c[key]:
                ref[i, j] = v
            if np.abs(arr - ref).max() > 1e-12:
                return False
        return True

    src = g["source_case"]
    zs = np.zeros((src["nx"], src["ny"]), np.float32)

    def source_ok(res):
        return np.allclose(res[1][0], src["ey_row0"]) and np.allclose(res[2][0], src["hz_row0"])

    assert golden_ok(_fdtd_np(1, z, z, hz, f)) and source_ok(_fdtd_np(1, zs, zs, zs, np.array(src["fict"], np.float32)))
    for mut in ("swap_coef", "hz_first", "ey_sign", "ex_rows", "no_source"):
        res = _fdtd_np(1, z, z, hz, f, mut)
        res_s = _fdtd_np(1, zs, zs, zs, np.array(src["fict"], np.float32), mut)
        assert not (golden_ok(res) and source_ok(res_s)), mut


def test_conv_pins_reject_mutants():
    """scipy's correlate rejects a convolution (flipped kernel), transposed weights,
    a dropped tap and a shifted window."""
    A = _rand(9, 11, lo=-1, hi=1).astype(np.float64)
    w = RNG.normal(size=(3, 3))
    ref = signal.correlate2d(A, w, mode="valid")
    mutants = [signal.convolve2d(A, w, mode="valid"), signal.correlate2d(A, w.T, mode="valid"),
               signal.correlate2d(A, np.where(np.arange(9).reshape(3, 3) == 4, 0, w), mode="valid"),
               signal.correlate2d(A, w, mode="full")[2:-2, 1:-3]]
    for mtt in mutants:
        assert np.abs(mtt - ref).max() > 1e-6


def test_gramschmidt_pins_reject_mutants():
    """The LAPACK-QR pin rejects an unnormalised Q, a missing projection and a wrong sign."""
    A = _rand(20, 12, lo=-1, hi=1).astype(np.float64)
    Qn, Rn = _qr_pos(A.astype(np.float32))
    Ao, R, Q = oracle.gramschmidt(A.astype(np.float32))
    assert np.abs(Q - Qn).max() < 1e-9
    bad_unnorm = Q * np.diag(R)[None, :]
    bad_sign = Q.copy()
    bad_sign[:, 3] *= -1
    # classical GS with one projection dropped (q_0 never removed from column 2)
    Qd = np.zeros_like(A)
    for k in range(A.shape[1]):
        v = A[:, k].copy()
        for i in range(k):
            if not (k == 2 and i == 0):
                v -= (Qd[:, i] @ A[:, k]) * Qd[:, i]
        Qd[:, k] = v / np.linalg.norm(v)
    for mtt in (bad_unnorm, bad_sign, Qd):
        assert np.abs(mtt - Qn).max() > 1e-6
