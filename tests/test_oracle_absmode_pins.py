"""Pins for the oracle's magnitude scale (``absmode``): the denominator s_e of the
componentwise parity gate, reading R8.

Every parity claim divides |gpu - oracle| by s_e, so a wrong s_e loosens (or
tightens) the gate silently. Each ``absmode`` path is checked here against
something other than itself, on SIGNED inputs (where s_e != |r_e|):
  * an independent numpy float64 formula of the definition on absolute values
    (|alpha| |A| |B| + |beta| |C|, |Xc|^T |Xc| / (n-1) with Xc = data - mean, ...);
  * hand-worked instances (tests/golden/absmode_hand.json, arithmetic written out);
  * the sampled-evaluation helpers (``*_at``, ``rows_mm``, ``mm2_rows``,
    ``mm3_rows``) against the full absmode oracle;
  * a source-level mutation test: pb_oracle.cpp is copied, one absmode statement
    is changed (e.g. |data| instead of |data - mean| for covariance/correlation),
    the copy is compiled and loaded, and the pins above must reject it.
"""
import ctypes
import json
import os
import re
import shutil
import subprocess

import numpy as np
import pytest

import oracle

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
rng = np.random.default_rng(131702)


def U(*shape, lo=-1.0, hi=1.0):
    return rng.uniform(lo, hi, size=shape).astype(np.float32)


def d(x):
    return np.asarray(x, np.float64)


def close(a, b, tol=1e-12):
    a, b = d(a), d(b)
    return np.max(np.abs(a - b)) <= tol * max(1.0, np.max(np.abs(b)))


# ------------------------------------------------------------------ numpy formulas
def pin_gemm(ora=oracle):
    A, B, C = U(13, 9), U(9, 11), U(13, 11)
    s = ora.gemm(-1.5, -1.2, C, A, B, absmode=True)
    assert close(s, 1.5 * np.abs(d(A)) @ np.abs(d(B)) + 1.2 * np.abs(d(C)))


def pin_2mm(ora=oracle):
    A, B, C, D = U(7, 5), U(5, 6), U(6, 4), U(7, 4)
    ts, Ds = ora.mm2(-1.5, -1.2, A, B, C, D, absmode=True)
    t_ref = 1.5 * np.abs(d(A)) @ np.abs(d(B))
    assert close(ts, t_ref)
    assert close(Ds, t_ref @ np.abs(d(C)) + 1.2 * np.abs(d(D)))


def pin_3mm(ora=oracle):
    A, B, C, D = U(6, 5), U(5, 7), U(7, 4), U(4, 3)
    Es, Fs, Gs = ora.mm3(A, B, C, D, absmode=True)
    E_ref, F_ref = np.abs(d(A)) @ np.abs(d(B)), np.abs(d(C)) @ np.abs(d(D))
    assert close(Es, E_ref) and close(Fs, F_ref) and close(Gs, E_ref @ F_ref)


def pin_syrk(ora=oracle):
    A, C = U(9, 6), U(9, 9)
    s = ora.syrk(-1.5, -1.2, C, A, absmode=True)
    a, c = np.abs(d(A)), np.abs(d(C))
    assert close(s, np.tril(1.5 * a @ a.T + 1.2 * c) + np.triu(c, 1))


def pin_syr2k(ora=oracle):
    A, B, C = U(9, 6), U(9, 6), U(9, 9)
    s = ora.syr2k(-1.5, -1.2, C, A, B, absmode=True)
    a, b, c = np.abs(d(A)), np.abs(d(B)), np.abs(d(C))
    # lower: |beta||C_ij| + |alpha| sum_k |A_jk||B_ik| + |B_jk||A_ik| = (b a^T + a b^T)_ij
    assert close(s, np.tril(1.5 * (b @ a.T + a @ b.T) + 1.2 * c) + np.triu(c, 1))


def _cov_data(n=40, m=7):
    # signed, non-zero means (U[-0.25, 1)), so |data| and |data - mean| differ
    return U(n, m, lo=-0.25, hi=1.0)


def pin_covariance(ora=oracle):
    data = _cov_data()
    n = data.shape[0]
    s, ms = ora.covariance(float(n), data, absmode=True)
    Xc = d(data) - d(data).mean(axis=0)
    assert close(s, np.abs(Xc).T @ np.abs(Xc) / (n - 1))
    assert close(ms, np.abs(d(data)).sum(axis=0) / n)
    # float_n != n: mean uses float_n, the normaliser is |float_n - 1|
    fn = 3214212.01
    s2, _ = ora.covariance(fn, data, absmode=True)
    Xc2 = d(data) - d(data).sum(axis=0) / fn
    assert close(s2, np.abs(Xc2).T @ np.abs(Xc2) / (fn - 1))


def pin_correlation(ora=oracle):
    data = _cov_data()
    n = data.shape[0]
    data[:, 3] = 0.5 + data[:, 3] / 512  # sd <= eps: replaced by 1 (reading R5)
    eps = 0.1
    s, ms, sds = ora.correlation(float(n), eps, data, absmode=True)
    x = d(data)
    mu = x.mean(axis=0)
    sd = np.sqrt(((x - mu) ** 2).sum(axis=0) / n)
    assert sd[3] <= eps and np.all(np.delete(sd, 3) > 2 * eps)
    sd = np.where(sd <= eps, 1.0, sd)
    Xn = np.abs((x - mu) / (np.sqrt(n) * sd))
    ref = Xn.T @ Xn
    np.fill_diagonal(ref, 1.0)
    assert close(s, ref)
    assert close(ms, np.abs(x).sum(axis=0) / n)
    assert close(sds, sd)


def pin_atax(ora=oracle):
    A, x = U(11, 8), U(8)
    ys, ts = ora.atax(A, x, absmode=True)
    t_ref = np.abs(d(A)) @ np.abs(d(x))
    assert close(ts, t_ref) and close(ys, np.abs(d(A)).T @ t_ref)


def pin_bicg(ora=oracle):
    A, p, r = U(11, 8), U(8), U(11)
    ss, qs = ora.bicg(A, p, r, absmode=True)
    assert close(qs, np.abs(d(A)) @ np.abs(d(p)))
    assert close(ss, np.abs(d(A)).T @ np.abs(d(r)))


def pin_mvt(ora=oracle):
    A, x1, x2, y1, y2 = U(9, 9), U(9), U(9), U(9), U(9)
    o1, o2 = ora.mvt(x1, x2, y1, y2, A, absmode=True)
    a = np.abs(d(A))
    assert close(o1, np.abs(d(x1)) + a @ np.abs(d(y1)))
    assert close(o2, np.abs(d(x2)) + a.T @ np.abs(d(y2)))


def pin_gesummv(ora=oracle):
    A, B, x = U(9, 9), U(9, 9), U(9)
    ts, ys = ora.gesummv(1.5, -1.2, A, B, x, absmode=True)
    xa = np.abs(d(x))
    assert close(ts, np.abs(d(A)) @ xa)
    assert close(ys, 1.5 * np.abs(d(A)) @ xa + 1.2 * np.abs(d(B)) @ xa)


PINS = [pin_gemm, pin_2mm, pin_3mm, pin_syrk, pin_syr2k, pin_covariance, pin_correlation,
        pin_atax, pin_bicg, pin_mvt, pin_gesummv]


@pytest.mark.parametrize("pin", PINS, ids=[p.__name__ for p in PINS])
def test_absmode_numpy(pin):
    pin()


def test_absmode_is_magnitude_bound():
    """s_e >= |r_e| for every kernel (triangle inequality), with equality on
    non-negative inputs (the plain max-relative-error case of R8)."""
    A, B, C = U(8, 8), U(8, 8), U(8, 8)
    r, s = oracle.gemm(-1.5, 1.2, C, A, B), oracle.gemm(-1.5, 1.2, C, A, B, absmode=True)
    assert np.all(s >= np.abs(r) * (1 - 1e-15))
    data = _cov_data()
    r, _ = oracle.covariance(40.0, data)
    s, _ = oracle.covariance(40.0, data, absmode=True)
    assert np.all(s >= np.abs(r) * (1 - 1e-15)) and np.any(s > 1.5 * np.abs(r))
    P = np.abs(A)
    assert np.array_equal(oracle.gemm(1.5, 1.2, np.abs(C), P, np.abs(B)),
                          oracle.gemm(1.5, 1.2, np.abs(C), P, np.abs(B), absmode=True))


def test_absmode_hand_worked():
    g = json.load(open(os.path.join(HERE, "golden", "absmode_hand.json")))
    f = lambda v: np.array(v, np.float32)  # noqa: E731
    ok = lambda a, b: np.allclose(d(a), d(b), rtol=0, atol=1e-12)  # noqa: E731
    c = g["covariance"]
    cov, mean = oracle.covariance(c["float_n"], f(c["data"]))
    s, ms = oracle.covariance(c["float_n"], f(c["data"]), absmode=True)
    assert ok(cov, c["cov"]) and ok(mean, c["mean"]) and ok(s, c["scale"]) and ok(ms, c["mean_scale"])
    c = g["correlation"]
    assert ok(oracle.correlation(c["float_n"], c["eps"], f(c["data"]))[0], c["corr"])
    assert ok(oracle.correlation(c["float_n"], c["eps"], f(c["data"]), absmode=True)[0], c["scale"])
    c = g["syrk"]
    assert ok(oracle.syrk(c["alpha"], c["beta"], f(c["C"]), f(c["A"]), absmode=True), c["scale"])
    c = g["syr2k"]
    assert ok(oracle.syr2k(c["alpha"], c["beta"], f(c["C"]), f(c["A"]), f(c["B"]), absmode=True), c["scale"])
    c = g["2mm"]
    ts, Ds = oracle.mm2(c["alpha"], c["beta"], f(c["A"]), f(c["B"]), f(c["C"]), f(c["D"]), absmode=True)
    assert ok(ts, c["tmp_scale"]) and ok(Ds, c["D_scale"])
    c = g["atax"]
    ys, ts = oracle.atax(f(c["A"]), f(c["x"]), absmode=True)
    assert ok(ts, c["tmp_scale"]) and ok(ys, c["y_scale"])
    c = g["gesummv"]
    ts, ys = oracle.gesummv(c["alpha"], c["beta"], f(c["A"]), f(c["B"]), f(c["x"]), absmode=True)
    assert ok(ts, c["tmp_scale"]) and ok(ys, c["y_scale"])


def test_sampled_helpers_absmode_match_full():
    """The samplers used by the full-size parity tests give the same scale as the
    full absmode oracle (signed inputs)."""
    A, B, C = U(20, 12), U(12, 16), U(20, 16)
    rows = np.array([0, 3, 19, 7]); cols = np.array([15, 0, 2, 9])
    full = oracle.gemm(-1.5, 1.2, C, A, B, absmode=True)
    assert close(oracle.gemm_at(-1.5, 1.2, C, A, B, rows, cols, absmode=True), full[rows, cols])
    S, Bs, Cs = U(16, 10), U(16, 10), U(16, 16)
    r2, c2 = np.array([5, 15, 2, 9]), np.array([5, 3, 11, 0])
    assert close(oracle.syrk_at(-1.5, 1.2, Cs, S, r2, c2, absmode=True),
                 oracle.syrk(-1.5, 1.2, Cs, S, absmode=True)[r2, c2])
    assert close(oracle.syrk_at(-1.5, 1.2, Cs, S, r2, c2, B=Bs, absmode=True),
                 oracle.syr2k(-1.5, 1.2, Cs, S, Bs, absmode=True)[r2, c2])
    A2, B2, C2, D2 = U(10, 6), U(6, 8), U(8, 5), U(10, 5)
    sel = np.array([1, 2, 3, 8])
    t_full, D_full = oracle.mm2(-1.5, 1.2, A2, B2, C2, D2, absmode=True)
    t_r, D_r = oracle.mm2_rows(-1.5, 1.2, A2, B2, C2, D2, sel, absmode=True)
    assert close(t_r, t_full[sel]) and close(D_r, D_full[sel])
    D3 = U(5, 4)
    E_f, F_f, G_f = oracle.mm3(A2, B2, C2, D3, absmode=True)
    E_r, F_r, G_r = oracle.mm3_rows(A2, B2, C2, D3, sel, absmode=True)
    assert close(E_r, E_f[sel]) and close(F_r, F_f) and close(G_r, G_f[sel])


# ------------------------------------------------------------------ mutation test
# (mutated statement regex in pb_oracle.cpp, replacement, pins that must fail)
MUTANTS = {
    # covariance absmode uses |data| instead of |data - mean|
    "cov_abs_data": (r"X\[\(size_t\)i \* m \+ j\] = S\(\(double\)data\[\(size_t\)i \* m \+ j\] - mean\[j\], absmode\);",
                     "X[(size_t)i * m + j] = absmode ? std::fabs((double)data[(size_t)i * m + j]) : (double)data[(size_t)i * m + j] - mean[j];",
                     ["pin_covariance"]),
    # correlation absmode normalises |data| instead of |data - mean|
    "corr_abs_data": (r"X\[\(size_t\)i \* m \+ j\] = S\(\(\(double\)data\[\(size_t\)i \* m \+ j\] - mean\[j\]\) / \(sq \* stddev\[j\]\), absmode\);",
                      "X[(size_t)i * m + j] = absmode ? std::fabs((double)data[(size_t)i * m + j]) / (sq * stddev[j]) : ((double)data[(size_t)i * m + j] - mean[j]) / (sq * stddev[j]);",
                      ["pin_correlation"]),
    # syrk absmode keeps the signed beta*C term
    "syrk_signed_c": (r"Cout\[e\] = beta \* V\(C\[e\], absmode\) \+ alpha \* acc;\n    \}\n  \}\n\}\n\n// syr2k",
                      "Cout[e] = beta * (double)C[e] + alpha * acc;\n    }\n  }\n}\n\n// syr2k",
                      ["pin_syrk"]),
    # syr2k absmode drops the abs on the B_jk*A_ik term
    "syr2k_signed_term": (r"V\(B\[\(size_t\)j \* m \+ k\], absmode\) \* V\(A\[\(size_t\)i \* m \+ k\], absmode\);\n      Cout",
                          "(double)B[(size_t)j * m + k] * V(A[(size_t)i * m + k], absmode);\n      Cout",
                          ["pin_syr2k"]),
    # the transposed product (atax/bicg/mvt) keeps the signed matrix element
    "col_dots_signed": (r"acc\[j - j0\] \+= wi \* V\(Mi\[j\], absmode\);",
                        "acc[j - j0] += wi * (double)Mi[j];",
                        ["pin_atax", "pin_bicg", "pin_mvt"]),
    # 2mm absmode keeps the signed alpha
    "mm2_signed_alpha": (r"void pbo_2mm\(([^{]*)\{\n  alpha = S\(alpha, absmode\);",
                         r"void pbo_2mm(\1{\n  alpha = alpha;",
                         ["pin_2mm"]),
}


@pytest.fixture(scope="module")
def mutant_libs(tmp_path_factory):
    if shutil.which("g++") is None:
        pytest.skip("g++ not available")
    src = open(os.path.join(ROOT, "oracle", "pb_oracle.cpp")).read()
    out = {}
    tmp = tmp_path_factory.mktemp("mutants")
    for name, (pat, rep, _) in MUTANTS.items():
        msrc, k = re.subn(pat, rep, src, count=1)
        assert k == 1, f"mutation {name} did not apply"
        cpp, so = tmp / f"{name}.cpp", tmp / f"{name}.so"
        cpp.write_text(msrc)
        subprocess.check_call(["g++", "-O1", "-std=c++17", "-fopenmp", "-ffp-contract=off", "-shared",
                               "-fPIC", "-w", "-o", str(so), str(cpp)])
        L = ctypes.CDLL(str(so))
        for fn, sig in oracle._SIGS.items():
            f = getattr(L, fn)
            f.argtypes = sig
            f.restype = None
        out[name] = L
    return out


@pytest.mark.parametrize("name", list(MUTANTS))
def test_absmode_pins_catch_mutations(name, mutant_libs):
    pins = {p.__name__: p for p in PINS}
    oracle.lib()
    saved = oracle._lib
    try:
        oracle._lib = mutant_libs[name]
        for pn in MUTANTS[name][2]:
            with pytest.raises(AssertionError):
                pins[pn]()
        # the mutant leaves the non-absmode result alone (a scale-only mutation)
        for pn in set(pins) - set(MUTANTS[name][2]):
            pins[pn]()
    finally:
        oracle._lib = saved
