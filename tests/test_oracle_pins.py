"""Pins for the CPU oracle (task rule ③): each oracle function is checked
against something other than itself — exact rational brute force, closed
forms, invariants, textbook library routines (numpy float64, np.cov,
np.corrcoef) and the golden fixtures in tests/golden/. The pins are chosen so
that a dropped term, wrong sign/index or transposed operand fails one of them
(see test_pins_catch_mutations for that claim checked directly).

Pin ids (P1..P34) follow SURVEY.md §8(c) "What pins each part".
"""
import json
import os
from fractions import Fraction

import numpy as np
import pytest

import oracle
import pbgen

HERE = os.path.dirname(os.path.abspath(__file__))
rng = np.random.default_rng(2312)


def U(*shape, lo=0.0, hi=1.0):
    return rng.uniform(lo, hi, size=shape).astype(np.float32)


def F(x):
    return Fraction(float(x))


def close(a, b, tol):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    s = np.maximum(np.abs(b), 1e-300)
    return np.max(np.abs(a - b) / np.where(np.abs(b) > 0, s, 1.0)) <= tol


# ------------------------------------------------------------------ generator
def test_pbgen_splitmix64_known_value():
    # splitmix64 seeded with state 0 produces 0xE220A8397B1DCDAF as its first
    # output (Steele, Lea & Flood 2014 reference implementation; golden file).
    g = json.load(open(os.path.join(HERE, "golden", "pbgen.json")))
    z = pbgen._splitmix64(np.array([0], dtype=np.uint64))[0]
    assert int(z) == int(g["splitmix64_state0_first"], 16)


def test_pbgen_host_matches_numpy_bitwise():
    for mode in (pbgen.U01, pbgen.INT8, pbgen.BIN, pbgen.U01 | pbgen.SYM):
        a = pbgen.gen_numpy(37, 41, 5, mode=mode, scale=0.5, offset=-0.25, row0=3, ld=41)
        b = pbgen.gen_host(37, 41, 5, mode=mode, scale=0.5, offset=-0.25, row0=3, ld=41)
        assert np.array_equal(a.view(np.uint32), b.view(np.uint32))


def test_pbgen_shards_are_rows_of_full():
    full = pbgen.gen_host(64, 24, 1)
    part = pbgen.gen_host(16, 24, 1, row0=20)
    assert np.array_equal(full[20:36], part)


def test_pbgen_ranges():
    u = pbgen.gen_host(256, 256, 1)
    assert u.min() >= 0 and u.max() < 1 and abs(u.mean() - 0.5) < 0.01
    i8 = pbgen.gen_host(64, 64, 1, mode=pbgen.INT8)
    assert set(np.unique(i8)) <= set(range(8)) and len(np.unique(i8)) == 8
    s = pbgen.gen_host(33, 33, 3, mode=pbgen.SYM)
    assert np.array_equal(s, s.T)


# ------------------------------------------------------------------ gemm
def test_gemm_golden_worked_example():
    g = json.load(open(os.path.join(HERE, "golden", "gemm_2x3x2.json")))
    out = oracle.gemm(g["alpha"], g["beta"], np.array(g["C"]), np.array(g["A"]), np.array(g["B"]))
    assert np.array_equal(out, np.array(g["expected"], dtype=np.float64))


def test_gemm_exact_rationals_P5():
    for (ni, nj, nk) in [(3, 5, 4), (6, 2, 5), (1, 1, 6)]:
        A, B, C = U(ni, nk, lo=-1), U(nk, nj, lo=-1), U(ni, nj, lo=-1)
        al, be = 1.5, 1.2
        out = oracle.gemm(al, be, C, A, B)
        for i in range(ni):
            for j in range(nj):
                ex = F(be) * F(C[i, j]) + F(al) * sum(F(A[i, k]) * F(B[k, j]) for k in range(nk))
                mag = F(be) * abs(F(C[i, j])) + F(al) * sum(abs(F(A[i, k]) * F(B[k, j])) for k in range(nk))
                assert abs(F(out[i, j]) - ex) <= mag * (nk + 2) * Fraction(1, 2**53)


def test_gemm_numpy_P6():
    A, B, C = U(37, 29, lo=-1), U(29, 53, lo=-1), U(37, 53, lo=-1)
    out = oracle.gemm(1.5, 1.2, C, A, B)
    ref = 1.5 * (A.astype(np.float64) @ B.astype(np.float64)) + 1.2 * C.astype(np.float64)
    assert np.max(np.abs(out - ref)) <= 1e-12 * np.max(np.abs(ref))


def test_gemm_identity_and_alpha0_P2_P3():
    B, C = U(16, 9), U(16, 9)
    out = oracle.gemm(1.5, 0.5, C, np.eye(16, dtype=np.float32), B)
    assert np.array_equal(out, 1.5 * B.astype(np.float64) + 0.5 * C.astype(np.float64))
    out = oracle.gemm(0.0, 0.5, C, U(16, 7), U(7, 9))
    assert np.array_equal(out, 0.5 * C.astype(np.float64))


def test_gemm_rank1_P4():
    u, v, w, z = U(8, lo=-1), U(5, lo=-1), U(5, lo=-1), U(11, lo=-1)
    A = np.outer(u, v).astype(np.float32)
    B = np.outer(w, z).astype(np.float32)
    out = oracle.gemm(1.0, 0.0, np.zeros((8, 11), np.float32), A, B)
    # (A)(B) = sum_k A[i,k] B[k,j]: closed form on the stored fp32 factors
    ref = np.einsum("ik,kj->ij", A.astype(np.float64), B.astype(np.float64))
    assert np.max(np.abs(out - ref)) <= 1e-14 * np.max(np.abs(ref))
    ref2 = np.outer(u.astype(np.float64), z.astype(np.float64)) * float(np.dot(v.astype(np.float64), w.astype(np.float64)))
    assert np.max(np.abs(out - ref2)) <= 1e-6 * np.max(np.abs(ref2))  # fp32 rounding of the outer products


def test_gemm_absmode_is_magnitude():
    A, B, C = U(9, 7, lo=-1), U(7, 5, lo=-1), U(9, 5, lo=-1)
    s = oracle.gemm(-1.5, -1.2, C, A, B, absmode=True)
    ref = 1.5 * np.abs(A.astype(np.float64)) @ np.abs(B.astype(np.float64)) + 1.2 * np.abs(C.astype(np.float64))
    assert close(s, ref, 1e-14)


def test_gemm_at_matches_full():
    A, B, C = U(33, 17), U(17, 21), U(33, 21)
    full = oracle.gemm(1.5, 1.2, C, A, B)
    r = rng.integers(0, 33, 50)
    c = rng.integers(0, 21, 50)
    assert np.array_equal(oracle.gemm_at(1.5, 1.2, C, A, B, r, c), full[r, c])


# ------------------------------------------------------------------ 2mm / 3mm
def test_2mm_chain_identity_P7():
    A, B, D = U(12, 9), U(9, 10), U(12, 10)
    tmp, Dp = oracle.mm2(1.5, 1.2, A, B, np.eye(10, dtype=np.float32), D)
    g = oracle.gemm(1.5, 1.2, D, A, B)
    assert np.array_equal(Dp, g)
    assert np.array_equal(tmp, oracle.gemm(1.5, 0.0, np.zeros((12, 10), np.float32), A, B))


def test_2mm_numpy():
    A, B, C, D = U(13, 7, lo=-1), U(7, 11, lo=-1), U(11, 5, lo=-1), U(13, 5, lo=-1)
    tmp, Dp = oracle.mm2(1.5, 1.2, A, B, C, D)
    a, b, c, d = (x.astype(np.float64) for x in (A, B, C, D))
    assert close(tmp, 1.5 * a @ b, 1e-12)
    ref = (1.5 * a @ b) @ c + 1.2 * d
    assert np.max(np.abs(Dp - ref)) <= 1e-12 * np.max(np.abs(ref))


def test_2mm_rows_matches_full():
    A, B, C, D = U(20, 8), U(8, 9), U(9, 6), U(20, 6)
    tmp, Dp = oracle.mm2(1.5, 1.2, A, B, C, D)
    rows = np.array([0, 3, 19])
    t2, d2 = oracle.mm2_rows(1.5, 1.2, A, B, C, D, rows)
    assert np.array_equal(t2, tmp[rows]) and np.allclose(d2, Dp[rows], rtol=1e-15, atol=0)


def test_3mm_identity_and_numpy_P7_P8():
    A, B = U(9, 6), U(6, 8)
    I = np.eye(8, dtype=np.float32)
    E, Fm, G = oracle.mm3(A, B, I, I)
    assert np.array_equal(Fm, np.eye(8)) and np.array_equal(G, E)
    A, B, C, D = U(9, 6, lo=-1), U(6, 8, lo=-1), U(8, 5, lo=-1), U(5, 7, lo=-1)
    E, Fm, G = oracle.mm3(A, B, C, D)
    a, b, c, d = (x.astype(np.float64) for x in (A, B, C, D))
    assert close(E, a @ b, 1e-12) and close(Fm, c @ d, 1e-12)
    ref = a @ (b @ (c @ d))  # associativity (P8)
    assert np.max(np.abs(G - ref)) <= 1e-12 * np.max(np.abs(ref))
    E2, F2, G2 = oracle.mm3_rows(A, B, C, D, np.array([1, 4]))
    assert np.array_equal(E2, E[[1, 4]]) and np.allclose(G2, G[[1, 4]], rtol=1e-14)


# ------------------------------------------------------------------ syrk / syr2k
def test_syrk_tril_of_gemm_P9_P10():
    A, C = U(14, 9, lo=-1), U(14, 14, lo=-1)
    out = oracle.syrk(1.5, 1.2, C, A)
    g = oracle.gemm(1.5, 1.2, C, A, np.ascontiguousarray(A.T))
    low = np.tril_indices(14)
    up = np.triu_indices(14, 1)
    assert np.array_equal(out[low], g[low])
    assert np.array_equal(out[up], C.astype(np.float64)[up])  # strict upper untouched bitwise
    full = oracle.gemm(1.0, 0.0, np.zeros((14, 14), np.float32), A, np.ascontiguousarray(A.T))
    assert np.array_equal(full, full.T)  # P10 bitwise symmetric


def test_syrk_orthonormal_rows_P11():
    P = np.eye(6, dtype=np.float32)[[3, 0, 5, 1, 4, 2]] * np.float32(0.5)
    out = oracle.syrk(4.0, 0.0, np.zeros((6, 6), np.float32), P)
    assert np.array_equal(np.tril(out), np.eye(6))


def test_syrk_exact_rationals():
    A, C = U(5, 4, lo=-1), U(5, 5, lo=-1)
    out = oracle.syrk(1.5, 1.2, C, A)
    for i in range(5):
        for j in range(i + 1):
            ex = F(1.2) * F(C[i, j]) + F(1.5) * sum(F(A[i, k]) * F(A[j, k]) for k in range(4))
            mag = F(1.2) * abs(F(C[i, j])) + F(1.5) * sum(abs(F(A[i, k]) * F(A[j, k])) for k in range(4))
            # fp64 summation error bound: (K+2) u sum|terms|, u = 2^-53
            assert abs(F(out[i, j]) - ex) <= mag * 6 * Fraction(1, 2**53)


def test_syr2k_equals_syrk_doubled_P12():
    A, C = U(11, 7, lo=-1), U(11, 11, lo=-1)
    assert np.array_equal(oracle.syr2k(1.5, 1.2, C, A, A), oracle.syrk(3.0, 1.2, C, A))


def test_syr2k_numpy_P13_and_index_order():
    A, B, C = U(10, 6, lo=-1), U(10, 6, lo=-1), U(10, 10, lo=-1)
    out = oracle.syr2k(1.5, 1.2, C, A, B)
    a, b, c = (x.astype(np.float64) for x in (A, B, C))
    ref = 1.5 * (b @ a.T + a @ b.T) + 1.2 * c  # C[i][j] += A[j]B[i] + B[j]A[i]
    low = np.tril_indices(10)
    assert close(out[low], ref[low], 1e-12)
    assert np.array_equal(out[np.triu_indices(10, 1)], c[np.triu_indices(10, 1)])
    for i in range(3, 6):
        for j in range(i + 1):
            ex = F(1.2) * F(C[i, j]) + F(1.5) * sum(F(A[j, k]) * F(B[i, k]) + F(B[j, k]) * F(A[i, k]) for k in range(6))
            mag = F(1.2) * abs(F(C[i, j])) + F(1.5) * sum(abs(F(A[j, k]) * F(B[i, k])) + abs(F(B[j, k]) * F(A[i, k])) for k in range(6))
            assert abs(F(out[i, j]) - ex) <= mag * 16 * Fraction(1, 2**53)


def test_syrk_at_matches_full():
    A, B, C = U(19, 8), U(19, 8), U(19, 19)
    r = rng.integers(0, 19, 60)
    c = rng.integers(0, 19, 60)
    assert np.array_equal(oracle.syrk_at(1.5, 1.2, C, A, r, c), oracle.syrk(1.5, 1.2, C, A)[r, c])
    assert np.array_equal(oracle.syrk_at(1.5, 1.2, C, A, r, c, B=B), oracle.syr2k(1.5, 1.2, C, A, B)[r, c])


# ------------------------------------------------------------------ covariance
def test_covariance_numpy_cov_P15_and_mean():
    data = U(50, 12)
    cov, mean = oracle.covariance(50.0, data)
    d = data.astype(np.float64)
    assert close(mean, d.mean(axis=0), 1e-14)
    assert np.max(np.abs(cov - np.cov(d, rowvar=False, ddof=1))) <= 1e-12 * np.max(np.abs(cov))


def test_covariance_constant_column_P14_and_symmetry_P16():
    data = U(40, 9)
    data[:, 2] = 0.5
    cov, mean = oracle.covariance(40.0, data)
    assert np.all(cov[2, :] == 0.0) and np.all(cov[:, 2] == 0.0)
    assert np.array_equal(cov, cov.T)
    assert np.all(np.diag(cov) >= 0)
    ev = np.linalg.eigvalsh(cov)
    assert ev.min() >= -1e-12 * ev.max()


def test_covariance_affine_closed_form_P17():
    n = 64
    t = (np.floor(U(n) * 1024) / 1024).astype(np.float32)  # 10-bit values: 0.25 + 2t is exact in fp32
    data = np.stack([t, 0.25 + 2.0 * t, U(n)], axis=1).astype(np.float32)
    cov, _ = oracle.covariance(float(n), data)
    td = t.astype(np.float64)
    var = np.sum((td - td.mean()) ** 2) / (n - 1)
    assert abs(cov[1, 1] - 4.0 * var) <= 1e-12 * cov[1, 1]
    assert abs(cov[0, 1] - 2.0 * var) <= 1e-12 * cov[0, 1]


def test_covariance_exact_rationals():
    data = U(6, 3)
    cov, mean = oracle.covariance(6.0, data)
    cols = [[F(data[i, j]) for i in range(6)] for j in range(3)]
    mu = [sum(c) / 6 for c in cols]
    for i in range(3):
        for j in range(3):
            ex = sum((cols[i][k] - mu[i]) * (cols[j][k] - mu[j]) for k in range(6)) / 5
            assert abs(F(cov[i, j]) - ex) <= abs(ex) * Fraction(1, 10**13) + Fraction(1, 10**20)


# ------------------------------------------------------------------ correlation
def test_correlation_diag_bounds_dup_neg_P18_P19_P20():
    data = U(64, 8)
    data[:, 3] = data[:, 2]
    data[:, 4] = 1.0 - data[:, 2]
    corr, mean, sd = oracle.correlation(64.0, 0.1, data)
    assert np.all(np.diag(corr) == 1.0)
    assert np.max(np.abs(corr)) <= 1 + 1e-12
    assert abs(corr[2, 3] - 1.0) <= 1e-12 and abs(corr[2, 4] + 1.0) <= 1e-6
    assert np.array_equal(corr, corr.T)


def test_correlation_numpy_corrcoef_P21():
    data = U(80, 10)
    corr, mean, sd = oracle.correlation(80.0, 0.1, data)
    assert np.max(np.abs(corr - np.corrcoef(data.astype(np.float64), rowvar=False))) <= 1e-12
    assert close(sd, data.astype(np.float64).std(axis=0), 1e-13)


def test_correlation_eps_rule_P22():
    n = 128
    data = U(n, 4)
    data[:, 1] = (U(n) * np.float32(1.0 / 64)).astype(np.float32)  # sd ~ 0.0045 <= eps
    corr, mean, sd = oracle.correlation(float(n), 0.1, data)
    assert sd[1] == 1.0
    d = data.astype(np.float64)
    m = d.mean(axis=0)
    sdj = np.sqrt(np.sum((d[:, 2] - m[2]) ** 2) / n)
    ex = np.sum((d[:, 1] - m[1]) * (d[:, 2] - m[2])) / (n * sdj)
    assert abs(corr[1, 2] - ex) <= 1e-12 * abs(ex) + 1e-18
    # the eps comparison is inclusive: sd == eps exactly -> replaced
    x = np.array([0.0, 0.0, 0.25, 0.25] * 4, np.float32)  # mean 0.125, sd exactly 0.125
    c2, _, sd2 = oracle.correlation(16.0, 0.125, np.stack([x, U(16)], 1))
    assert sd2[0] == 1.0


# ------------------------------------------------------------------ matvec family
def test_atax_closed_forms_P23_P24_and_numpy_P25():
    x = U(9)
    y, tmp = oracle.atax(np.eye(9, dtype=np.float32), x)
    assert np.array_equal(y, x.astype(np.float64))
    x = U(7)
    y, tmp = oracle.atax(np.ones((5, 7), np.float32), x)
    sx = float(np.sum(x.astype(np.float64)))
    assert close(tmp, np.full(5, sx), 1e-15) and close(y, np.full(7, 5 * sx), 1e-15)
    A, x = U(13, 17, lo=-1), U(17, lo=-1)
    y, tmp = oracle.atax(A, x)
    a = A.astype(np.float64)
    assert close(tmp, a @ x.astype(np.float64), 1e-12)
    ref = a.T @ (a @ x.astype(np.float64))
    assert np.max(np.abs(y - ref)) <= 1e-12 * np.max(np.abs(ref))


def test_bicg_P26_P27():
    p, r = U(8), U(8)
    s, q = oracle.bicg(np.eye(8, dtype=np.float32), p, r)
    assert np.array_equal(q, p.astype(np.float64)) and np.array_equal(s, r.astype(np.float64))
    A, p, r = U(11, 6, lo=-1), U(6, lo=-1), U(11, lo=-1)  # A n x m: q has n, s has m
    s, q = oracle.bicg(A, p, r)
    a = A.astype(np.float64)
    assert s.shape == (6,) and q.shape == (11,)
    assert close(q, a @ p.astype(np.float64), 1e-12) and close(s, a.T @ r.astype(np.float64), 1e-12)


def test_mvt_P28_P29_numpy():
    n = 12
    A = pbgen.gen_host(n, n, 1, mode=pbgen.INT8 | pbgen.SYM)
    x1, x2, y = U(n), U(n), pbgen.gen_host(1, n, 6, mode=pbgen.INT8)[0]
    o1, o2 = oracle.mvt(x1, x2, y, y, A)
    assert np.array_equal(o1 - x1.astype(np.float64), o2 - x2.astype(np.float64))
    o1, o2 = oracle.mvt(x1, x2, y, U(n), np.eye(n, dtype=np.float32))
    assert np.array_equal(o1, x1.astype(np.float64) + y.astype(np.float64))
    A, y1, y2 = U(n, n, lo=-1), U(n), U(n)
    o1, o2 = oracle.mvt(x1, x2, y1, y2, A)
    a = A.astype(np.float64)
    assert close(o1, x1 + a @ y1.astype(np.float64), 1e-12)
    assert close(o2, x2 + a.T @ y2.astype(np.float64), 1e-12)


def test_gesummv_P30_P31_numpy():
    A, x = U(10, 10), U(10)
    tmp, y = oracle.gesummv(1.5, 1.2, A, A, x)
    assert close(y, 2.7 * (A.astype(np.float64) @ x.astype(np.float64)), 1e-14)
    B = U(10, 10)
    tmp, y = oracle.gesummv(1.5, 0.0, A, B, x)
    assert np.array_equal(y, 1.5 * tmp)
    tmp, y = oracle.gesummv(1.5, 1.2, np.eye(10, dtype=np.float32), B, x)
    assert close(y, 1.5 * x.astype(np.float64) + 1.2 * B.astype(np.float64) @ x.astype(np.float64), 1e-14)
    A, B, x = U(9, 9, lo=-1), U(9, 9, lo=-1), U(9, lo=-1)
    tmp, y = oracle.gesummv(1.5, 1.2, A, B, x)
    a, b, xx = A.astype(np.float64), B.astype(np.float64), x.astype(np.float64)
    assert close(y, 1.5 * a @ xx + 1.2 * b @ xx, 1e-12)


def test_oracle_thread_count_invariance():
    """Bitwise identical for 1 and many threads (fixed per-output order)."""
    import subprocess
    import sys
    code = ("import numpy as np, oracle, pbgen;"
            "A=pbgen.gen_host(300,257,1);x=pbgen.gen_host(1,257,6)[0];"
            "y,t=oracle.atax(A,x);import hashlib;print(hashlib.sha1(y.tobytes()+t.tobytes()).hexdigest())")
    root = os.path.dirname(HERE)
    outs = []
    for th in ("1", "5"):
        env = dict(os.environ, OMP_NUM_THREADS=th, PYTHONPATH=root)
        outs.append(subprocess.check_output([sys.executable, "-c", code], env=env, cwd=root).strip())
    assert outs[0] == outs[1]


# ------------------------------------------------------------------ pin strength
def test_pins_catch_mutations():
    """Each plausible oracle mistake (dropped term, wrong sign, wrong index,
    transposed operand, wrong normaliser) produces outputs that the pins'
    references above reject at the pins' tolerances."""
    A, B, C, D = U(12, 12), U(12, 12), U(12, 12), U(12, 12)
    a, b, c, d = (x.astype(np.float64) for x in (A, B, C, D))
    x, y = U(12).astype(np.float64), U(12).astype(np.float64)
    al, be = 1.5, 1.2
    good = {
        "gemm": al * a @ b + be * c,
        "syrk": np.tril(al * a @ a.T + be * c) + np.triu(c, 1),
        "syr2k": np.tril(al * (b @ a.T + a @ b.T) + be * c) + np.triu(c, 1),
        "cov": np.cov(a, rowvar=False, ddof=1),
        "corr": np.corrcoef(a, rowvar=False),
        "atax": a.T @ (a @ x),
        "bicg_s": a.T @ y,
        "mvt_x2": a.T @ y,
        "gesummv": al * a @ x + be * b @ x,
    }
    mutants = {
        "gemm": [al * a @ b, al * a @ b.T + be * c, al * a.T @ b + be * c, al * a @ b - be * c,
                 be * a @ b + al * c],
        "syrk": [np.tril(al * a.T @ a + be * c) + np.triu(c, 1), al * a @ a.T + be * c,
                 np.tril(al * a @ a.T) + np.triu(c, 1)],
        "syr2k": [np.tril(al * (a @ b.T) + be * c) + np.triu(c, 1),
                  np.tril(al * (a.T @ b + b.T @ a) + be * c) + np.triu(c, 1)],
        "cov": [np.cov(a, rowvar=False, ddof=0), np.cov(a, rowvar=True), (a.T @ a) / 11],
        "corr": [np.cov(a, rowvar=False), np.corrcoef(a, rowvar=True)],
        "atax": [a @ (a @ x), a @ (a.T @ x), a.T @ x],
        "bicg_s": [a @ y],
        "mvt_x2": [a @ y],
        "gesummv": [al * a @ x + be * a @ x, al * a @ x, al * a.T @ x + be * b @ x],
    }
    for k, refs in mutants.items():
        for m in refs:
            assert not close(m, good[k], 1e-6), k


def test_hand_worked_goldens_all_kernels():
    """Hand-worked PolyBench instances (tests/golden/polybench_hand.json, arithmetic in
    each entry's 'how') for every kernel besides gemm's own golden."""
    g = json.load(open(os.path.join(HERE, "golden", "polybench_hand.json")))
    f32 = lambda v: np.array(v, np.float32)  # noqa: E731
    ok = lambda a, b: np.allclose(np.asarray(a, np.float64), np.asarray(b, np.float64), rtol=0, atol=1e-12)  # noqa: E731
    c = g["covariance"]
    cov, mean = oracle.covariance(c["float_n"], f32(c["data"]))
    assert ok(cov, c["cov"]) and ok(mean, c["mean"])
    c = g["correlation"]
    assert ok(oracle.correlation(c["float_n"], c["eps"], f32(c["data"]))[0], c["corr"])
    c = g["atax"]
    y, tmp = oracle.atax(f32(c["A"]), f32(c["x"]))
    assert ok(y, c["y"]) and ok(tmp, c["tmp"])
    c = g["bicg"]
    s, q = oracle.bicg(f32(c["A"]), f32(c["p"]), f32(c["r"]))
    assert ok(s, c["s"]) and ok(q, c["q"])
    c = g["mvt"]
    o1, o2 = oracle.mvt(f32(c["x1"]), f32(c["x2"]), f32(c["y_1"]), f32(c["y_2"]), f32(c["A"]))
    assert ok(o1, c["x1_out"]) and ok(o2, c["x2_out"])
    c = g["gesummv"]
    tmp, y = oracle.gesummv(1.5, 1.2, f32(c["A"]), f32(c["B"]), f32(c["x"]))
    assert ok(tmp, c["tmp"]) and ok(y, c["y"])
    c = g["syrk"]
    assert ok(oracle.syrk(1.5, 1.2, f32(c["C"]), f32(c["A"])), c["C_out"])
    c = g["syr2k"]
    assert ok(oracle.syr2k(1.5, 1.2, f32(c["C"]), f32(c["A"]), f32(c["B"])), c["C_out"])
    c = g["2mm"]
    tmp, D = oracle.mm2(1.5, 1.2, f32(c["A"]), f32(c["B"]), f32(c["C"]), f32(c["D"]))
    assert ok(tmp, c["tmp"]) and ok(D, c["D_out"])
    c = g["3mm"]
    E, F, G = oracle.mm3(f32(c["A"]), f32(c["B"]), f32(c["C"]), f32(c["D"]))
    assert ok(E, c["E"]) and ok(F, c["F"]) and ok(G, c["G"])
