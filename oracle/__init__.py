"""CPU oracle for the PolyBench hot path — TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (the
``cpu_baseline`` leg and ``--impl reference``) may import this package. The
product path (``paper_2312_13170_b200`` / ``libpb.so``) never imports it and
shares no code with it.

Every function here is a ctypes call into ``pb_oracle.cpp`` (plain C++,
fp64 accumulation, OpenMP over outputs), whose header cites the definitions
(Listing 8; PolyBench/C 4.2 statements per SURVEY.md §8(c)).
Inputs are float32 numpy arrays; outputs are float64 numpy arrays.

``absmode=True`` evaluates the same definition on absolute values (the
per-element magnitude scale used by the componentwise parity gate, reading R8).

Parity status: every function is pinned in tests/test_oracle_pins.py
(closed forms, exact rationals, numpy library cross-checks, invariants).
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_lib = None

_F = ctypes.c_void_p
_I = ctypes.c_int
_D = ctypes.c_double

_SIGS = {
    "pbo_gemm": [_I, _I, _I, _D, _D, _F, _F, _F, _F, _I],
    "pbo_2mm": [_I, _I, _I, _I, _D, _D, _F, _F, _F, _F, _F, _F, _I],
    "pbo_3mm": [_I, _I, _I, _I, _I, _F, _F, _F, _F, _F, _F, _F, _I],
    "pbo_syrk": [_I, _I, _D, _D, _F, _F, _F, _I],
    "pbo_syr2k": [_I, _I, _D, _D, _F, _F, _F, _F, _I],
    "pbo_covariance": [_I, _I, _D, _F, _F, _F, _I],
    "pbo_correlation": [_I, _I, _D, _D, _F, _F, _F, _F, _I],
    "pbo_atax": [_I, _I, _F, _F, _F, _F, _I],
    "pbo_bicg": [_I, _I, _F, _F, _F, _F, _F, _I],
    "pbo_mvt": [_I, _F, _F, _F, _F, _F, _F, _F, _I],
    "pbo_gesummv": [_I, _D, _D, _F, _F, _F, _F, _F, _I],
    "pbo_gemm_at": [_I, _I, _I, _D, _D, _F, _F, _F, _I, _F, _F, _F, _I],
    "pbo_syrk_at": [_I, _I, _D, _D, _F, _F, _F, _I, _F, _F, _F, _I],
    "pbo_rows_mm": [_I, _I, _I, _I, _F, _F, _F, _I],
    "pbo_dmm": [_I, _I, _I, _F, _F, _F, _I],
    "pbo_conv2d": [_I, _I, _F, _F, _F, _I, _I, _F, _I],
    "pbo_conv3d": [_I, _I, _I, _F, _F, _F, _I, _I, _F, _I],
    "pbo_fdtd2d": [_I, _I, _I, _F, _F, _F, _F, _F, _F, _F],
    "pbo_fdtd2d_f32": [_I, _I, _I, _F, _F, _F, _F, _F, _F, _F],
    "pbo_gramschmidt": [_I, _I, _F, _F, _F, _F],
}


def lib():
    global _lib
    if _lib is None:
        path = os.path.join(_HERE, "libpb_oracle.so")
        if not os.path.exists(path):
            raise RuntimeError(f"{path} missing: run __graft_entry__.build()")
        L = ctypes.CDLL(path)
        for name, sig in _SIGS.items():
            fn = getattr(L, name)
            fn.argtypes = sig
            fn.restype = None
        _lib = L
    return _lib


def _f32(x):
    a = np.ascontiguousarray(x, dtype=np.float32)
    return a


def _p(a):
    return None if a is None else a.ctypes.data


def gemm(alpha, beta, C, A, B, absmode=False):
    A, B, C = _f32(A), _f32(B), _f32(C)
    ni, nk = A.shape
    nj = B.shape[1]
    out = np.empty((ni, nj))
    lib().pbo_gemm(ni, nj, nk, alpha, beta, _p(C), _p(A), _p(B), _p(out), int(absmode))
    return out


def mm2(alpha, beta, A, B, C, D, absmode=False):
    """2mm: returns (tmp, D')."""
    A, B, C, D = map(_f32, (A, B, C, D))
    ni, nk = A.shape
    nj = B.shape[1]
    nl = C.shape[1]
    tmp = np.empty((ni, nj))
    Dout = np.empty((ni, nl))
    lib().pbo_2mm(ni, nj, nk, nl, alpha, beta, _p(A), _p(B), _p(C), _p(D), _p(tmp), _p(Dout),
                  int(absmode))
    return tmp, Dout


def mm3(A, B, C, D, absmode=False):
    """3mm: returns (E, F, G)."""
    A, B, C, D = map(_f32, (A, B, C, D))
    ni, nk = A.shape
    nj = B.shape[1]
    nm = C.shape[1]
    nl = D.shape[1]
    E = np.empty((ni, nj))
    F = np.empty((nj, nl))
    G = np.empty((ni, nl))
    lib().pbo_3mm(ni, nj, nk, nl, nm, _p(A), _p(B), _p(C), _p(D), _p(E), _p(F), _p(G),
                  int(absmode))
    return E, F, G


def syrk(alpha, beta, C, A, absmode=False):
    A, C = _f32(A), _f32(C)
    n, m = A.shape
    out = np.empty((n, n))
    lib().pbo_syrk(n, m, alpha, beta, _p(C), _p(A), _p(out), int(absmode))
    return out


def syr2k(alpha, beta, C, A, B, absmode=False):
    A, B, C = _f32(A), _f32(B), _f32(C)
    n, m = A.shape
    out = np.empty((n, n))
    lib().pbo_syr2k(n, m, alpha, beta, _p(C), _p(A), _p(B), _p(out), int(absmode))
    return out


def covariance(float_n, data, absmode=False):
    """returns (cov, mean)."""
    data = _f32(data)
    n, m = data.shape
    cov = np.empty((m, m))
    mean = np.empty(m)
    lib().pbo_covariance(m, n, float_n, _p(data), _p(cov), _p(mean), int(absmode))
    return cov, mean


def correlation(float_n, eps, data, absmode=False):
    """returns (corr, mean, stddev)."""
    data = _f32(data)
    n, m = data.shape
    corr = np.empty((m, m))
    mean = np.empty(m)
    sd = np.empty(m)
    lib().pbo_correlation(m, n, float_n, eps, _p(data), _p(corr), _p(mean), _p(sd), int(absmode))
    return corr, mean, sd


def atax(A, x, absmode=False):
    """returns (y, tmp)."""
    A, x = _f32(A), _f32(x)
    m, n = A.shape
    y = np.empty(n)
    tmp = np.empty(m)
    lib().pbo_atax(m, n, _p(A), _p(x), _p(y), _p(tmp), int(absmode))
    return y, tmp


def bicg(A, p, r, absmode=False):
    """returns (s, q)."""
    A, p, r = _f32(A), _f32(p), _f32(r)
    n, m = A.shape
    s = np.empty(m)
    q = np.empty(n)
    lib().pbo_bicg(m, n, _p(A), _p(p), _p(r), _p(s), _p(q), int(absmode))
    return s, q


def mvt(x1, x2, y_1, y_2, A, absmode=False):
    """returns (x1', x2')."""
    x1, x2, y_1, y_2, A = map(_f32, (x1, x2, y_1, y_2, A))
    n = A.shape[0]
    o1 = np.empty(n)
    o2 = np.empty(n)
    lib().pbo_mvt(n, _p(x1), _p(x2), _p(y_1), _p(y_2), _p(A), _p(o1), _p(o2), int(absmode))
    return o1, o2


def gesummv(alpha, beta, A, B, x, absmode=False):
    """returns (tmp, y)."""
    A, B, x = _f32(A), _f32(B), _f32(x)
    n = A.shape[0]
    tmp = np.empty(n)
    y = np.empty(n)
    lib().pbo_gesummv(n, alpha, beta, _p(A), _p(B), _p(x), _p(tmp), _p(y), int(absmode))
    return tmp, y


# ---- sampled evaluation (full-size parity: entries the oracle computes one by one) ----

def gemm_at(alpha, beta, C, A, B, rows, cols, absmode=False):
    A, B, C = _f32(A), _f32(B), _f32(C)
    ni, nk = A.shape
    nj = B.shape[1]
    rows = np.ascontiguousarray(rows, dtype=np.int32)
    cols = np.ascontiguousarray(cols, dtype=np.int32)
    out = np.empty(len(rows))
    lib().pbo_gemm_at(ni, nj, nk, alpha, beta, _p(C), _p(A), _p(B), len(rows), _p(rows),
                      _p(cols), _p(out), int(absmode))
    return out


def syrk_at(alpha, beta, C, A, rows, cols, B=None, absmode=False):
    """syrk (B None) or syr2k entries at (rows[t], cols[t])."""
    A, C = _f32(A), _f32(C)
    Bp = None if B is None else _f32(B)
    n, m = A.shape
    rows = np.ascontiguousarray(rows, dtype=np.int32)
    cols = np.ascontiguousarray(cols, dtype=np.int32)
    out = np.empty(len(rows))
    lib().pbo_syrk_at(n, m, alpha, beta, _p(C), _p(A), _p(Bp), len(rows), _p(rows), _p(cols),
                      _p(out), int(absmode))
    return out


def rows_mm(X, Y, r0, r1, absmode=False):
    """double rows [r0,r1) of X @ Y (fp32 inputs)."""
    X, Y = _f32(X), _f32(Y)
    inner = X.shape[1]
    cols = Y.shape[1]
    out = np.empty((r1 - r0, cols))
    lib().pbo_rows_mm(r0, r1, inner, cols, _p(X), _p(Y), _p(out), int(absmode))
    return out


def dmm(X, Y, absmode=False):
    """X (double) @ Y (fp32) in double."""
    X = np.ascontiguousarray(X, dtype=np.float64)
    Y = _f32(Y)
    rows, inner = X.shape
    cols = Y.shape[1]
    out = np.empty((rows, cols))
    lib().pbo_dmm(rows, inner, cols, _p(X), _p(Y), _p(out), int(absmode))
    return out


def mm2_rows(alpha, beta, A, B, C, D, rows, absmode=False):
    """Rows `rows` (sorted, contiguous ranges allowed) of 2mm's tmp and D'.
    tmp[r] = alpha*A[r]B;  D'[r] = tmp[r] C + beta D[r]  (PolyBench kernel_2mm)."""
    a_alpha = abs(alpha) if absmode else alpha
    a_beta = abs(beta) if absmode else beta
    Ar = _f32(A)[rows]
    ab = rows_mm(Ar, B, 0, len(rows), absmode)
    tmp = a_alpha * ab
    Dr = _f32(D)[rows].astype(np.float64)
    if absmode:
        Dr = np.abs(Dr)
    return tmp, dmm(tmp, C, absmode) + a_beta * Dr


def mm3_rows(A, B, C, D, rows, absmode=False):
    """Rows `rows` of 3mm's E and G, plus full F (F = C D is needed by every G row)."""
    Ar = _f32(A)[rows]
    E = rows_mm(Ar, B, 0, len(rows), absmode)
    F = rows_mm(C, D, 0, _f32(C).shape[0], absmode)
    Fd = F
    # G rows = E rows (double) * F (double): reuse mm with double F via dmm on fp32 is not exact,
    # so do the double x double product here in plain numpy (library primitive, R14).
    G = E @ Fd
    return E, F, G


# ---------------------------------------------------------------- stencils
def _w(w, n):
    w = np.ascontiguousarray(np.asarray(w, dtype=np.float64).reshape(-1))
    assert w.size == n
    return w


def conv2d(w, A, B_in, rows=None, absmode=False):
    """2DConvolution (reading R19): rows [i0, i1) of B (default: all), float64."""
    A, B_in = _f32(A), _f32(B_in)
    ni, nj = A.shape
    i0, i1 = (0, ni) if rows is None else rows
    w = _w(w, 9)
    out = np.empty((i1 - i0, nj))
    lib().pbo_conv2d(ni, nj, _p(w), _p(A), _p(B_in), i0, i1, _p(out), int(absmode))
    return out


def conv3d(w, A, B_in, planes=None, absmode=False):
    """3DConvolution (reading R20): planes [i0, i1) of B (default: all), float64."""
    A, B_in = _f32(A), _f32(B_in)
    ni, nj, nk = A.shape
    i0, i1 = (0, ni) if planes is None else planes
    w = _w(w, 27)
    out = np.empty((i1 - i0, nj, nk))
    lib().pbo_conv3d(ni, nj, nk, _p(w), _p(A), _p(B_in), i0, i1, _p(out), int(absmode))
    return out


def fdtd2d(tmax, ex, ey, hz, fict, f32=False):
    """FDTD-2D (reading R21): returns (ex, ey, hz) after tmax steps; float64 state,
    or (f32=True) the PolyBench statements evaluated in fp32."""
    ex, ey, hz, fict = _f32(ex), _f32(ey), _f32(hz), _f32(fict)
    nx, ny = ex.shape
    assert fict.size >= tmax
    dt = np.float32 if f32 else np.float64
    o = [np.empty((nx, ny), dtype=dt) for _ in range(3)]
    fn = lib().pbo_fdtd2d_f32 if f32 else lib().pbo_fdtd2d
    fn(tmax, nx, ny, _p(ex), _p(ey), _p(hz), _p(fict), _p(o[0]), _p(o[1]), _p(o[2]))
    return tuple(o)


def gramschmidt(A):
    """Modified Gram-Schmidt (reading R22): returns (A_out, R, Q) in float64 for the
    fp32 input A (m x n); R's strict lower triangle is 0 (not written by the kernel)."""
    A = _f32(A)
    m, n = A.shape
    Ao, R, Q = np.empty((m, n)), np.empty((n, n)), np.empty((m, n))
    lib().pbo_gramschmidt(m, n, _p(A), _p(Ao), _p(R), _p(Q))
    return Ao, R, Q
