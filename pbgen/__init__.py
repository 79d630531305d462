"""pbgen — seeded, counter-based synthetic inputs shared by the oracle harness
and the GPU harness (task rule ③: the only code both sides share).

It contains no PolyBench arithmetic. The formula is in ``pbgen_core.h``;
``gen_numpy`` re-implements it in numpy (tests pin the C host library and the
CUDA kernel against it bit for bit).

Streams follow SURVEY.md §8(d): A=1, B=2, C=3, D=4, data=5, x/p/y_1=6,
r/y_2=7, x1=8, x2=9, y=10 (E/F/G for 3mm reuse 11-13).
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

SEED = 13170
U01, INT8, BIN = 0, 1, 2
SYM = 1 << 8
STREAM = dict(A=1, B=2, C=3, D=4, data=5, x=6, p=6, y_1=6, r=7, y_2=7, x1=8, x2=9, y=10,
              E=11, F=12, G=13, tmp=14, ex=8, ey=9, hz=10, fict=6)

# Workload constants of the SYCL-Bench / PolyBench-GPU stencils (inputs, not
# method arithmetic; R19/R20). 2DConvolution's c11..c33 laid out as
# w[(di+1)*3 + (dj+1)] (row = row offset di, column = column offset dj).
CONV2D_W = [0.2, 0.5, -0.8, -0.3, 0.6, -0.9, 0.4, 0.7, 0.1]
# 3DConvolution's 15 source terms [weight, di, dj, dk] (tests/golden/conv3d_3x3x3.json).
CONV3D_TERMS = [[2, -1, -1, -1], [4, 1, -1, -1], [5, -1, -1, -1], [7, 1, -1, -1], [-8, -1, -1, -1],
                [10, 1, -1, -1], [-3, 0, -1, 0], [6, 0, 0, 0], [-9, 0, 1, 0], [2, -1, -1, 1], [4, 1, -1, 1],
                [5, -1, 0, 1], [7, 1, 0, 1], [-8, -1, 1, 1], [10, 1, 1, 1]]


def conv3d_w27(terms=None):
    """27-tap table w[(di+1)*9 + (dj+1)*3 + (dk+1)] with equal-offset terms added."""
    w = [0.0] * 27
    for c, di, dj, dk in (CONV3D_TERMS if terms is None else terms):
        w[(di + 1) * 9 + (dj + 1) * 3 + (dk + 1)] += float(c)
    return w

_HERE = os.path.dirname(os.path.abspath(__file__))
_host = None
_dev = None

M64 = (1 << 64) - 1


def _splitmix64(x: np.ndarray) -> np.ndarray:
    with np.errstate(over="ignore"):
        z = x + np.uint64(0x9E3779B97F4A7C15)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        return z ^ (z >> np.uint64(31))


def gen_numpy(rows, cols, stream, seed=SEED, mode=U01, scale=1.0, offset=0.0, row0=0, ld=None):
    """Pure-numpy generator (reference for the C/CUDA versions; small sizes)."""
    ld = cols if ld is None else ld
    r = np.arange(row0, row0 + rows, dtype=np.int64)[:, None]
    c = np.arange(cols, dtype=np.int64)[None, :]
    i, j = np.broadcast_arrays(r, c)
    if mode & SYM:
        i, j = np.maximum(i, j), np.minimum(i, j)
    idx = (i * ld + j).astype(np.uint64)
    base_key = np.uint64((seed * 0x9E3779B97F4A7C15 + stream * 0xD1B54A32D192ED03) & M64)
    with np.errstate(over="ignore"):
        z = _splitmix64(base_key + idx)
    m = mode & 0xFF
    if m == INT8:
        v = (z >> np.uint64(61)).astype(np.float64)
    elif m == BIN:
        v = (z >> np.uint64(63)).astype(np.float64)
    else:
        v = (z >> np.uint64(40)).astype(np.float64) * (1.0 / 16777216.0)
    return (v * scale + offset).astype(np.float32)


def _load_host():
    global _host
    if _host is None:
        path = os.path.join(_HERE, "libpbgen_host.so")
        if not os.path.exists(path):
            raise RuntimeError(f"{path} missing: run __graft_entry__.build()")
        lib = ctypes.CDLL(path)
        lib.pbgen_fill_host.argtypes = [ctypes.c_void_p, ctypes.c_longlong, ctypes.c_longlong,
                                        ctypes.c_longlong, ctypes.c_longlong, ctypes.c_ulonglong,
                                        ctypes.c_ulonglong, ctypes.c_int, ctypes.c_double,
                                        ctypes.c_double]
        lib.pbgen_fill_host.restype = None
        _host = lib
    return _host


def _load_dev():
    global _dev
    if _dev is None:
        path = os.path.join(_HERE, "libpbgen_dev.so")
        if not os.path.exists(path):
            raise RuntimeError(f"{path} missing: run __graft_entry__.build()")
        lib = ctypes.CDLL(path)
        lib.pbgen_fill_device.argtypes = [ctypes.c_void_p, ctypes.c_longlong, ctypes.c_longlong,
                                          ctypes.c_longlong, ctypes.c_longlong,
                                          ctypes.c_ulonglong, ctypes.c_ulonglong, ctypes.c_int,
                                          ctypes.c_double, ctypes.c_double, ctypes.c_void_p]
        lib.pbgen_fill_device.restype = ctypes.c_int
        _dev = lib
    return _dev


def gen_host(rows, cols, stream, seed=SEED, mode=U01, scale=1.0, offset=0.0, row0=0, ld=None,
             out=None):
    """C/OpenMP host generator; returns a float32 numpy array rows x cols."""
    ld = cols if ld is None else ld
    if out is None:
        out = np.empty((rows, cols), dtype=np.float32)
    assert out.dtype == np.float32 and out.flags.c_contiguous and out.size == rows * cols
    _load_host().pbgen_fill_host(out.ctypes.data, row0, row0 + rows, cols, ld, seed, stream,
                                 mode, float(scale), float(offset))
    return out


def gen_device(t, stream, seed=SEED, mode=U01, scale=1.0, offset=0.0, row0=0, ld=None,
               cuda_stream=None):
    """Fill a contiguous float32 CUDA tensor (2-D rows x cols, or 1-D) in place."""
    import torch
    assert t.is_cuda and t.dtype == torch.float32 and t.is_contiguous()
    rows, cols = (t.shape[0], t.shape[1]) if t.dim() == 2 else (1, t.shape[0])
    ld = cols if ld is None else ld
    s = torch.cuda.current_stream().cuda_stream if cuda_stream is None else cuda_stream
    rc = _load_dev().pbgen_fill_device(t.data_ptr(), row0, row0 + rows, cols, ld, seed, stream,
                                       mode, float(scale), float(offset), s)
    if rc != 0:
        raise RuntimeError(f"pbgen_fill_device failed: cuda error {rc}")
    return t


# ---------------------------------------------------------------- PolyBench/C 4.2 init_array
# the PolyBench/C 4.2 `init_array` formulas (recollection of the
# suite's sources), evaluated with PolyBench's DATA_TYPE
# float arithmetic: (float)(integer expression) / n is one fp32 division (RN), as
# numpy float32 does it. Inputs only - no kernel arithmetic. Returns float32 arrays.
def _q(num, den):
    return (np.asarray(num).astype(np.float32) / np.float32(den)).astype(np.float32)


def polybench_init(kernel, *dims):
    i2 = lambda r, c: np.meshgrid(np.arange(r, dtype=np.int64), np.arange(c, dtype=np.int64), indexing="ij")  # noqa: E731
    if kernel == "gemm":
        ni, nj, nk = dims
        i, j = i2(ni, nj); C = _q((i * j + 1) % ni, ni)
        i, j = i2(ni, nk); A = _q(i * (j + 1) % nk, nk)
        i, j = i2(nk, nj); B = _q(i * (j + 2) % nj, nj)
        return dict(alpha=1.5, beta=1.2, C=C, A=A, B=B)
    if kernel == "2mm":
        ni, nj, nk, nl = dims
        i, j = i2(ni, nk); A = _q((i * j + 1) % ni, ni)
        i, j = i2(nk, nj); B = _q(i * (j + 1) % nj, nj)
        i, j = i2(nj, nl); C = _q((i * (j + 3) + 1) % nl, nl)
        i, j = i2(ni, nl); D = _q(i * (j + 2) % nk, nk)
        return dict(alpha=1.5, beta=1.2, A=A, B=B, C=C, D=D)
    if kernel == "3mm":
        ni, nj, nk, nl, nm = dims
        i, j = i2(ni, nk); A = _q((i * j + 1) % ni, 5 * ni)
        i, j = i2(nk, nj); B = _q((i * (j + 1) + 2) % nj, 5 * nj)
        i, j = i2(nj, nm); C = _q(i * (j + 3) % nl, 5 * nl)
        i, j = i2(nm, nl); D = _q((i * (j + 2) + 2) % nk, 5 * nk)
        return dict(A=A, B=B, C=C, D=D)
    if kernel in ("syrk", "syr2k"):
        n, m = dims
        i, j = i2(n, m); A = _q((i * j + 1) % n, n); B = _q((i * j + 2) % m, m)
        i, j = i2(n, n)
        C = _q((i * j + 2) % m, m) if kernel == "syrk" else _q((i * j + 3) % n, m)
        return dict(alpha=1.5, beta=1.2, A=A, B=B, C=C)
    if kernel in ("covariance", "correlation"):
        m, n = dims
        i, j = i2(n, m)
        data = (i.astype(np.float32) * j.astype(np.float32)).astype(np.float32) / np.float32(m)
        if kernel == "correlation":
            data = (data + i.astype(np.float32)).astype(np.float32)
        return dict(float_n=float(n), data=data.astype(np.float32))
    if kernel == "atax":
        m, n = dims
        fn = np.float32(n)
        x = (np.float32(1) + np.arange(n, dtype=np.float32) / fn).astype(np.float32)
        i, j = i2(m, n); A = _q((i + j) % n, 5 * m)
        return dict(A=A, x=x)
    if kernel == "bicg":
        m, n = dims
        p = _q(np.arange(m) % m, m); r = _q(np.arange(n) % n, n)
        i, j = i2(n, m); A = _q(i * (j + 1) % n, n)
        return dict(A=A, p=p, r=r)
    if kernel == "mvt":
        (n,) = dims
        k = np.arange(n)
        i, j = i2(n, n)
        return dict(x1=_q(k % n, n), x2=_q((k + 1) % n, n), y_1=_q((k + 3) % n, n), y_2=_q((k + 4) % n, n),
                    A=_q(i * j % n, n))
    if kernel == "gesummv":
        (n,) = dims
        i, j = i2(n, n)
        return dict(alpha=1.5, beta=1.2, x=_q(np.arange(n) % n, n), A=_q((i * j + 1) % n, n), B=_q((i * j + 2) % n, n))
    if kernel == "fdtd_2d":
        tmax, nx, ny = dims
        i, j = i2(nx, ny)
        fi = i.astype(np.float32)
        return dict(fict=np.arange(tmax, dtype=np.float32),
                    ex=((fi * (j + 1).astype(np.float32)) / np.float32(nx)).astype(np.float32),
                    ey=((fi * (j + 2).astype(np.float32)) / np.float32(ny)).astype(np.float32),
                    hz=((fi * (j + 3).astype(np.float32)) / np.float32(nx)).astype(np.float32))
    if kernel == "gramschmidt":
        m, n = dims
        i, j = i2(m, n)
        A = (_q((i * j) % m, m) * np.float32(100) + np.float32(10)).astype(np.float32)
        return dict(A=A)
    raise ValueError(kernel)
