"""paper_2312_13170_b200 — thin Python binding of libpb (include/pb.h).

Argument marshalling only: every arithmetic step of the PolyBench hot path
runs in libpb's sm_100a kernels. PyTorch supplies device memory, streams and
(in ``dist``) process groups. There is no CPU fallback: if ``libpb.so`` is
missing or a call fails, a ``PBError`` is raised.

Function names and argument order are those of the C ABI; tensors are passed
where the ABI takes pointers. ``ws`` may be omitted, in which case a workspace
of ``workspace_size(...)`` bytes is allocated with torch on the tensors'
device (callers on the hot path should pass a preallocated one).
"""
from __future__ import annotations

import ctypes
import os

__all__ = [
    "PBError", "lib", "workspace_size", "workspace", "pb_gemm", "pb_2mm", "pb_3mm", "pb_syrk",
    "pb_syr2k", "pb_syrk_full", "pb_syr2k_full", "pb_covariance", "pb_correlation", "pb_atax", "pb_bicg", "pb_mvt", "pb_gesummv",
    "pb_row_partition", "pb_syrk_rows", "pb_gesummv_rows", "pb_syr2k_rows", "pb_matvec_partial", "pb_gemm_variant",
    "pb_version", "last_launch_count", "ABI_FUNCTIONS", "Comm", "pb_comm_unique_id", "pb_comm_init",
    "pb_comm_destroy", "pb_gemm_dist", "pb_2mm_dist", "pb_3mm_dist", "pb_syrk_dist", "pb_syr2k_dist",
    "pb_atax_dist", "pb_bicg_dist", "pb_mvt_dist", "pb_gesummv_dist", "Peer", "pb_peer_create",
    "pb_comm_init_local", "pb_comm_attach_peer", "pb_conv2d", "pb_conv3d", "pb_fdtd_2d",
    "pb_gramschmidt", "pb_covariance_rows", "pb_correlation_rows", "pb_conv2d_variant", "pb_conv3d_variant",
    "pb_gramschmidt_variant", "pb_covariance_dist", "pb_correlation_dist",
]

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libpb.so")

_P = ctypes.c_void_p
_I = ctypes.c_int
_F = ctypes.c_float
_Z = ctypes.c_size_t

# name -> argtypes, exactly as declared in include/pb.h
ABI_FUNCTIONS = {
    "pb_status_str": ([_I], ctypes.c_char_p),
    "pb_last_error": ([], ctypes.c_char_p),
    "pb_version": ([], ctypes.c_char_p),
    "pb_last_launch_count": ([], _I),
    "pb_workspace_size": ([ctypes.c_char_p, ctypes.POINTER(ctypes.c_longlong), _I,
                           ctypes.POINTER(_Z)], _I),
    "pb_gemm": ([_I, _I, _I, _F, _F, _P, _P, _P, _P, _Z, _P], _I),
    "pb_2mm": ([_I, _I, _I, _I, _F, _F, _P, _P, _P, _P, _P, _P, _Z, _P], _I),
    "pb_3mm": ([_I, _I, _I, _I, _I, _P, _P, _P, _P, _P, _P, _P, _P, _Z, _P], _I),
    "pb_syrk": ([_I, _I, _F, _F, _P, _P, _P, _Z, _P], _I),
    "pb_syr2k": ([_I, _I, _F, _F, _P, _P, _P, _P, _Z, _P], _I),
    "pb_syrk_full": ([_I, _I, _F, _F, _P, _P, _P, _Z, _P], _I),
    "pb_syr2k_full": ([_I, _I, _F, _F, _P, _P, _P, _P, _Z, _P], _I),
    "pb_covariance": ([_I, _I, _F, _P, _P, _P, _P, _Z, _P], _I),
    "pb_correlation": ([_I, _I, _F, _F, _P, _P, _P, _P, _P, _Z, _P], _I),
    "pb_atax": ([_I, _I, _P, _P, _P, _P, _P, _Z, _P], _I),
    "pb_bicg": ([_I, _I, _P, _P, _P, _P, _P, _P, _Z, _P], _I),
    "pb_mvt": ([_I, _P, _P, _P, _P, _P, _P, _Z, _P], _I),
    "pb_gesummv": ([_I, _F, _F, _P, _P, _P, _P, _P, _P, _Z, _P], _I),
    "pb_row_partition": ([_I, _I, _I, _I, _I, ctypes.POINTER(_I), ctypes.POINTER(_I)], _I),
    "pb_syrk_rows": ([_I, _I, _I, _I, _F, _F, _P, _P, _P, _Z, _P], _I),
    "pb_syr2k_rows": ([_I, _I, _I, _I, _F, _F, _P, _P, _P, _P, _Z, _P], _I),
    "pb_matvec_partial": ([_I, _I, _P, _P, _P, _P, _P, _P, _P, _P, _Z, _P], _I),
    "pb_gemm_variant": ([_I, _I, _I, _I, _F, _F, _P, _P, _P, _P, _Z, _P], _I),
    "pb_gesummv_rows": ([_I, _I, _F, _F, _P, _P, _P, _P, _P, _P, _Z, _P], _I),
    "pb_conv2d": ([_I, _I, ctypes.POINTER(_F), _P, _P, _P], _I),
    "pb_conv3d": ([_I, _I, _I, ctypes.POINTER(_F), _P, _P, _P], _I),
    "pb_conv2d_variant": ([_I, _I, _I, ctypes.POINTER(_F), _P, _P, _P], _I),
    "pb_conv3d_variant": ([_I, _I, _I, _I, ctypes.POINTER(_F), _P, _P, _P], _I),
    "pb_fdtd_2d": ([_I, _I, _I, _P, _P, _P, _P, _P, _Z, _P], _I),
    "pb_gramschmidt": ([_I, _I, _P, _P, _P, _P, _Z, _P], _I),
    "pb_gramschmidt_variant": ([_I, _I, _I, _P, _P, _P, _P, _Z, _P], _I),
    "pb_covariance_rows": ([_I, _I, _F, _I, _I, _P, _P, _P, _P, _Z, _P], _I),
    "pb_correlation_rows": ([_I, _I, _F, _F, _I, _I, _P, _P, _P, _P, _P, _Z, _P], _I),
    # multi-GPU (NCCL inside libpb)
    "pb_comm_unique_id": ([_P], _I),
    "pb_comm_init": ([_I, _I, _P, ctypes.POINTER(_P)], _I),
    "pb_comm_destroy": ([_P], _I),
    "pb_comm_size": ([_P, ctypes.POINTER(_I), ctypes.POINTER(_I)], _I),
    "pb_gemm_dist": ([_P, _I, _I, _I, _F, _F, _P, _P, _P, _P, _Z, _P], _I),
    "pb_2mm_dist": ([_P, _I, _I, _I, _I, _F, _F, _P, _P, _P, _P, _P, _P, _Z, _P], _I),
    "pb_3mm_dist": ([_P, _I, _I, _I, _I, _I, _P, _P, _P, _P, _P, _P, _P, _P, _Z, _P], _I),
    "pb_syrk_dist": ([_P, _I, _I, _F, _F, _P, _P, _P, _Z, _P], _I),
    "pb_syr2k_dist": ([_P, _I, _I, _F, _F, _P, _P, _P, _P, _Z, _P], _I),
    "pb_atax_dist": ([_P, _I, _I, _P, _P, _P, _P, _P, _Z, _P], _I),
    "pb_bicg_dist": ([_P, _I, _I, _P, _P, _P, _P, _P, _P, _Z, _P], _I),
    "pb_mvt_dist": ([_P, _I, _P, _P, _P, _P, _P, _P, _Z, _P], _I),
    "pb_gesummv_dist": ([_P, _I, _F, _F, _P, _P, _P, _P, _P, _P, _Z, _P], _I),
    "pb_covariance_dist": ([_P, _I, _I, _F, _P, _P, _P, _P, _Z, _P], _I),
    "pb_correlation_dist": ([_P, _I, _I, _F, _F, _P, _P, _P, _P, _P, _Z, _P], _I),
    # peer-memory collectives (CUDA IPC symmetric buffers)
    "pb_peer_create": ([_I, _I, _Z, ctypes.POINTER(_P), _P], _I),
    "pb_peer_open": ([_P, _P], _I),
    "pb_peer_destroy": ([_P], _I),
    "pb_peer_status": ([_P, ctypes.POINTER(ctypes.c_uint)], _I),
    "pb_peer_reduce_scatter": ([_P, _P, _P, _I, _P], _I),
    "pb_peer_all_gather": ([_P, _P, _P, _I, _I, _P], _I),
    "pb_comm_attach_peer": ([_P, _P], _I),
    "pb_comm_init_local": ([_I, _I, ctypes.POINTER(_P)], _I),
}

_lib = None


class PBError(RuntimeError):
    def __init__(self, fn, status, detail):
        super().__init__(f"{fn} failed with status {status}: {detail}")
        self.status = status


def lib():
    """Load libpb.so (raises if it was not built — there is no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise PBError("load", -1, f"{LIB_PATH} not built; run __graft_entry__.build()")
        L = ctypes.CDLL(LIB_PATH)
        for name, (args, res) in ABI_FUNCTIONS.items():
            fn = getattr(L, name)
            fn.argtypes = args
            fn.restype = res
        _lib = L
    return _lib


def pb_version():
    return lib().pb_version().decode()


def last_launch_count():
    return lib().pb_last_launch_count()


def _ptr(t, numel=None, name="tensor"):
    """Device pointer of a tensor argument (None -> NULL; an int is passed through as a
    raw address). The C side can only check a pointer's start (alignment, device,
    overlap), so the extent, dtype and layout are checked here: a CUDA, float32,
    contiguous tensor with at least `numel` elements."""
    if t is None:
        return None
    if isinstance(t, int):
        return t
    if not getattr(t, "is_cuda", False):
        raise PBError("argument", 1, f"{name} must be a CUDA tensor")
    import torch
    if t.dtype != torch.float32:
        raise PBError("argument", 1, f"{name} must be float32 (got {t.dtype})")
    if not t.is_contiguous():
        raise PBError("argument", 1, f"{name} must be contiguous (row-major, row pitch == #cols)")
    if numel is not None and t.numel() < numel:
        raise PBError("argument", 1, f"{name} has {t.numel()} elements, {numel} needed")
    return t.data_ptr()


def _stream(stream, ref=None):
    if stream is None:
        import torch
        dev = ref.device if ref is not None and hasattr(ref, "device") else None
        return torch.cuda.current_stream(dev).cuda_stream
    if isinstance(stream, int):
        return stream
    return stream.cuda_stream


def _check(name, st):
    if st != 0:
        raise PBError(name, st, lib().pb_last_error().decode())


def workspace_size(kernel: str, dims) -> int:
    arr = (ctypes.c_longlong * len(dims))(*[int(d) for d in dims])
    out = ctypes.c_size_t(0)
    _check("pb_workspace_size", lib().pb_workspace_size(kernel.encode(), arr, len(dims), ctypes.byref(out)))
    return out.value


def workspace(kernel: str, dims, device):
    import torch
    n = workspace_size(kernel, dims)
    return torch.empty(max(n, 256), dtype=torch.uint8, device=device)


_ws_cache = {}
_ws_retired = []  # outgrown cached workspaces: never freed (a captured graph may still use them)


def _ws(ws, kernel, dims, ref, stream=None):
    """Caller's workspace, or a cached one per (device, stream): calls on different
    streams never share a buffer (pb.h: such calls are independent). An outgrown
    buffer is retired, not freed, so in-flight kernels and CUDA graphs captured
    with it stay valid."""
    if ws is None:
        import torch
        need = max(workspace_size(kernel, dims), 256)
        device = ref.device if hasattr(ref, "device") else torch.device("cuda", torch.cuda.current_device())
        key = (device, _stream(stream, ref))
        cur = _ws_cache.get(key)
        if cur is None or cur.numel() < need:
            if cur is not None:
                _ws_retired.append(cur)
            cur = torch.empty(need, dtype=torch.uint8, device=device)
            _ws_cache[key] = cur
        ws = cur
    if hasattr(ws, "data_ptr"):
        if not ws.is_cuda or not ws.is_contiguous():
            raise PBError("argument", 1, "ws must be a contiguous CUDA tensor")
        return ws.data_ptr(), ws.numel() * ws.element_size(), ws
    return ws, 1 << 62, ws


def pb_gemm(ni, nj, nk, alpha, beta, C, A, B, ws=None, stream=None):
    p, n, keep = _ws(ws, "gemm", (ni, nj, nk), C, stream)
    _check("pb_gemm", lib().pb_gemm(ni, nj, nk, alpha, beta, _ptr(C, ni*nj, "C"), _ptr(A, ni*nk, "A"), _ptr(B, nk*nj, "B"), p, n, _stream(stream, C)))


def pb_gemm_variant(variant, ni, nj, nk, alpha, beta, C, A, B, ws=None, stream=None):
    p, n, keep = _ws(ws, "gemm_variant", (ni, nj, nk), C, stream)
    _check("pb_gemm_variant", lib().pb_gemm_variant(variant, ni, nj, nk, alpha, beta, _ptr(C, ni*nj, "C"), _ptr(A, ni*nk, "A"), _ptr(B, nk*nj, "B"),
                                                    p, n, _stream(stream, C)))


def pb_2mm(ni, nj, nk, nl, alpha, beta, tmp, A, B, C, D, ws=None, stream=None):
    p, n, keep = _ws(ws, "2mm", (ni, nj, nk, nl), D, stream)
    _check("pb_2mm", lib().pb_2mm(ni, nj, nk, nl, alpha, beta, _ptr(tmp, ni*nj, "tmp"), _ptr(A, ni*nk, "A"), _ptr(B, nk*nj, "B"), _ptr(C, nj*nl, "C"), _ptr(D, ni*nl, "D"),
                                  p, n, _stream(stream, D)))


def pb_3mm(ni, nj, nk, nl, nm, E, A, B, F, C, D, G, ws=None, stream=None):
    p, n, keep = _ws(ws, "3mm", (ni, nj, nk, nl, nm), G, stream)
    _check("pb_3mm", lib().pb_3mm(ni, nj, nk, nl, nm, _ptr(E, ni*nj, "E"), _ptr(A, ni*nk, "A"), _ptr(B, nk*nj, "B"), _ptr(F, nj*nl, "F"), _ptr(C, nj*nm, "C"), _ptr(D, nm*nl, "D"),
                                  _ptr(G, ni*nl, "G"), p, n, _stream(stream, G)))


def pb_syrk(n_, m, alpha, beta, C, A, ws=None, stream=None):
    p, n, keep = _ws(ws, "syrk", (n_, m), C, stream)
    _check("pb_syrk", lib().pb_syrk(n_, m, alpha, beta, _ptr(C, n_*n_, "C"), _ptr(A, n_*m, "A"), p, n, _stream(stream, C)))


def pb_syr2k(n_, m, alpha, beta, C, A, B, ws=None, stream=None):
    p, n, keep = _ws(ws, "syr2k", (n_, m), C, stream)
    _check("pb_syr2k", lib().pb_syr2k(n_, m, alpha, beta, _ptr(C, n_*n_, "C"), _ptr(A, n_*m, "A"), _ptr(B, n_*m, "B"), p, n, _stream(stream, C)))


def pb_syrk_full(n_, m, alpha, beta, C, A, ws=None, stream=None):
    p, n, keep = _ws(ws, "syrk_full", (n_, m), C, stream)
    _check("pb_syrk_full", lib().pb_syrk_full(n_, m, alpha, beta, _ptr(C, n_*n_, "C"), _ptr(A, n_*m, "A"), p, n, _stream(stream, C)))


def pb_syr2k_full(n_, m, alpha, beta, C, A, B, ws=None, stream=None):
    p, n, keep = _ws(ws, "syr2k_full", (n_, m), C, stream)
    _check("pb_syr2k_full", lib().pb_syr2k_full(n_, m, alpha, beta, _ptr(C, n_*n_, "C"), _ptr(A, n_*m, "A"), _ptr(B, n_*m, "B"), p, n,
                                                _stream(stream, C)))


def pb_syrk_rows(n_, m, r0, r1, alpha, beta, C_blk, A, ws=None, stream=None):
    p, n, keep = _ws(ws, "syrk_rows", (n_, m, r0, r1), A, stream)
    _check("pb_syrk_rows", lib().pb_syrk_rows(n_, m, r0, r1, alpha, beta, _ptr(C_blk, (r1-r0)*n_, "C_blk"), _ptr(A, r1*m, "A"), p, n,
                                              _stream(stream, A)))


def pb_syr2k_rows(n_, m, r0, r1, alpha, beta, C_blk, A, B, ws=None, stream=None):
    p, n, keep = _ws(ws, "syr2k_rows", (n_, m, r0, r1), A, stream)
    _check("pb_syr2k_rows", lib().pb_syr2k_rows(n_, m, r0, r1, alpha, beta, _ptr(C_blk, (r1-r0)*n_, "C_blk"), _ptr(A, r1*m, "A"), _ptr(B, r1*m, "B"), p, n,
                                                _stream(stream, A)))


def pb_covariance(m, n_, float_n, data, cov, mean=None, ws=None, stream=None):
    p, n, keep = _ws(ws, "covariance", (m, n_), cov, stream)
    _check("pb_covariance", lib().pb_covariance(m, n_, float_n, _ptr(data, n_*m, "data"), _ptr(cov, m*m, "cov"), _ptr(mean, m, "mean"), p, n,
                                                _stream(stream, cov)))


def pb_correlation(m, n_, float_n, eps, data, corr, mean=None, stddev=None, ws=None, stream=None):
    p, n, keep = _ws(ws, "correlation", (m, n_), corr, stream)
    _check("pb_correlation", lib().pb_correlation(m, n_, float_n, eps, _ptr(data, n_*m, "data"), _ptr(corr, m*m, "corr"), _ptr(mean, m, "mean"),
                                                  _ptr(stddev, m, "stddev"), p, n, _stream(stream, corr)))


def pb_covariance_rows(m, n_, float_n, r0, r1, data, cov_blk, mean=None, ws=None, stream=None):
    p, n, keep = _ws(ws, "covariance_rows", (m, n_, r0, r1), cov_blk, stream)
    _check("pb_covariance_rows", lib().pb_covariance_rows(m, n_, float_n, r0, r1, _ptr(data, n_*m, "data"), _ptr(cov_blk, (r1-r0)*m, "cov_blk"),
                                                          _ptr(mean, m, "mean"), p, n, _stream(stream, cov_blk)))


def pb_correlation_rows(m, n_, float_n, eps, r0, r1, data, corr_blk, mean=None, stddev=None, ws=None, stream=None):
    p, n, keep = _ws(ws, "correlation_rows", (m, n_, r0, r1), corr_blk, stream)
    _check("pb_correlation_rows", lib().pb_correlation_rows(m, n_, float_n, eps, r0, r1, _ptr(data, n_*m, "data"), _ptr(corr_blk, (r1-r0)*m, "corr_blk"),
                                                            _ptr(mean, m, "mean"), _ptr(stddev, m, "stddev"), p, n, _stream(stream, corr_blk)))


def pb_atax(m, n_, A, x, y, tmp=None, ws=None, stream=None):
    p, n, keep = _ws(ws, "atax", (m, n_), y, stream)
    _check("pb_atax", lib().pb_atax(m, n_, _ptr(A, m*n_, "A"), _ptr(x, n_, "x"), _ptr(y, n_, "y"), _ptr(tmp, m, "tmp"), p, n, _stream(stream, y)))


def pb_bicg(m, n_, A, s, q, p_, r, ws=None, stream=None):
    p, n, keep = _ws(ws, "bicg", (m, n_), q, stream)
    _check("pb_bicg", lib().pb_bicg(m, n_, _ptr(A, n_*m, "A"), _ptr(s, m, "s"), _ptr(q, n_, "q"), _ptr(p_, m, "p_"), _ptr(r, n_, "r"), p, n, _stream(stream, q)))


def pb_mvt(n_, x1, x2, y_1, y_2, A, ws=None, stream=None):
    p, n, keep = _ws(ws, "mvt", (n_,), x1, stream)
    _check("pb_mvt", lib().pb_mvt(n_, _ptr(x1, n_, "x1"), _ptr(x2, n_, "x2"), _ptr(y_1, n_, "y_1"), _ptr(y_2, n_, "y_2"), _ptr(A, n_*n_, "A"), p, n, _stream(stream, x1)))


def pb_gesummv(n_, alpha, beta, A, B, tmp, x, y, ws=None, stream=None):
    p, n, keep = _ws(ws, "gesummv", (n_,), y, stream)
    _check("pb_gesummv", lib().pb_gesummv(n_, alpha, beta, _ptr(A, n_*n_, "A"), _ptr(B, n_*n_, "B"), _ptr(tmp, n_, "tmp"), _ptr(x, n_, "x"), _ptr(y, n_, "y"), p, n,
                                          _stream(stream, y)))


def pb_gesummv_rows(rows, n_, alpha, beta, A_blk, B_blk, tmp_blk, x, y_blk, ws=None, stream=None):
    p, n, keep = _ws(ws, "gesummv_rows", (rows, n_), A_blk, stream)
    _check("pb_gesummv_rows", lib().pb_gesummv_rows(rows, n_, alpha, beta, _ptr(A_blk, rows*n_, "A_blk"), _ptr(B_blk, rows*n_, "B_blk"), _ptr(tmp_blk, rows, "tmp_blk"),
                                                    _ptr(x, n_, "x"), _ptr(y_blk, rows, "y_blk"), p, n, _stream(stream, A_blk)))


def pb_matvec_partial(rows, cols, A_blk, v, base_row, rowdot, w, base_col, colpart, ws=None, stream=None):
    p, n, keep = _ws(ws, "matvec_partial", (rows, cols), A_blk, stream)
    _check("pb_matvec_partial", lib().pb_matvec_partial(rows, cols, _ptr(A_blk, rows*cols, "A_blk"), _ptr(v, cols, "v"), _ptr(base_row, rows, "base_row"),
                                                        _ptr(rowdot, rows, "rowdot"), _ptr(w, rows, "w"), _ptr(base_col, cols, "base_col"), _ptr(colpart, cols, "colpart"),
                                                        p, n, _stream(stream, A_blk)))


def _host_w(w, n):
    vals = [float(v) for v in (w.reshape(-1).tolist() if hasattr(w, "reshape") else w)]
    if len(vals) != n:
        raise ValueError(f"expected {n} weights, got {len(vals)}")
    return (_F * n)(*vals)


def pb_conv2d(ni, nj, w, A, B, stream=None):
    """w: 9 weights (host), w[(di+1)*3 + (dj+1)]."""
    _check("pb_conv2d", lib().pb_conv2d(ni, nj, _host_w(w, 9), _ptr(A, ni*nj, "A"), _ptr(B, ni*nj, "B"), _stream(stream, B)))


def pb_conv3d(ni, nj, nk, w, A, B, stream=None):
    """w: 27 weights (host), w[(di+1)*9 + (dj+1)*3 + (dk+1)]."""
    _check("pb_conv3d", lib().pb_conv3d(ni, nj, nk, _host_w(w, 27), _ptr(A, ni*nj*nk, "A"), _ptr(B, ni*nj*nk, "B"), _stream(stream, B)))


def pb_conv2d_variant(variant, ni, nj, w, A, B, stream=None):
    _check("pb_conv2d_variant", lib().pb_conv2d_variant(variant, ni, nj, _host_w(w, 9), _ptr(A, ni*nj, "A"), _ptr(B, ni*nj, "B"),
                                                        _stream(stream, B)))


def pb_conv3d_variant(variant, ni, nj, nk, w, A, B, stream=None):
    _check("pb_conv3d_variant", lib().pb_conv3d_variant(variant, ni, nj, nk, _host_w(w, 27), _ptr(A, ni*nj*nk, "A"), _ptr(B, ni*nj*nk, "B"),
                                                        _stream(stream, B)))


def pb_fdtd_2d(tmax, nx, ny, ex, ey, hz, fict, ws=None, stream=None):
    p, n, keep = _ws(ws, "fdtd_2d", (nx, ny), ex, stream)
    _check("pb_fdtd_2d", lib().pb_fdtd_2d(tmax, nx, ny, _ptr(ex, nx*ny, "ex"), _ptr(ey, nx*ny, "ey"), _ptr(hz, nx*ny, "hz"), _ptr(fict, max(tmax, 1), "fict"), p, n,
                                          _stream(stream, ex)))


def pb_gramschmidt(m, n_, A, R, Q, ws=None, stream=None):
    p, n, keep = _ws(ws, "gramschmidt", (m, n_), A, stream)
    _check("pb_gramschmidt", lib().pb_gramschmidt(m, n_, _ptr(A, m*n_, "A"), _ptr(R, n_*n_, "R"), _ptr(Q, m*n_, "Q"), p, n, _stream(stream, A)))


def pb_gramschmidt_variant(variant, m, n_, A, R, Q, ws=None, stream=None):
    p, n, keep = _ws(ws, "gramschmidt", (m, n_), A, stream)
    _check("pb_gramschmidt_variant", lib().pb_gramschmidt_variant(variant, m, n_, _ptr(A, m*n_, "A"), _ptr(R, n_*n_, "R"), _ptr(Q, m*n_, "Q"), p, n,
                                                                  _stream(stream, A)))


def pb_row_partition(rows, nranks, rank, triangular=False, align=1):
    b = ctypes.c_int(0)
    e = ctypes.c_int(0)
    _check("pb_row_partition", lib().pb_row_partition(rows, nranks, rank, int(triangular), align,
                                                      ctypes.byref(b), ctypes.byref(e)))
    return b.value, e.value


# --------------------------------------------------------------------- multi-GPU (include/pb.h)
class Comm:
    """A libpb communicator (an NCCL communicator + side stream inside libpb)."""

    def __init__(self, handle, nranks, rank):
        self.handle, self.nranks, self.rank = handle, nranks, rank

    def close(self):
        if self.handle:
            _check("pb_comm_destroy", lib().pb_comm_destroy(self.handle))
            self.handle = None


def pb_comm_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    _check("pb_comm_unique_id", lib().pb_comm_unique_id(ctypes.cast(buf, ctypes.c_void_p)))
    return buf.raw


def pb_comm_init(nranks, rank, uid: bytes) -> Comm:
    if len(uid) != 128:
        raise ValueError("unique id must be 128 bytes")
    buf = ctypes.create_string_buffer(uid, 128)
    h = ctypes.c_void_p()
    _check("pb_comm_init", lib().pb_comm_init(nranks, rank, ctypes.cast(buf, ctypes.c_void_p), ctypes.byref(h)))
    return Comm(h.value, nranks, rank)


def pb_comm_destroy(comm: Comm):
    comm.close()


def _first(*ts):
    return next(t for t in ts if t is not None and hasattr(t, "device"))


def _dws(ws, name, dims, comm, *ts, stream=None):
    return _ws(ws, name + "_dist", tuple(dims) + (comm.nranks, comm.rank), _first(*ts), stream)


def pb_gemm_dist(comm, ni, nj, nk, alpha, beta, C_blk, A_blk, B, ws=None, stream=None):
    p, n, keep = _dws(ws, "gemm", (ni, nj, nk), comm, B, stream=stream)
    _check("pb_gemm_dist", lib().pb_gemm_dist(comm.handle, ni, nj, nk, alpha, beta, _ptr(C_blk, None, "C_blk"), _ptr(A_blk, None, "A_blk"),
                                              _ptr(B, None, "B"), p, n, _stream(stream, B)))


def pb_2mm_dist(comm, ni, nj, nk, nl, alpha, beta, tmp_blk, A_blk, B, C, D_blk, ws=None, stream=None):
    p, n, keep = _dws(ws, "2mm", (ni, nj, nk, nl), comm, B, stream=stream)
    _check("pb_2mm_dist", lib().pb_2mm_dist(comm.handle, ni, nj, nk, nl, alpha, beta, _ptr(tmp_blk, None, "tmp_blk"), _ptr(A_blk, None, "A_blk"),
                                            _ptr(B, None, "B"), _ptr(C, None, "C"), _ptr(D_blk, None, "D_blk"), p, n, _stream(stream, B)))


def pb_3mm_dist(comm, ni, nj, nk, nl, nm, E_blk, A_blk, B, F, C_blk, D, G_blk, ws=None, stream=None):
    p, n, keep = _dws(ws, "3mm", (ni, nj, nk, nl, nm), comm, F, stream=stream)
    _check("pb_3mm_dist", lib().pb_3mm_dist(comm.handle, ni, nj, nk, nl, nm, _ptr(E_blk, None, "E_blk"), _ptr(A_blk, None, "A_blk"), _ptr(B, None, "B"),
                                            _ptr(F, None, "F"), _ptr(C_blk, None, "C_blk"), _ptr(D, None, "D"), _ptr(G_blk, None, "G_blk"), p, n, _stream(stream, F)))


def pb_covariance_dist(comm, m, n_, float_n, data_blk, cov_blk, mean=None, ws=None, stream=None):
    p, n, keep = _dws(ws, "covariance", (m, n_), comm, data_blk, cov_blk, mean, stream=stream)
    _check("pb_covariance_dist", lib().pb_covariance_dist(comm.handle, m, n_, float_n, _ptr(data_blk, None, "data_blk"),
                                                          _ptr(cov_blk, None, "cov_blk"), _ptr(mean, m, "mean"), p, n,
                                                          _stream(stream, _first(data_blk, cov_blk, mean))))


def pb_correlation_dist(comm, m, n_, float_n, eps, data_blk, corr_blk, mean=None, stddev=None, ws=None, stream=None):
    p, n, keep = _dws(ws, "correlation", (m, n_), comm, data_blk, corr_blk, mean, stream=stream)
    _check("pb_correlation_dist", lib().pb_correlation_dist(comm.handle, m, n_, float_n, eps, _ptr(data_blk, None, "data_blk"),
                                                            _ptr(corr_blk, None, "corr_blk"), _ptr(mean, m, "mean"),
                                                            _ptr(stddev, m, "stddev"), p, n,
                                                            _stream(stream, _first(data_blk, corr_blk, mean))))


def pb_syrk_dist(comm, n_, m, alpha, beta, C_blk, A, ws=None, stream=None):
    p, n, keep = _dws(ws, "syrk", (n_, m), comm, A, stream=stream)
    _check("pb_syrk_dist", lib().pb_syrk_dist(comm.handle, n_, m, alpha, beta, _ptr(C_blk, None, "C_blk"), _ptr(A, None, "A"), p, n,
                                              _stream(stream, A)))


def pb_syr2k_dist(comm, n_, m, alpha, beta, C_blk, A, B, ws=None, stream=None):
    p, n, keep = _dws(ws, "syr2k", (n_, m), comm, A, stream=stream)
    _check("pb_syr2k_dist", lib().pb_syr2k_dist(comm.handle, n_, m, alpha, beta, _ptr(C_blk, None, "C_blk"), _ptr(A, None, "A"), _ptr(B, None, "B"),
                                                p, n, _stream(stream, A)))


def pb_atax_dist(comm, m, n_, A_blk, x, y_blk, tmp_blk=None, ws=None, stream=None):
    p, n, keep = _dws(ws, "atax", (m, n_), comm, x, stream=stream)
    _check("pb_atax_dist", lib().pb_atax_dist(comm.handle, m, n_, _ptr(A_blk, None, "A_blk"), _ptr(x, None, "x"), _ptr(y_blk, None, "y_blk"), _ptr(tmp_blk, None, "tmp_blk"),
                                              p, n, _stream(stream, x)))


def pb_bicg_dist(comm, m, n_, A_blk, s_blk, q_blk, p_, r_blk, ws=None, stream=None):
    p, n, keep = _dws(ws, "bicg", (m, n_), comm, p_, stream=stream)
    _check("pb_bicg_dist", lib().pb_bicg_dist(comm.handle, m, n_, _ptr(A_blk, None, "A_blk"), _ptr(s_blk, None, "s_blk"), _ptr(q_blk, None, "q_blk"), _ptr(p_, None, "p_"),
                                              _ptr(r_blk, None, "r_blk"), p, n, _stream(stream, p_)))


def pb_mvt_dist(comm, n_, x1_blk, x2_blk, y_1, y_2_blk, A_blk, ws=None, stream=None):
    p, n, keep = _dws(ws, "mvt", (n_,), comm, y_1, stream=stream)
    _check("pb_mvt_dist", lib().pb_mvt_dist(comm.handle, n_, _ptr(x1_blk, None, "x1_blk"), _ptr(x2_blk, None, "x2_blk"), _ptr(y_1, None, "y_1"), _ptr(y_2_blk, None, "y_2_blk"),
                                            _ptr(A_blk, None, "A_blk"), p, n, _stream(stream, y_1)))


def pb_gesummv_dist(comm, n_, alpha, beta, A_blk, B_blk, tmp_blk, x, y_blk, ws=None, stream=None):
    p, n, keep = _dws(ws, "gesummv", (n_,), comm, x, stream=stream)
    _check("pb_gesummv_dist", lib().pb_gesummv_dist(comm.handle, n_, alpha, beta, _ptr(A_blk, None, "A_blk"), _ptr(B_blk, None, "B_blk"),
                                                    _ptr(tmp_blk, None, "tmp_blk"), _ptr(x, None, "x"), _ptr(y_blk, None, "y_blk"), p, n, _stream(stream, x)))


class Peer:
    """A libpb peer group: one symmetric device buffer per rank, mapped into every
    rank with CUDA IPC (include/pb.h, pb_peer_*)."""

    def __init__(self, handle, nranks, rank, ipc_handle):
        self.handle, self.nranks, self.rank, self.ipc_handle = handle, nranks, rank, ipc_handle

    def open(self, handles: bytes):
        buf = ctypes.create_string_buffer(handles, len(handles))
        _check("pb_peer_open", lib().pb_peer_open(self.handle, ctypes.cast(buf, ctypes.c_void_p)))

    def status(self) -> int:
        v = ctypes.c_uint(0)
        _check("pb_peer_status", lib().pb_peer_status(self.handle, ctypes.byref(v)))
        return v.value

    def reduce_scatter(self, partial, out_blk, total, stream=None):
        _check("pb_peer_reduce_scatter", lib().pb_peer_reduce_scatter(self.handle, _ptr(partial, None, "partial"), _ptr(out_blk, None, "out_blk"),
                                                                      total, _stream(stream, partial)))

    def all_gather(self, send_blk, recv, rows, cols, stream=None):
        _check("pb_peer_all_gather", lib().pb_peer_all_gather(self.handle, _ptr(send_blk, None, "send_blk"), _ptr(recv, None, "recv"), rows, cols,
                                                              _stream(stream, recv)))

    def close(self):
        if self.handle:
            _check("pb_peer_destroy", lib().pb_peer_destroy(self.handle))
            self.handle = None


def pb_peer_create(nranks, rank, data_bytes) -> Peer:
    h = ctypes.c_void_p()
    buf = ctypes.create_string_buffer(64)
    _check("pb_peer_create", lib().pb_peer_create(nranks, rank, data_bytes, ctypes.byref(h),
                                                  ctypes.cast(buf, ctypes.c_void_p)))
    return Peer(h.value, nranks, rank, buf.raw)


def pb_comm_init_local(nranks, rank) -> Comm:
    h = ctypes.c_void_p()
    _check("pb_comm_init_local", lib().pb_comm_init_local(nranks, rank, ctypes.byref(h)))
    return Comm(h.value, nranks, rank)


def pb_comm_attach_peer(comm: Comm, peer: Peer):
    _check("pb_comm_attach_peer", lib().pb_comm_attach_peer(comm.handle, peer.handle if peer else None))
