"""GPU-vs-oracle parity harness (test infrastructure; imports oracle/).

Inputs come from pbgen (host C generator) — never from the CUDA path — and
are uploaded to the GPU; the CUDA path runs through the C ABI
(paper_2312_13170_b200 binding) and its outputs are compared element by
element with the fp64 oracle using the componentwise relative error of
reading R8:

    err = max_e |g_e - r_e| / s_e,  s_e = oracle evaluated on |terms|  (0/0 := 0)

TOL = 1e-4 is BASELINE.json north_star's "max relative error 1e-4".
"""
from __future__ import annotations

import numpy as np
import torch

import oracle
import paper_2312_13170_b200 as pb
import pbgen

TOL = 1e-4
S = pbgen.STREAM


def cerr(g, r, s):
    g = np.asarray(g, np.float64)
    r = np.asarray(r, np.float64)
    s = np.asarray(s, np.float64)
    d = np.abs(g - r)
    with np.errstate(divide="ignore", invalid="ignore"):
        e = np.where(s > 0, d / np.where(s > 0, s, 1.0), np.where(d == 0, 0.0, np.inf))
    return float(e.max()) if e.size else 0.0


def H(rows, cols, stream, mode=pbgen.U01, scale=1.0, offset=0.0, seed=pbgen.SEED):
    return pbgen.gen_host(rows, cols, stream, seed=seed, mode=mode, scale=scale, offset=offset)


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def host(t):
    torch.cuda.synchronize()
    return t.cpu().numpy()


def _res(**errs):
    e = max(errs.values())
    return {"err": e, "ok": e <= TOL, "parts": errs}


# ---------------------------------------------------------------- contractions
def check_gemm(ni, nj, nk, alpha=1.5, beta=1.2, mode=pbgen.U01, seed=pbgen.SEED, variant=None):
    A, B, C = H(ni, nk, S["A"], mode, seed=seed), H(nk, nj, S["B"], mode, seed=seed), H(ni, nj, S["C"], mode, seed=seed)
    dC = dev(C)
    if variant is None:
        pb.pb_gemm(ni, nj, nk, alpha, beta, dC, dev(A), dev(B))
    else:
        pb.pb_gemm_variant(variant, ni, nj, nk, alpha, beta, dC, dev(A), dev(B))
    g = host(dC)
    r = oracle.gemm(alpha, beta, C, A, B)
    s = oracle.gemm(alpha, beta, C, A, B, absmode=True)
    out = _res(C=cerr(g, r, s))
    out["g"], out["r"] = g, r
    return out


def check_2mm(ni, nj, nk, nl, alpha=1.5, beta=1.2, mode=pbgen.U01):
    A, B = H(ni, nk, S["A"], mode), H(nk, nj, S["B"], mode)
    C, D = H(nj, nl, S["C"], mode), H(ni, nl, S["D"], mode)
    dtmp = torch.empty(ni, nj, device="cuda")
    dD = dev(D)
    pb.pb_2mm(ni, nj, nk, nl, alpha, beta, dtmp, dev(A), dev(B), dev(C), dD)
    t_r, D_r = oracle.mm2(alpha, beta, A, B, C, D)
    t_s, D_s = oracle.mm2(alpha, beta, A, B, C, D, absmode=True)
    return _res(tmp=cerr(host(dtmp), t_r, t_s), D=cerr(host(dD), D_r, D_s))


def check_3mm(ni, nj, nk, nl, nm, mode=pbgen.U01):
    A, B = H(ni, nk, S["A"], mode), H(nk, nj, S["B"], mode)
    C, D = H(nj, nm, S["C"], mode), H(nm, nl, S["D"], mode)
    dE, dF, dG = (torch.empty(*sh, device="cuda") for sh in ((ni, nj), (nj, nl), (ni, nl)))
    pb.pb_3mm(ni, nj, nk, nl, nm, dE, dev(A), dev(B), dF, dev(C), dev(D), dG)
    E_r, F_r, G_r = oracle.mm3(A, B, C, D)
    E_s, F_s, G_s = oracle.mm3(A, B, C, D, absmode=True)
    return _res(E=cerr(host(dE), E_r, E_s), F=cerr(host(dF), F_r, F_s), G=cerr(host(dG), G_r, G_s))


def check_syrk(n, m, alpha=1.5, beta=1.2, mode=pbgen.U01):
    A = H(n, m, S["A"], mode)
    C = H(n, n, S["C"], mode | pbgen.SYM)
    dC = dev(C)
    pb.pb_syrk(n, m, alpha, beta, dC, dev(A))
    g = host(dC)
    r = oracle.syrk(alpha, beta, C, A)
    s = oracle.syrk(alpha, beta, C, A, absmode=True)
    up = np.triu_indices(n, 1)
    out = _res(C=cerr(g, r, s))
    out["upper_untouched"] = bool(np.array_equal(g[up], C[up]))
    out["ok"] = out["ok"] and out["upper_untouched"]
    return out


def check_syr2k(n, m, alpha=1.5, beta=1.2, mode=pbgen.U01):
    A, B = H(n, m, S["A"], mode), H(n, m, S["B"], mode)
    C = H(n, n, S["C"], mode | pbgen.SYM)
    dC = dev(C)
    pb.pb_syr2k(n, m, alpha, beta, dC, dev(A), dev(B))
    g = host(dC)
    r = oracle.syr2k(alpha, beta, C, A, B)
    s = oracle.syr2k(alpha, beta, C, A, B, absmode=True)
    up = np.triu_indices(n, 1)
    out = _res(C=cerr(g, r, s))
    out["upper_untouched"] = bool(np.array_equal(g[up], C[up]))
    out["ok"] = out["ok"] and out["upper_untouched"]
    return out


def check_syrk_full(n, m, two=False, alpha=1.5, beta=1.2, mode=pbgen.U01):
    """Full-matrix syrk / syr2k (SYCL-Bench form, reading R3): every C[i][j], with a
    NON-symmetric C. Reference: the gemm oracle (the plain definition) with B = A^T
    (syr2k: the sum of the B A^T and A B^T products), plus the symmetry of the
    product part."""
    A, B = H(n, m, S["A"], mode), H(n, m, S["B"], mode)
    C = H(n, n, S["C"], mode)
    dC, dA, dB = dev(C), dev(A), dev(B)
    if two:
        pb.pb_syr2k_full(n, m, alpha, beta, dC, dA, dB)
        z = np.zeros((n, n), np.float32)
        r = oracle.gemm(alpha, beta, C, B, A.T) + oracle.gemm(alpha, 0.0, z, A, B.T)
        s = oracle.gemm(alpha, beta, C, B, A.T, absmode=True) + oracle.gemm(alpha, 0.0, z, A, B.T, absmode=True)
    else:
        pb.pb_syrk_full(n, m, alpha, beta, dC, dA)
        r = oracle.gemm(alpha, beta, C, A, A.T)
        s = oracle.gemm(alpha, beta, C, A, A.T, absmode=True)
    g = host(dC)
    out = _res(C=cerr(g, r, s))
    # property: the product part (g - beta C) is symmetric (each entry computed independently
    # by a different tile; plans differ from the lower-only kernel, so no bitwise pin)
    P_ = g.astype(np.float64) - beta * C.astype(np.float64)
    Ps = s - abs(beta) * np.abs(C.astype(np.float64))
    out["symmetry"] = float(np.max(np.abs(P_ - P_.T) / np.maximum(Ps, 1e-30)))
    out["ok"] = out["ok"] and out["symmetry"] <= 2 * TOL
    return out


def structured_data(n, m, seed=pbgen.SEED):
    """data n x m ~ U[0,1) with the parity columns of DESIGN.md's input recipe:
    col 0 constant 0.5; col 2 = col 1 (duplicate); col 3 = 1 - col 1 (negated);
    col 4 ~ U[0, 1/64) (stddev <= eps)."""
    d = H(n, m, S["data"], seed=seed)
    if m >= 5:
        d[:, 0] = 0.5
        d[:, 2] = d[:, 1]
        d[:, 3] = np.float32(1.0) - d[:, 1]
        d[:, 4] = pbgen.gen_host(n, 1, 15, seed=seed, scale=1.0 / 64)[:, 0]
    return d


def check_covariance(m, n, structured=True, float_n=None):
    data = structured_data(n, m) if structured else H(n, m, S["data"])
    fn = float(n) if float_n is None else float(float_n)
    dcov = torch.empty(m, m, device="cuda")
    dmean = torch.empty(m, device="cuda")
    ddata = dev(data)
    pb.pb_covariance(m, n, fn, ddata, dcov, dmean)
    cov_r, mean_r = oracle.covariance(fn, data)
    cov_s, mean_s = oracle.covariance(fn, data, absmode=True)
    g = host(dcov)
    out = _res(cov=cerr(g, cov_r, cov_s), mean=cerr(host(dmean), mean_r, mean_s))
    out["symmetric"] = bool(np.array_equal(g, g.T))
    out["data_untouched"] = bool(np.array_equal(host(ddata), data))
    if structured and m >= 5 and float_n is None:  # with float_n != n the "mean" is not the mean
        out["const_col_zero"] = bool(np.all(g[0, :] == 0) and np.all(g[:, 0] == 0))
    else:
        out["const_col_zero"] = True
    out["ok"] = out["ok"] and out["symmetric"] and out["data_untouched"] and out["const_col_zero"]
    return out


def check_correlation(m, n, eps=0.1, structured=True, float_n=None):
    data = structured_data(n, m) if structured else H(n, m, S["data"])
    fn = float(n) if float_n is None else float(float_n)
    dcorr = torch.empty(m, m, device="cuda")
    dmean = torch.empty(m, device="cuda")
    dsd = torch.empty(m, device="cuda")
    pb.pb_correlation(m, n, fn, eps, dev(data), dcorr, dmean, dsd)
    c_r, m_r, sd_r = oracle.correlation(fn, eps, data)
    c_s, m_s, sd_s = oracle.correlation(fn, eps, data, absmode=True)
    g = host(dcorr)
    out = _res(corr=cerr(g, c_r, c_s), mean=cerr(host(dmean), m_r, m_s), stddev=cerr(host(dsd), sd_r, sd_r))
    out["diag_one"] = bool(np.all(np.diag(g) == 1.0))
    out["symmetric"] = bool(np.array_equal(g, g.T))
    out["ok"] = out["ok"] and out["diag_one"] and out["symmetric"]
    return out


# ---------------------------------------------------------------- matrix-vector
def check_atax(m, n):
    A, x = H(m, n, S["A"]), H(1, n, S["x"])[0]
    dy, dt = torch.empty(n, device="cuda"), torch.empty(m, device="cuda")
    pb.pb_atax(m, n, dev(A), dev(x), dy, dt)
    y_r, t_r = oracle.atax(A, x)
    y_s, t_s = oracle.atax(A, x, absmode=True)
    return _res(y=cerr(host(dy), y_r, y_s), tmp=cerr(host(dt), t_r, t_s))


def check_bicg(m, n):
    A, p, r = H(n, m, S["A"]), H(1, m, S["p"])[0], H(1, n, S["r"])[0]
    ds, dq = torch.empty(m, device="cuda"), torch.empty(n, device="cuda")
    pb.pb_bicg(m, n, dev(A), ds, dq, dev(p), dev(r))
    s_r, q_r = oracle.bicg(A, p, r)
    s_s, q_s = oracle.bicg(A, p, r, absmode=True)
    return _res(s=cerr(host(ds), s_r, s_s), q=cerr(host(dq), q_r, q_s))


def check_mvt(n):
    A = H(n, n, S["A"])
    x1, x2 = H(1, n, S["x1"])[0], H(1, n, S["x2"])[0]
    y1, y2 = H(1, n, S["y_1"])[0], H(1, n, S["y_2"])[0]
    d1, d2 = dev(x1), dev(x2)
    pb.pb_mvt(n, d1, d2, dev(y1), dev(y2), dev(A))
    o1, o2 = oracle.mvt(x1, x2, y1, y2, A)
    s1, s2 = oracle.mvt(x1, x2, y1, y2, A, absmode=True)
    return _res(x1=cerr(host(d1), o1, s1), x2=cerr(host(d2), o2, s2))


def check_gesummv(n, alpha=1.5, beta=1.2):
    A, B, x = H(n, n, S["A"]), H(n, n, S["B"]), H(1, n, S["x"])[0]
    dt, dy = torch.empty(n, device="cuda"), torch.empty(n, device="cuda")
    pb.pb_gesummv(n, alpha, beta, dev(A), dev(B), dt, dev(x), dy)
    t_r, y_r = oracle.gesummv(alpha, beta, A, B, x)
    t_s, y_s = oracle.gesummv(alpha, beta, A, B, x, absmode=True)
    return _res(tmp=cerr(host(dt), t_r, t_s), y=cerr(host(dy), y_r, y_s))


# ---------------------------------------------------------------- stencils (NEXT-3)
def _border_mask(shape):
    m = np.ones(shape, bool)
    m[(slice(1, -1),) * len(shape)] = False
    return m


def check_conv2d(ni, nj, w=None, seed=pbgen.SEED):
    w = pbgen.CONV2D_W if w is None else list(w)
    A = H(ni, nj, S["A"], seed=seed)
    B0 = H(ni, nj, S["B"], seed=seed)
    dB = dev(B0)
    pb.pb_conv2d(ni, nj, w, dev(A), dB)
    g = host(dB)
    r, s = oracle.conv2d(w, A, B0), oracle.conv2d(w, A, B0, absmode=True)
    border_ok = bool(np.array_equal(g[_border_mask(g.shape)].view(np.uint32), B0[_border_mask(g.shape)].view(np.uint32)))
    out = _res(B=cerr(g, r, s) if border_ok else float("inf"))
    out["border_bitwise"] = border_ok
    return out


def check_conv3d(ni, nj, nk, w=None, seed=pbgen.SEED):
    w = pbgen.conv3d_w27() if w is None else list(w)
    A = H(ni * nj, nk, S["A"], seed=seed).reshape(ni, nj, nk)
    B0 = H(ni * nj, nk, S["B"], seed=seed).reshape(ni, nj, nk)
    dB = dev(B0)
    pb.pb_conv3d(ni, nj, nk, w, dev(A), dB)
    g = host(dB)
    r, s = oracle.conv3d(w, A, B0), oracle.conv3d(w, A, B0, absmode=True)
    m = _border_mask(g.shape)
    border_ok = bool(np.array_equal(g[m].view(np.uint32), B0[m].view(np.uint32)))
    out = _res(B=cerr(g, r, s) if border_ok else float("inf"))
    out["border_bitwise"] = border_ok
    return out


def fdtd_inputs(nx, ny, tmax, seed=pbgen.SEED):
    return (H(nx, ny, S["ex"], seed=seed), H(nx, ny, S["ey"], seed=seed), H(nx, ny, S["hz"], seed=seed),
            H(1, max(tmax, 1), S["fict"], seed=seed).reshape(-1))


FDTD_TOL = 1e-4  # fp64 check: |g - r| <= FDTD_TOL * max|r| (reading R21); the fp32 check is bitwise


def check_fdtd2d(nx, ny, tmax, seed=pbgen.SEED):
    ex, ey, hz, f = fdtd_inputs(nx, ny, tmax, seed)
    d = [dev(a) for a in (ex, ey, hz)]
    pb.pb_fdtd_2d(tmax, nx, ny, d[0], d[1], d[2], dev(f))
    g = [host(t) for t in d]
    r32 = oracle.fdtd2d(tmax, ex, ey, hz, f, f32=True)
    r64 = oracle.fdtd2d(tmax, ex, ey, hz, f)
    bitwise = all(np.array_equal(a.view(np.uint32), b.view(np.uint32)) for a, b in zip(g, r32))
    scale = max(float(np.abs(a).max()) for a in r64)
    e64 = max(float(np.abs(a.astype(np.float64) - b).max()) for a, b in zip(g, r64)) / scale
    return {"err": e64, "ok": bool(bitwise and e64 <= FDTD_TOL), "bitwise_f32": bitwise,
            "parts": {"rel_to_max_f64": e64}}


def check_gramschmidt(m, n, seed=pbgen.SEED):
    """Reading R22: Q and the final A columnwise against max|column| of the oracle's,
    R[k][j] against ||A_in[:, j]||_2 (a bound on |R[k][j]|); R's strict lower
    triangle must keep its input bitwise."""
    A = H(m, n, S["A"], seed=seed)
    R0 = H(n, n, S["B"], seed=seed)
    dA, dR, dQ = dev(A), dev(R0), torch.zeros(m, n, device="cuda")
    pb.pb_gramschmidt(m, n, dA, dR, dQ)
    gA, gR, gQ = host(dA), host(dR), host(dQ)
    rA, rR, rQ = oracle.gramschmidt(A)
    low = np.tril(np.ones((n, n), bool), -1)
    lower_ok = bool(np.array_equal(gR[low].view(np.uint32), R0[low].view(np.uint32)))
    colA = np.abs(rA).max(0)
    colQ = np.abs(rQ).max(0)
    cn = np.sqrt((A.astype(np.float64) ** 2).sum(0))
    eA = float((np.abs(gA - rA) / colA[None, :]).max())
    eQ = float((np.abs(gQ - rQ) / colQ[None, :]).max())
    up = ~low
    eR = float((np.abs(gR - rR) / cn[None, :])[up].max())
    out = _res(A=eA, Q=eQ, R=eR if lower_ok else float("inf"))
    out["lower_untouched"] = lower_ok
    return out


def check_all_small(n=132, seed=pbgen.SEED):
    """One ragged-size pass over the eleven kernels and the three stencils (used by smoke())."""
    m = n + 4
    return {
        "gemm": check_gemm(n + 3, n - 4, m),
        "2mm": check_2mm(n + 1, n, m, n - 8),
        "3mm": check_3mm(n - 3, n, m, n + 4, n - 4),
        "syrk": check_syrk(n, m),
        "syr2k": check_syr2k(n, m),
        "covariance": check_covariance(n, m + 1),
        "correlation": check_correlation(n, m + 1),
        "atax": check_atax(m + 1, n),
        "bicg": check_bicg(n, m + 1),
        "mvt": check_mvt(n),
        "gesummv": check_gesummv(n),
        "conv2d": check_conv2d(n + 5, n),
        "conv3d": check_conv3d(n // 4 + 3, n // 4 + 5, n),
        "fdtd_2d": check_fdtd2d(n - 3, n, 7),
        "gramschmidt": check_gramschmidt(n + 7, n - 5),
    }
