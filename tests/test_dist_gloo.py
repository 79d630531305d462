"""World-size-2 (and 3) gloo tests of the row-block data-parallel layer
(paper_2312_13170_b200.dist) on CPU: partitions, the 3mm all-gather, the
reduce-scatter of transposed-product partials and mvt's base folding. The
per-shard arithmetic is supplied by an oracle-backed stand-in for the kernel
namespace (test infrastructure only; on GPUs the same code calls libpb), and
the reassembled sharded results must equal the single-process oracle.
"""
import os
import socket
import types

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
import paper_2312_13170_b200 as pb
import pbgen
from paper_2312_13170_b200 import dist as D


def _np(t):
    return t.detach().cpu().numpy()


def host_all_gather_rows(full, local, world, bounds):
    """full[rows] <- concat of every rank's `local` row block (gloo, host-staged; test only)."""
    rank = dist.get_rank()
    sizes = [e - b for b, e in bounds]
    mx = max(sizes)
    pad = torch.zeros((mx,) + tuple(local.shape[1:]), dtype=local.dtype)
    pad[: sizes[rank]].copy_(local[: sizes[rank]].cpu())
    bufs = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(bufs, pad)
    for g, (b, e) in enumerate(bounds):
        full[b:e].copy_(bufs[g][: e - b])


def host_reduce_scatter_vec(out_local, partial, world, bounds):
    """out_local <- (sum over ranks of partial)[bounds[rank]] (gloo, host-staged; test only)."""
    h = partial.cpu().clone()
    dist.all_reduce(h)
    b, e = bounds[dist.get_rank()]
    out_local.copy_(h[b:e])


def fake_kernels():
    """Oracle-backed CPU stand-ins with the binding's signatures (test only)."""
    K = types.SimpleNamespace()
    K.pb_row_partition = pb.pb_row_partition  # host-only C ABI entry point
    K.last_launch_count = lambda: 1

    def gemm(ni, nj, nk, alpha, beta, C, A, B, ws=None):
        if beta == 0:  # ABI: beta == 0 means C is not read (BLAS convention)
            C.zero_()
        C.copy_(torch.from_numpy(oracle.gemm(alpha, beta, _np(C), _np(A), _np(B)).astype(np.float32)))

    def mm2(ni, nj, nk, nl, alpha, beta, tmp, A, B, C, Dm, ws=None):
        t, d = oracle.mm2(alpha, beta, _np(A), _np(B), _np(C), _np(Dm))
        if tmp is not None:
            tmp.copy_(torch.from_numpy(t.astype(np.float32)))
        Dm.copy_(torch.from_numpy(d.astype(np.float32)))

    def matvec_partial(rows, cols, A, v, base_row, rowdot, w, base_col, colpart, ws=None):
        a = _np(A).astype(np.float64)
        if v is not None:
            r = a @ _np(v).astype(np.float64)
            if base_row is not None:
                r = r + _np(base_row)
            rowdot.copy_(torch.from_numpy(r.astype(np.float32)))
        if w is not None:
            c = a.T @ _np(w).astype(np.float64)
            if base_col is not None:
                c = c + _np(base_col)
            colpart.copy_(torch.from_numpy(c.astype(np.float32)))

    def syrk_rows(n, m, r0, r1, alpha, beta, C_blk, A, ws=None, B=None):
        full = np.zeros((n, n), np.float32)
        full[r0:r1] = _np(C_blk)
        if B is None:
            out = oracle.syrk(alpha, beta, full, _np(A))
        else:
            out = oracle.syr2k(alpha, beta, full, _np(A), _np(B))
        C_blk.copy_(torch.from_numpy(out[r0:r1].astype(np.float32)))

    def gesummv_rows(rows, n, alpha, beta, A, B, tmp, x, y, ws=None):
        t, yy = oracle.gesummv(alpha, beta, _np(A), _np(B), _np(x)) if rows == n else (None, None)
        a, b, xx = _np(A).astype(np.float64), _np(B).astype(np.float64), _np(x).astype(np.float64)
        y.copy_(torch.from_numpy((alpha * (a @ xx) + beta * (b @ xx)).astype(np.float32)))
        if tmp is not None:
            tmp.copy_(torch.from_numpy((a @ xx).astype(np.float32)))

    def atax(m, n, A, x, y, tmp, ws=None):  # tmp = A x; y = A^T tmp (A: this rank's rows)
        a, xx = _np(A).astype(np.float64), _np(x).astype(np.float64)
        t = a @ xx
        y.copy_(torch.from_numpy((a.T @ t).astype(np.float32)))
        if tmp is not None:
            tmp.copy_(torch.from_numpy(t.astype(np.float32)))

    K.pb_atax = atax
    K.pb_gemm = gemm
    K.pb_2mm = mm2
    K.pb_matvec_partial = matvec_partial
    K.all_gather_rows = host_all_gather_rows
    K.reduce_scatter_vec = host_reduce_scatter_vec
    K.pb_syrk_rows = lambda n, m, r0, r1, al, be, C, A, ws=None: syrk_rows(n, m, r0, r1, al, be, C, A)
    K.pb_syr2k_rows = lambda n, m, r0, r1, al, be, C, A, B, ws=None: syrk_rows(n, m, r0, r1, al, be, C, A, B=B)
    K.pb_gesummv_rows = gesummv_rows
    return K


def H(r, c, s, **kw):
    return torch.from_numpy(pbgen.gen_host(r, c, s, **kw))


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        K = fake_kernels()
        res = {}
        # ---- 3mm: F row blocks + all-gather, E/G local rows
        n = 384
        r0, r1 = D.partition(n, world, rank, False, 128, K)
        A, B, C, Dm = H(n, n, 1), H(n, n, 2), H(n, n, 3), H(n, n, 4)
        E, G, F = torch.empty(r1 - r0, n), torch.empty(r1 - r0, n), torch.empty(n, n)
        f0, f1 = r0, r1
        Fl = torch.empty(f1 - f0, n)
        D.mm3_rows(None, n, E, A[r0:r1].contiguous(), B, Fl, F, C, Dm, G, None, K=K)
        res["3mm_G"] = (r0, r1, _np(G))
        res["3mm_F"] = _np(F)
        # ---- 2mm: row-local
        tmp = torch.empty(r1 - r0, n)
        D2 = H(n, n, 4)[r0:r1].contiguous()
        D.mm2_rows(None, n, 1.5, 1.2, tmp, A[r0:r1].contiguous(), B, C, D2, None, K=K)
        res["2mm_D"] = (r0, r1, _np(D2))
        # ---- syrk / syr2k triangular bands
        n2, m2 = 384, 40
        s0, s1 = D.partition(n2, world, rank, 2, 256, K)
        A2, B2 = H(n2, m2, 1), H(n2, m2, 2)
        Cfull = H(n2, n2, 3, mode=pbgen.SYM)
        Cb = Cfull[s0:s1].clone()
        Cb2 = Cfull[s0:s1].clone()
        D.syrk_rows(None, n2, m2, 1.5, 1.2, Cb, A2, None, K=K)
        D.syrk_rows(None, n2, m2, 1.5, 1.2, Cb2, A2, None, B=B2, K=K)
        res["syrk"] = (s0, s1, _np(Cb))
        res["syr2k"] = (s0, s1, _np(Cb2))
        # ---- matvec family: row blocks + reduce-scatter
        nv = 96
        v0, v1 = D.partition(nv, world, rank, False, 4, K)
        Av, Bv = H(nv, nv, 1), H(nv, nv, 2)
        vec = {k: H(1, nv, s)[0] for k, s in (("x", 6), ("r", 7), ("y2", 7), ("x1", 8), ("x2", 9))}
        for kern in ("atax", "bicg", "mvt", "gesummv"):
            v = dict(A=Av[v0:v1].contiguous(), B=Bv[v0:v1].contiguous(), x=vec["x"].clone(), r=vec["r"].clone(),
                     y2=vec["y2"].clone(), x1=vec["x1"].clone(), x2=vec["x2"].clone(), y=torch.zeros(nv),
                     s=torch.zeros(nv), q=torch.zeros(nv), yo=torch.zeros(nv), tmp=torch.zeros(v1 - v0))
            D.matvec(None, kern, nv, v, None, 1.5, 1.2, K=K)
            out = {"atax": v["y"], "bicg": v["s"], "mvt": v["x2"], "gesummv": v["yo"]}[kern]
            extra = {"bicg": v["q"], "mvt": v["x1"], "atax": v["tmp"], "gesummv": v["yo"]}[kern]
            res[kern] = (v0, v1, _np(out)[v0:v1], _np(extra))
        q.put((rank, res))
    finally:
        dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("world", [2, 3])
def test_dist_row_blocks_gloo(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = dict(q.get(timeout=300) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    n = 384
    A, B, C, Dm = (pbgen.gen_host(n, n, s) for s in (1, 2, 3, 4))
    E_r, F_r, G_r = oracle.mm3(A, B, C, Dm)
    t_r, D_r = oracle.mm2(1.5, 1.2, A, B, C, Dm)
    got_G = np.zeros((n, n), np.float32)
    got_D = np.zeros((n, n), np.float32)
    for r in range(world):
        r0, r1, g = out[r]["3mm_G"]
        got_G[r0:r1] = g
        r0, r1, d = out[r]["2mm_D"]
        got_D[r0:r1] = d
        assert np.allclose(out[r]["3mm_F"], F_r, rtol=1e-6)  # all-gather delivered all of F
    assert np.allclose(got_G, G_r, rtol=1e-5) and np.allclose(got_D, D_r, rtol=1e-6)
    n2, m2 = 384, 40
    A2, B2 = pbgen.gen_host(n2, m2, 1), pbgen.gen_host(n2, m2, 2)
    Cf = pbgen.gen_host(n2, n2, 3, mode=pbgen.SYM)
    for name, ref in (("syrk", oracle.syrk(1.5, 1.2, Cf, A2)), ("syr2k", oracle.syr2k(1.5, 1.2, Cf, A2, B2))):
        got = np.zeros((n2, n2), np.float32)
        covered = np.zeros(n2, bool)
        for r in range(world):
            s0, s1, blk = out[r][name]
            got[s0:s1] = blk
            covered[s0:s1] = True
        assert covered.all()
        assert np.allclose(got, ref, rtol=1e-6)
    nv = 96
    Av, Bv = pbgen.gen_host(nv, nv, 1), pbgen.gen_host(nv, nv, 2)
    x, rr, y2, x1, x2 = (pbgen.gen_host(1, nv, s)[0] for s in (6, 7, 7, 8, 9))
    refs = {"atax": oracle.atax(Av, x)[0], "bicg": oracle.bicg(Av, x, rr)[0],
            "mvt": oracle.mvt(x1, x2, x, y2, Av)[1], "gesummv": oracle.gesummv(1.5, 1.2, Av, Bv, x)[1]}
    for k, ref in refs.items():
        got = np.zeros(nv)
        for r in range(world):
            v0, v1, blk, _ = out[r][k]
            got[v0:v1] = blk
        assert np.allclose(got, ref, rtol=1e-5), k
    q_ref = oracle.bicg(Av, x, rr)[1]
    x1_ref = oracle.mvt(x1, x2, x, y2, Av)[0]
    for r in range(world):
        v0, v1, _, q = out[r]["bicg"]
        assert np.allclose(q[v0:v1], q_ref[v0:v1], rtol=1e-5)
        v0, v1, _, xx1 = out[r]["mvt"]
        assert np.allclose(xx1[v0:v1], x1_ref[v0:v1], rtol=1e-5)


def _covobs_worker(rank, world, port, q):
    """The observations-split covariance / correlation decomposition that
    pb_<k>_dist implements (k_covdist.cu, pb_dist.cu), emulated with gloo
    collectives on the host: the same partitions (libpb's pb_row_partition,
    observations align 32, output rows align 32), fp64 column sums gathered and
    added in rank order, local partial Grams of the centred block, a reduce-scatter
    of the m x m sum into row bands (test only: the CUDA steps are checked against
    the oracle on the GPU in tests/test_gpu_dist.py)."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from tests import parity as P
        m, n, eps = 36, 203, 0.1
        data = P.structured_data(n, m)
        o0, o1 = pb.pb_row_partition(n, world, rank, False, 32)
        b0, b1 = pb.pb_row_partition(m, world, rank, False, 32)
        X = data[o0:o1].astype(np.float64)
        sums = torch.from_numpy(np.stack([X.sum(0), (X * X).sum(0)]))  # [2][m]
        allsums = [torch.empty_like(sums) for _ in range(world)]
        dist.all_gather(allsums, sums)
        S1 = np.zeros(m)
        S2 = np.zeros(m)
        for g in range(world):  # rank order, as obs_center_t_kernel
            S1 += allsums[g][0].numpy()
            S2 += allsums[g][1].numpy()
        res = {}
        for corr in (False, True):
            mean = S1 / n
            inv = np.ones(m)
            if corr:
                sd = np.sqrt(np.maximum((S2 - 2 * mean * S1 + n * mean * mean) / n, 0.0))
                sd[sd <= eps] = 1.0
                inv = 1.0 / (np.sqrt(n) * sd)
            Y = (X - mean) * inv
            Pg = torch.from_numpy(Y.T @ Y)
            dist.all_reduce(Pg)  # reduce-scatter = sum, then this rank's row band
            band = Pg.numpy()[b0:b1].copy()
            if corr:
                for i in range(b0, b1):
                    band[i - b0, i] = 1.0
            else:
                band /= n - 1
            res[corr] = (b0, b1, band)
        q.put((rank, res))
    except Exception as e:
        q.put((rank, {"error": repr(e)}))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_cov_corr_observation_split_gloo(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_covobs_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = dict(q.get(timeout=300) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
    from tests import parity as P
    m, n = 36, 203
    data = P.structured_data(n, m)
    for corr in (False, True):
        got = np.zeros((m, m))
        for r in range(world):
            assert "error" not in out[r], out[r]
            b0, b1, band = out[r][corr]
            got[b0:b1] = band
        if corr:
            ref, sc = oracle.correlation(float(n), 0.1, data)[0], oracle.correlation(float(n), 0.1, data, absmode=True)[0]
        else:
            ref, sc = oracle.covariance(float(n), data)[0], oracle.covariance(float(n), data, absmode=True)[0]
        assert P.cerr(got, ref, sc) <= 1e-12, corr
