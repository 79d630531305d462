"""The row-block data-parallel layer (paper_2312_13170_b200.dist) with the REAL
libpb kernels: two ranks share cuda:0 over gloo (collectives staged through
the host), each computes its row shard through the C ABI, and the reassembled
results must match the single-process oracle. This exercises every N>1 code
path of the kernels' sharded entry points on the one GPU this build has; the
NCCL transport itself is only exercised on a multi-GPU box.
"""
import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import oracle  # noqa: E402
import pbgen  # noqa: E402
from tests import parity as P  # noqa: E402


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q, backend="gloo"):
    import torch.distributed as dist

    import paper_2312_13170_b200 as pb
    from paper_2312_13170_b200 import dist as D
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    if backend.startswith("nccl"):  # world size 1 kept on the sharded path
        os.environ["PB_FORCE_DIST"] = "1"
        dist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device("cuda", 0))
        # the pb_<k>_dist entry points: NCCL inside libpb, or NCCL + peer-memory collectives
        D.init_comm(transport="peer" if backend == "nccl-peer" else "nccl", peer_bytes=4 << 20)
    else:
        dist.init_process_group("gloo", rank=rank, world_size=world)
        if backend == "gloo-peer":  # local libpb comm: collectives = peer-memory kernels over CUDA IPC
            D.init_comm(transport="local", peer_bytes=4 << 20)
    K = pb
    if backend == "gloo":  # no libpb comm: the collectives are host-staged test stand-ins
        import types

        from tests.test_dist_gloo import host_all_gather_rows, host_reduce_scatter_vec
        K = types.SimpleNamespace(**{a: getattr(pb, a) for a in dir(pb) if a.startswith("pb_")})
        K.last_launch_count = pb.last_launch_count
        K.all_gather_rows, K.reduce_scatter_vec = host_all_gather_rows, host_reduce_scatter_vec
    dev = torch.device("cuda", 0)
    H = lambda r, c, s, **kw: torch.from_numpy(pbgen.gen_host(r, c, s, **kw)).to(dev)  # noqa: E731
    res = {}
    try:
        # 3mm: F row blocks + all-gather, E/G local rows
        n = 512
        r0, r1 = D.partition(n, world, rank, False, 128)
        A, B, C, Dm = H(n, n, 1), H(n, n, 2), H(n, n, 3), H(n, n, 4)
        E, G, F = (torch.empty(r1 - r0, n, device=dev), torch.empty(r1 - r0, n, device=dev),
                   torch.empty(n, n, device=dev))
        Fl = torch.empty(r1 - r0, n, device=dev)
        def wsz(*named):  # local and (with a libpb comm) "<k>_dist" workspaces
            need = max(pb.workspace_size(k, d) for k, d in named)
            if D.comm() is not None:
                for k, d in named:
                    if k in ("gemm", "2mm", "3mm", "syrk", "syr2k", "atax", "bicg", "mvt", "gesummv"):
                        need = max(need, pb.workspace_size(k + "_dist", tuple(d) + (world, rank)))
            return torch.empty(max(need, 256), dtype=torch.uint8, device=dev)
        ws = wsz(("3mm", (n, n, n, n, n)))
        D.mm3_rows(None, n, E, A[r0:r1].contiguous(), B, Fl, F, C, Dm, G, ws, K=K)
        # 2mm: row-local
        tmp = torch.empty(r1 - r0, n, device=dev)
        D2 = Dm[r0:r1].clone()
        D.mm2_rows(None, n, 1.5, 1.2, tmp, A[r0:r1].contiguous(), B, C, D2, wsz(("2mm", (n,) * 4)), K=K)
        torch.cuda.synchronize()
        res["3mm"] = (r0, r1, G.cpu().numpy(), F.cpu().numpy())
        res["2mm"] = (r0, r1, D2.cpu().numpy())
        # syrk / syr2k triangular bands
        n2, m2 = 768, 260
        s0, s1 = D.partition(n2, world, rank, 2, 256)
        A2, B2 = H(n2, m2, 1), H(n2, m2, 2)
        Cf = H(n2, n2, 3, mode=pbgen.SYM)
        Cb, Cb2 = Cf[s0:s1].clone(), Cf[s0:s1].clone()
        wsy = wsz(("syr2k_rows", (n2, m2, 0, n2)), ("syr2k", (n2, m2)))
        D.syrk_rows(None, n2, m2, 1.5, 1.2, Cb, A2, wsy, K=K)
        D.syrk_rows(None, n2, m2, 1.5, 1.2, Cb2, A2, wsy, B=B2, K=K)
        torch.cuda.synchronize()
        res["syrk"] = (s0, s1, Cb.cpu().numpy())
        res["syr2k"] = (s0, s1, Cb2.cpu().numpy())
        # matvec family
        nv = 2048
        v0, v1 = D.partition(nv, world, rank, False, 4)
        Av, Bv = H(nv, nv, 1), H(nv, nv, 2)
        vec = {k: H(1, nv, s).view(-1) for k, s in (("x", 6), ("r", 7), ("y2", 7), ("x1", 8), ("x2", 9))}
        wsm = wsz(("atax", (nv, nv)), ("bicg", (nv, nv)), ("mvt", (nv,)), ("matvec_partial", (nv, nv)))
        for kern in ("atax", "bicg", "mvt", "gesummv"):
            v = dict(A=Av[v0:v1].contiguous(), B=Bv[v0:v1].contiguous(), x=vec["x"].clone(), r=vec["r"].clone(),
                     y2=vec["y2"].clone(), x1=vec["x1"].clone(), x2=vec["x2"].clone(),
                     y=torch.zeros(nv, device=dev), s=torch.zeros(nv, device=dev), q=torch.zeros(nv, device=dev),
                     yo=torch.zeros(nv, device=dev), tmp=torch.zeros(v1 - v0, device=dev))
            D.matvec(None, kern, nv, v, wsm, 1.5, 1.2, K=K)
            torch.cuda.synchronize()
            out = {"atax": v["y"], "bicg": v["s"], "mvt": v["x2"], "gesummv": v["yo"]}[kern]
            extra = {"bicg": v["q"], "mvt": v["x1"], "atax": v["tmp"], "gesummv": v["yo"]}[kern]
            res[kern] = (v0, v1, out.cpu().numpy()[v0:v1], extra.cpu().numpy())
        if D.comm() is not None:  # covariance / correlation, observations split (pb_<k>_dist)
            ms, ns = 516, 700
            data = P.structured_data(ns, ms)
            o0, o1 = D.partition(ns, world, rank, False, 32)
            b0, b1 = D.partition(ms, world, rank, False, 32)
            dblk = torch.from_numpy(data[o0:o1].copy()).to(dev)
            wsc = torch.empty(max(pb.workspace_size(k, (ms, ns, world, rank))
                                  for k in ("covariance_dist", "correlation_dist")), dtype=torch.uint8, device=dev)
            cb, kb = torch.empty(b1 - b0, ms, device=dev), torch.empty(b1 - b0, ms, device=dev)
            mean, mean2, sd = (torch.empty(ms, device=dev) for _ in range(3))
            D.stat_obs(None, "covariance", ms, ns, float(ns), 0.1, dblk, cb, mean, None, wsc)
            D.stat_obs(None, "correlation", ms, ns, float(ns), 0.1, dblk, kb, mean2, sd, wsc)
            torch.cuda.synchronize()
            res["covcorr"] = (b0, b1, cb.cpu().numpy(), kb.cpu().numpy(), mean.cpu().numpy(), mean2.cpu().numpy(),
                              sd.cpu().numpy())
            # tiny: at world 3 the last rank has no observations and no output rows
            mt, nt = 36, 40
            data = P.structured_data(nt, mt)
            o0, o1 = D.partition(nt, world, rank, False, 32)
            b0, b1 = D.partition(mt, world, rank, False, 32)
            dblk = torch.from_numpy(data[o0:o1].copy()).to(dev) if o1 > o0 else None
            wst = torch.empty(max(pb.workspace_size(k, (mt, nt, world, rank))
                                  for k in ("covariance_dist", "correlation_dist")), dtype=torch.uint8, device=dev)
            cb = torch.empty(b1 - b0, mt, device=dev) if b1 > b0 else None
            mean, sd = torch.empty(mt, device=dev), torch.empty(mt, device=dev)
            D.stat_obs(None, "correlation", mt, nt, float(nt), 0.1, dblk, cb, mean, sd, wst)
            torch.cuda.synchronize()
            res["covcorr_tiny"] = (b0, b1, None if cb is None else cb.cpu().numpy(), mean.cpu().numpy())
            # PolyBench-GPU's constants: FLOAT_N = 3214212.01 (not the observation count), eps = 0.005
            FN = 3214212.01
            cb2 = torch.empty(b1 - b0, mt, device=dev) if b1 > b0 else None
            kb2 = torch.empty(b1 - b0, mt, device=dev) if b1 > b0 else None
            mean3, sd3 = torch.empty(mt, device=dev), torch.empty(mt, device=dev)
            D.stat_obs(None, "covariance", mt, nt, FN, 0.005, dblk, cb2, mean3, None, wst)
            D.stat_obs(None, "correlation", mt, nt, FN, 0.005, dblk, kb2, mean3, sd3, wst)
            torch.cuda.synchronize()
            res["covcorr_fn"] = (b0, b1, None if cb2 is None else cb2.cpu().numpy(),
                                 None if kb2 is None else kb2.cpu().numpy(), mean3.cpu().numpy(), sd3.cpu().numpy())
        q.put((rank, res))
    except Exception as e:  # report instead of hanging the parent
        q.put((rank, {"error": repr(e)}))
    finally:
        torch.cuda.synchronize()
        D.close_comm()
        dist.destroy_process_group()


@pytest.mark.parametrize("backend,world", [("gloo", 2), ("nccl", 1), ("gloo-peer", 2), ("nccl-peer", 1),
                                           ("gloo-peer", 3)])
def test_dist_ranks_one_gpu_real_kernels(backend, world):
    """gloo: two ranks share cuda:0 (host-staged test stand-ins for the two
    collectives, injected through the kernel namespace). nccl: one rank
    with PB_FORCE_DIST and a libpb communicator, i.e. the N>1 code path through
    the C ABI's pb_<k>_dist entry points (NCCL all-gather / reduce-scatter inside
    libpb, 3mm's side stream) end to end. gloo-peer: two processes on cuda:0 with
    a local libpb comm whose collectives are the peer-memory push/consume kernels
    over CUDA IPC (the fused path). nccl-peer: the same kernels at world size 1."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q, backend)) for r in range(world)]
    for p in procs:
        p.start()
    out = dict(q.get(timeout=600) for _ in range(world))
    for p in procs:
        p.join(timeout=120)
    for r in range(world):
        assert "error" not in out[r], out[r]
    n = 512
    A, B, C, Dm = (pbgen.gen_host(n, n, s) for s in (1, 2, 3, 4))
    E_r, F_r, G_r = oracle.mm3(A, B, C, Dm)
    _, _, G_s = oracle.mm3(A, B, C, Dm, absmode=True)
    F_s = oracle.mm3(A, B, C, Dm, absmode=True)[1]
    t_r, D_r = oracle.mm2(1.5, 1.2, A, B, C, Dm)
    t_s, D_s = oracle.mm2(1.5, 1.2, A, B, C, Dm, absmode=True)
    G = np.zeros((n, n))
    Dg = np.zeros((n, n))
    for r in range(world):
        r0, r1, g, f = out[r]["3mm"]
        G[r0:r1] = g
        assert P.cerr(f, F_r, F_s) <= P.TOL  # all-gather delivered all of F
        r0, r1, d = out[r]["2mm"]
        Dg[r0:r1] = d
    assert P.cerr(G, G_r, G_s) <= P.TOL and P.cerr(Dg, D_r, D_s) <= P.TOL
    n2, m2 = 768, 260
    A2, B2 = pbgen.gen_host(n2, m2, 1), pbgen.gen_host(n2, m2, 2)
    Cf = pbgen.gen_host(n2, n2, 3, mode=pbgen.SYM)
    for name, ref, sc in (("syrk", oracle.syrk(1.5, 1.2, Cf, A2), oracle.syrk(1.5, 1.2, Cf, A2, absmode=True)),
                          ("syr2k", oracle.syr2k(1.5, 1.2, Cf, A2, B2),
                           oracle.syr2k(1.5, 1.2, Cf, A2, B2, absmode=True))):
        got = np.zeros((n2, n2))
        for r in range(world):
            s0, s1, blk = out[r][name]
            got[s0:s1] = blk
        assert P.cerr(got, ref, sc) <= P.TOL, name
    if backend != "gloo":  # observations-split covariance / correlation (column-sum allreduce)
        ms, ns = 516, 700
        data = P.structured_data(ns, ms)
        cov_r, mean_r = oracle.covariance(float(ns), data)
        cov_s, mean_s = oracle.covariance(float(ns), data, absmode=True)
        corr_r, _, sd_r = oracle.correlation(float(ns), 0.1, data)
        corr_s, _, sd_s = oracle.correlation(float(ns), 0.1, data, absmode=True)
        cov, corr = np.zeros((ms, ms)), np.zeros((ms, ms))
        for r in range(world):
            b0, b1, cb, kb, mean, mean2, sd = out[r]["covcorr"]
            cov[b0:b1], corr[b0:b1] = cb, kb
            assert P.cerr(mean, mean_r, mean_s) <= P.TOL and np.array_equal(mean, mean2)
            assert P.cerr(sd, sd_r, sd_s) <= P.TOL
            assert np.array_equal(mean, out[0]["covcorr"][4])  # every rank holds the same statistics
        assert P.cerr(cov, cov_r, cov_s) <= P.TOL, P.cerr(cov, cov_r, cov_s)
        assert P.cerr(corr, corr_r, corr_s) <= P.TOL, P.cerr(corr, corr_r, corr_s)
        assert np.all(np.diag(corr) == 1.0) and np.all(cov[0] == 0.0)  # R6; constant column 0
        mt, nt = 36, 40
        data = P.structured_data(nt, mt)
        cr, mr, _ = oracle.correlation(float(nt), 0.1, data)
        cs, ms_, _ = oracle.correlation(float(nt), 0.1, data, absmode=True)
        got = np.zeros((mt, mt))
        for r in range(world):
            b0, b1, blk, mean = out[r]["covcorr_tiny"]
            if b1 > b0:
                got[b0:b1] = blk
            assert P.cerr(mean, mr, ms_) <= P.TOL
        assert P.cerr(got, cr, cs) <= P.TOL
        FN = 3214212.01
        cv_r, mean_r = oracle.covariance(FN, data)
        cv_s, mean_s = oracle.covariance(FN, data, absmode=True)
        co_r, _, sd_r = oracle.correlation(FN, 0.005, data)
        co_s, _, sd_s = oracle.correlation(FN, 0.005, data, absmode=True)
        gcv, gco = np.zeros((mt, mt)), np.zeros((mt, mt))
        for r in range(world):
            b0, b1, cb2, kb2, mean3, sd3 = out[r]["covcorr_fn"]
            if b1 > b0:
                gcv[b0:b1], gco[b0:b1] = cb2, kb2
            assert P.cerr(mean3, mean_r, mean_s) <= P.TOL and P.cerr(sd3, sd_r, sd_s) <= P.TOL
        assert P.cerr(gcv, cv_r, cv_s) <= P.TOL and P.cerr(gco, co_r, co_s) <= P.TOL
    nv = 2048
    Av, Bv = pbgen.gen_host(nv, nv, 1), pbgen.gen_host(nv, nv, 2)
    x, rr, y2, x1, x2 = (pbgen.gen_host(1, nv, s)[0] for s in (6, 7, 7, 8, 9))
    refs = {"atax": oracle.atax(Av, x)[0], "bicg": oracle.bicg(Av, x, rr)[0],
            "mvt": oracle.mvt(x1, x2, x, y2, Av)[1], "gesummv": oracle.gesummv(1.5, 1.2, Av, Bv, x)[1]}
    for k, ref in refs.items():
        got = np.zeros(nv)
        for r in range(world):
            v0, v1, blk, _ = out[r][k]
            got[v0:v1] = blk
        assert np.max(np.abs(got - ref) / np.abs(ref)) <= P.TOL, k


@pytest.mark.parametrize("transport", ["peer", "nccl"])
def test_bench_forced_sharded_nccl(transport):
    """bench.py on the sharded path over a world-size-1 NCCL group (collectives:
    libpb's peer-memory kernels, or NCCL inside libpb): one JSON line, every
    kernel timed, e2e included."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import json
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, PB_FORCE_DIST="1", PB_TRANSPORT=transport, MASTER_ADDR="127.0.0.1",
               MASTER_PORT=str(_free_port()))
    r = subprocess.run([sys.executable, "bench.py", "--steps", "1", "--warmup", "3", "--no-cpu"], cwd=root, env=env,
                       capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-2000:]
    line = json.loads(r.stdout.strip().splitlines()[-1])
    assert line["value"] > 0 and line["e2e"]["value"] > 0
    assert all(v["ms"] > 0 for v in line["kernels"].values())
    assert ("peer" in line["config"]["transport"]) == (transport == "peer")


def _peer_worker(rank, world, port, q):
    import torch.distributed as dist

    import paper_2312_13170_b200 as pb
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    res = {}
    try:
        P = pb.pb_peer_create(world, rank, 1 << 20)
        hs = [None] * world
        dist.all_gather_object(hs, P.ipc_handle)
        P.open(b"".join(hs))
        dev = torch.device("cuda", 0)
        out = []
        for it, total in enumerate([1004, 4096, 12, 1004, 65536]):  # several epochs, uneven blocks
            part = torch.from_numpy(pbgen.gen_host(1, total, 20 + it + 7 * rank)[0]).to(dev)
            b, e = pb.pb_row_partition(total, world, rank, False, 4)
            blk = torch.full((max(e - b, 1),), float("nan"), device=dev)
            P.reduce_scatter(part, blk, total)
            rows, cols = 300 + it, 8
            fb, fe = pb.pb_row_partition(rows, world, rank, False, 128)
            full = torch.full((rows, cols), float("nan"), device=dev)
            mine = torch.from_numpy(pbgen.gen_host(rows, cols, 40 + it)[fb:fe].copy()).to(dev)
            full[fb:fe].copy_(mine)
            P.all_gather(full[fb:fe], full, rows, cols)  # in place
            torch.cuda.synchronize()
            out.append((total, b, e, blk.cpu().numpy()[: e - b], rows, full.cpu().numpy()))
        res["out"] = out
        res["status"] = P.status()
        dist.barrier()
        P.close()
        q.put((rank, res))
    except Exception as ex:  # report instead of hanging the parent
        q.put((rank, {"error": repr(ex)}))
    finally:
        dist.destroy_process_group()


def test_peer_collectives_two_processes_one_gpu():
    """pb_peer reduce-scatter / all-gather between two processes sharing cuda:0
    (CUDA IPC): bitwise equal to the fp32 sum in rank order / the gathered rows,
    over several epochs (the ack handshake lets a slot be reused)."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    world, port = 2, _free_port()
    procs = [ctx.Process(target=_peer_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=600) for _ in range(world))
    for p in procs:
        p.join(timeout=120)
    for r in range(world):
        assert "error" not in res[r], res[r]
        assert res[r]["status"] == 0
    for it in range(5):
        total = res[0]["out"][it][0]
        parts = [pbgen.gen_host(1, total, 20 + it + 7 * r)[0] for r in range(world)]
        ref = parts[0].copy()
        for r in range(1, world):
            ref = (ref + parts[r]).astype(np.float32)  # fp32, rank order
        rows = res[0]["out"][it][4]
        full_ref = pbgen.gen_host(rows, 8, 40 + it)
        for r in range(world):
            _, b, e, blk, _, full = res[r]["out"][it]
            assert np.array_equal(blk.view(np.uint32), ref[b:e].view(np.uint32)), (it, r)
            assert np.array_equal(full.view(np.uint32), full_ref.view(np.uint32)), (it, r)


@pytest.mark.parametrize("transport", ["local"])
def test_bench_two_ranks_share_gpu(transport):
    """bench.py under torchrun with 2 ranks on cuda:0 (PB_SHARE_GPU): libpb's
    peer-memory kernels between the two processes (PB_TRANSPORT=local; the product
    path has no host-staged collectives). Checks the N=2 launch path end to end (timings are not
    meaningful: the ranks share one GPU)."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import json
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, PB_SHARE_GPU="1")
    if transport == "local":
        env["PB_TRANSPORT"] = "local"
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2", "--master-addr",
           "127.0.0.1", "--master-port", str(_free_port()), "bench.py", "--gpus", "2", "--steps", "1", "--warmup", "3",
           "--no-cpu", "--no-e2e", "--kernels", "3mm,covariance,correlation,atax,bicg,mvt,gesummv"]
    r = subprocess.run(cmd, cwd=root, env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
    line = json.loads([ln for ln in r.stdout.strip().splitlines() if ln.startswith("{")][-1])
    assert line["n_gpus"] == 2 and line["value"] > 0
    assert (line["config"]["transport"] or "").startswith("peer") == (transport == "local")
    chk = line["sharded_check"]  # atax y, 3mm G and the observations-split covariance vs one-GPU calls
    assert chk["ok"] and "cov_max_abs_over_max" in chk, chk


def test_peer_collectives_graph_replay():
    """pb_atax_dist / pb_mvt_dist over a (world-size-1, local) peer group captured
    into one CUDA graph and replayed with new inputs: the collective epoch lives in
    device memory, so every replay waits for (and sums) the right data."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2312_13170_b200 as pb
    dev = torch.device("cuda", 0)
    comm = pb.pb_comm_init_local(1, 0)
    peer = pb.pb_peer_create(1, 0, 1 << 20)
    peer.open(peer.ipc_handle)
    pb.pb_comm_attach_peer(comm, peer)
    try:
        m, n = 1000, 2048
        A = torch.from_numpy(pbgen.gen_host(m, n, 1)).to(dev)
        x = torch.empty(n, device=dev)
        y, tmp = torch.empty(n, device=dev), torch.empty(m, device=dev)
        ws = pb.workspace("atax_dist", (m, n, 1, 0), dev)
        An = torch.from_numpy(pbgen.gen_host(n, n, 2)).to(dev)
        x1, x2 = torch.empty(n, device=dev), torch.empty(n, device=dev)
        y1 = torch.from_numpy(pbgen.gen_host(1, n, 8)[0]).to(dev)
        wsm = pb.workspace("mvt_dist", (n, 1, 0), dev)
        s = torch.cuda.Stream()
        g = torch.cuda.CUDAGraph()
        x.copy_(torch.from_numpy(pbgen.gen_host(1, n, 6)[0]))
        with torch.cuda.graph(g, stream=s):
            pb.pb_atax_dist(comm, m, n, A, x, y, tmp, ws=ws, stream=s)
            pb.pb_mvt_dist(comm, n, x1, x2, y1, x, An, ws=wsm, stream=s)
        for it in range(4):
            xh = pbgen.gen_host(1, n, 30 + it)[0]
            x1h, x2h = pbgen.gen_host(1, n, 40 + it)[0], pbgen.gen_host(1, n, 50 + it)[0]
            x.copy_(torch.from_numpy(xh))
            x1.copy_(torch.from_numpy(x1h))
            x2.copy_(torch.from_numpy(x2h))
            g.replay()
            torch.cuda.synchronize()
            y_r = oracle.atax(pbgen.gen_host(m, n, 1), xh)[0]
            assert np.max(np.abs(y.cpu().numpy() - y_r) / np.abs(y_r)) <= P.TOL, it
            o1, o2 = oracle.mvt(x1h, x2h, pbgen.gen_host(1, n, 8)[0], xh, pbgen.gen_host(n, n, 2))
            assert np.max(np.abs(x1.cpu().numpy() - o1) / np.abs(o1)) <= P.TOL, it
            assert np.max(np.abs(x2.cpu().numpy() - o2) / np.abs(o2)) <= P.TOL, it
        assert peer.status() == 0
    finally:
        torch.cuda.synchronize()
        comm.close()
        peer.close()


def test_comm_and_peer_argument_errors():
    """Multi-GPU ABI validation: a peer group that does not match the comm, an
    unopened peer group, and collectives on a comm without any transport are
    rejected with PB_ERR_INVALID_ARG before anything is enqueued."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2312_13170_b200 as pb
    comm = pb.pb_comm_init_local(2, 0)
    p1 = pb.pb_peer_create(1, 0, 1 << 16)
    p1.open(p1.ipc_handle)
    p2 = pb.pb_peer_create(2, 0, 1 << 16)  # not opened
    try:
        with pytest.raises(pb.PBError) as e:
            pb.pb_comm_attach_peer(comm, p1)  # nranks mismatch
        assert e.value.status == 1
        with pytest.raises(pb.PBError) as e:
            pb.pb_comm_attach_peer(comm, p2)  # not opened
        assert e.value.status == 1
        y = torch.full((1024,), 5.0, device="cuda")
        with pytest.raises(pb.PBError) as e:  # local comm, no peer attached: no transport
            pb.pb_atax_dist(comm, 2048, 2048, torch.ones(1024, 2048, device="cuda"), torch.ones(2048, device="cuda"),
                            y, None)
        assert e.value.status == 1 and bool((y == 5.0).all())
        with pytest.raises(pb.PBError):
            pb.pb_peer_create(9, 0, 1 << 16)  # more than 8 ranks
    finally:
        comm.close()
        p1.close()
        p2.close()


@pytest.mark.parametrize("m,n,G", [(260, 300, 2), (516, 2048, 3), (2048, 2048, 8), (128, 3000, 1)])
def test_cov_corr_row_bands(m, n, G):
    """pb_covariance_rows / pb_correlation_rows (replicated data, output row blocks, no
    exchange): the bands of every rank assemble the full result within the parity
    tolerance; correlation's diagonal is exactly 1."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2312_13170_b200 as pb
    from tests import parity as P
    data = P.structured_data(n, m)
    dd = P.dev(data)
    for corr in (False, True):
        full = np.zeros((m, m), np.float32)
        for g in range(G):
            r0, r1 = pb.pb_row_partition(m, G, g, False, 128)
            if r1 <= r0:
                continue
            blk = torch.empty(r1 - r0, m, device="cuda")
            if corr:
                pb.pb_correlation_rows(m, n, float(n), 0.1, r0, r1, dd, blk)
            else:
                pb.pb_covariance_rows(m, n, float(n), r0, r1, dd, blk)
            full[r0:r1] = P.host(blk)
        if corr:
            r, s = oracle.correlation(float(n), 0.1, data)[0], oracle.correlation(float(n), 0.1, data, absmode=True)[0]
            assert np.all(np.diag(full) == 1.0)
        else:
            r, s = oracle.covariance(float(n), data)[0], oracle.covariance(float(n), data, absmode=True)[0]
        assert P.cerr(full, r, s) <= P.TOL, (corr, P.cerr(full, r, s))
