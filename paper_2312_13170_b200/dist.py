"""Row-block data parallelism over the GPUs of one node (DESIGN.md §Multi-GPU,
SURVEY.md §8(e)). One process per GPU; torch.distributed (NCCL over
NVLink/NVSwitch on GPUs, gloo in the CPU tests) carries the only exchange
steps the math needs:

  gemm, 2mm, gesummv, syrk, syr2k   no collective: rank g owns output rows R_g and
                                    computes them from its row block + replicated
                                    operands (2mm: tmp[R] = alpha A[R] B is exactly
                                    what D[R] = tmp[R] C + beta D[R] needs)
  covariance, correlation           observations split: column sums ALL-GATHERed and summed in
                                    rank order (the allreduce), local partial Gram, REDUCE-SCATTER
                                    of the m x m sum into output row bands (stat_obs)
  3mm                               F = C D by row blocks, ALL-GATHER of F (async, overlapped
                                    with E[R] = A[R] B), then G[R] = E[R] F
  atax, bicg, mvt                   row dots local; the transposed product's per-rank
                                    partial vector is REDUCE-SCATTERed into the same
                                    row partition (mvt folds x2's old value into rank 0's
                                    partial, so the sum is x2 + A^T y_2)

Every arithmetic step runs in libpb through the C ABI (`K` below defaults to
the binding; the CPU gloo tests inject an oracle-backed namespace, with
host-staged stand-ins for the two collectives, to check the partition and
collective logic without a GPU). Outputs stay row-sharded (reading R15).

With an NCCL process group, `init_comm()` creates a libpb communicator and
every call below goes to the C ABI's `pb_<k>_dist` entry points, which run the
collectives with NCCL inside libpb (3mm's all-gather on the comm's side
stream, overlapped with E = A B). A sharded call without one raises.
"""
from __future__ import annotations

import os

import torch
import torch.distributed as dist

import paper_2312_13170_b200 as _pb


_COMM = None  # libpb communicator (pb_comm_init / pb_comm_init_local), set by init_comm()
_PEER = None  # libpb peer group attached to it (fused peer-memory collectives)


def init_comm(transport=None, peer_bytes=64 << 20):
    """Create the libpb communicator over the current torch.distributed group.

    transport (default: env PB_TRANSPORT, else "nccl"):
      "nccl"   NCCL inside libpb (rank 0's unique id broadcast through torch.distributed)
      "peer"   NCCL comm + an attached peer group: the exchange steps run as libpb's
               push/consume kernels over CUDA IPC mappings (NVLink/NVSwitch P2P)
      "local"  no NCCL, peer group only (e.g. several processes sharing one GPU)
    peer_bytes: data region of the peer group (3mm's all-gather needs n*n*4)."""
    global _COMM, _PEER
    transport = transport or os.environ.get("PB_TRANSPORT", "nccl")
    world, rank = _world()
    if transport == "local":
        _COMM = _pb.pb_comm_init_local(world, rank)
    else:
        uid = [_pb.pb_comm_unique_id() if rank == 0 else None]
        if world > 1:
            dist.broadcast_object_list(uid, src=0)
        _COMM = _pb.pb_comm_init(world, rank, uid[0])
    if transport in ("peer", "local"):
        err = None
        try:
            _PEER = _pb.pb_peer_create(world, rank, peer_bytes)
            handles = [None] * world
            if world > 1:
                dist.all_gather_object(handles, _PEER.ipc_handle)
            else:
                handles = [_PEER.ipc_handle]
            _PEER.open(b"".join(handles))
        except _pb.PBError as e:  # e.g. no P2P between these GPUs
            err = repr(e)
        errs = [None] * world
        if world > 1:
            dist.all_gather_object(errs, err)
        else:
            errs = [err]
        if any(errs):  # every rank must agree on the transport
            if _PEER is not None:
                _PEER.close()
                _PEER = None
            if transport == "local":
                raise RuntimeError(f"peer group unavailable: {errs}")
            import sys
            print(f"pb: peer-memory collectives unavailable ({[e for e in errs if e][0]}); using NCCL",
                  file=sys.stderr)
        else:
            _pb.pb_comm_attach_peer(_COMM, _PEER)
    return _COMM


def close_comm():
    """Destroy the communicator (and peer group). Call after every rank is done
    (the caller synchronises and barriers first)."""
    global _COMM, _PEER
    if _COMM is not None:
        _COMM.close()
        _COMM = None
    if _PEER is not None:
        if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
            dist.barrier()  # no rank may still write into this buffer
        _PEER.close()
        _PEER = None


def peer():
    return _PEER


def comm():
    return _COMM


def _world():
    if dist.is_available() and dist.is_initialized():
        return dist.get_world_size(), dist.get_rank()
    return 1, 0


def _single(world):
    """True when the unsharded single-GPU entry points apply. PB_FORCE_DIST=1 (test
    aid) keeps a world-size-1 process group on the sharded path, so one GPU runs
    every N>1 call, NCCL collectives included."""
    return world == 1 and not os.environ.get("PB_FORCE_DIST")


def partition(rows, world, rank, triangular=False, align=128, K=_pb):
    return K.pb_row_partition(rows, world, rank, triangular, align)


def _collectives(K):
    """The exchange steps of a sharded call. With a libpb communicator they run inside
    libpb (`pb_<k>_dist`: NCCL or the peer-memory kernels); a kernel namespace without
    one must supply them (the CPU gloo tests inject host-staged stand-ins). The product
    package performs no arithmetic outside libpb."""
    ag = getattr(K, "all_gather_rows", None)
    rs = getattr(K, "reduce_scatter_vec", None)
    if ag is None or rs is None:
        raise RuntimeError("sharded call without a libpb communicator: call dist.init_comm() first")
    return ag, rs


# --------------------------------------------------------------------- contractions
def mm2_rows(ctx, n, alpha, beta, tmp, A, B, C, D, ws, K=_pb):
    """2mm on this rank's rows (A, tmp, D are the local row blocks)."""
    if _COMM is not None and K is _pb:
        K.pb_2mm_dist(_COMM, n, n, n, n, alpha, beta, tmp, A, B, C, D, ws=ws)
        return K.last_launch_count()
    rows = A.shape[0]
    if rows == 0:
        return 0
    K.pb_2mm(rows, n, n, n, alpha, beta, tmp, A, B, C, D, ws=ws)
    return K.last_launch_count()


def mm3_rows(ctx, n, E, A, B, Fl, F, C, D, G, ws, K=_pb):
    """3mm: F row block -> async all-gather of F overlapped with E[R] = A[R] B -> G[R] = E[R] F."""
    world, rank = _world()
    L = 0
    if _single(world):
        K.pb_3mm(A.shape[0], n, n, n, n, E, A, B, F, C, D, G, ws=ws)
        return K.last_launch_count()
    bounds = [partition(n, world, g, False, 128, K) for g in range(world)]
    f0, f1 = bounds[rank]
    if _COMM is not None and K is _pb:  # F rows -> all-gather (libpb side stream) || E -> G
        K.pb_3mm_dist(_COMM, n, n, n, n, n, E, A, B, F, C[f0:f1], D, G, ws=ws)
        return K.last_launch_count()
    all_gather_rows, _ = _collectives(K)
    if f1 > f0:
        K.pb_gemm(f1 - f0, n, n, 1.0, 0.0, Fl, C[f0:f1], D, ws=ws)  # F[R'] = C[R'] D
        L += K.last_launch_count()
    work = all_gather_rows(F, Fl, world, bounds)
    rows = A.shape[0]
    if rows:
        K.pb_gemm(rows, n, n, 1.0, 0.0, E, A, B, ws=ws)  # E[R] = A[R] B, overlaps the all-gather
        L += K.last_launch_count()
    if work is not None and hasattr(work, "wait"):
        work.wait()
    if rows:
        K.pb_gemm(rows, n, n, 1.0, 0.0, G, E, F, ws=ws)  # G[R] = E[R] F
        L += K.last_launch_count()
    return L


def syrk_rows(ctx, n, m, alpha, beta, C_blk, A, ws, B=None, K=_pb):
    world, rank = _world()
    if _COMM is not None and K is _pb:
        if B is None:
            K.pb_syrk_dist(_COMM, n, m, alpha, beta, C_blk, A, ws=ws)
        else:
            K.pb_syr2k_dist(_COMM, n, m, alpha, beta, C_blk, A, B, ws=ws)
        return K.last_launch_count()
    r0, r1 = partition(n, world, rank, 2, 256, K)
    if r1 <= r0:
        return 0
    if B is None:
        K.pb_syrk_rows(n, m, r0, r1, alpha, beta, C_blk, A, ws=ws)
    else:
        K.pb_syr2k_rows(n, m, r0, r1, alpha, beta, C_blk, A, B, ws=ws)
    return K.last_launch_count()


# --------------------------------------------------------------------- covariance / correlation
def stat_obs(ctx, kernel, m, n, float_n, eps, data_blk, out_blk, mean, sd, ws, K=_pb):
    """covariance / correlation with the OBSERVATIONS split (north_star: "an allreduce of
    column sums"): data_blk = this rank's observations block(n, G, g, 0, 32), out_blk =
    rows block(m, G, g, 0, 32) of the result. Everything (column sums, their all-gather and
    rank-order sum, centring, the tcgen05 partial Gram, the reduce-scatter of the m x m sum,
    the scaling) runs in libpb (pb_<k>_dist); a sharded call needs init_comm()."""
    if _COMM is None or K is not _pb:
        raise RuntimeError("stat_obs needs a libpb communicator: call dist.init_comm() first")
    if kernel == "covariance":
        K.pb_covariance_dist(_COMM, m, n, float_n, data_blk, out_blk, mean, ws=ws)
    else:
        K.pb_correlation_dist(_COMM, m, n, float_n, eps, data_blk, out_blk, mean, sd, ws=ws)
    return K.last_launch_count()


# --------------------------------------------------------------------- matrix-vector
def matvec(ctx, kernel, n, v, ws, alpha, beta, K=_pb):
    """atax / bicg / mvt / gesummv on this rank's row block of A (and B).
    v: dict with A (local rows x n), x, r, x1, x2, y2 (full n vectors), y, s, yo
    (full-length partial buffers), q/tmp outputs."""
    world, rank = _world()
    A = v["A"]
    rows = A.shape[0]
    if _single(world):
        if kernel == "atax":
            K.pb_atax(rows, n, A, v["x"], v["y"], v["tmp"], ws=ws)
        elif kernel == "bicg":
            K.pb_bicg(n, rows, A, v["s"], v["q"], v["x"], v["r"], ws=ws)
        elif kernel == "mvt":
            K.pb_mvt(n, v["x1"], v["x2"], v["x"], v["y2"], A, ws=ws)
        else:
            K.pb_gesummv(n, alpha, beta, A, v["B"], v["tmp"], v["x"], v["yo"], ws=ws)
        return K.last_launch_count()
    bounds = [partition(n, world, g, False, 4, K) for g in range(world)]
    r0, r1 = bounds[rank]
    if _COMM is not None and K is _pb:  # local pass + NCCL reduce-scatter inside libpb
        c = _COMM
        if kernel == "atax":
            K.pb_atax_dist(c, n, n, A, v["x"], v["y"][r0:r1], v["tmp"][:rows], ws=ws)
        elif kernel == "bicg":
            K.pb_bicg_dist(c, n, n, A, v["s"][r0:r1], v["q"][r0:r1], v["x"], v["r"][r0:r1], ws=ws)
        elif kernel == "mvt":
            K.pb_mvt_dist(c, n, v["x1"][r0:r1], v["x2"][r0:r1], v["x"], v["y2"][r0:r1], A, ws=ws)
        else:
            K.pb_gesummv_dist(c, n, alpha, beta, A, v["B"], v["tmp"][:rows], v["x"], v["yo"][r0:r1], ws=ws)
        return K.last_launch_count()
    _, reduce_scatter_vec = _collectives(K)
    L = 0
    if kernel == "atax":  # tmp[R] = A[R] x ; y = sum_g A[R_g]^T tmp[R_g]
        part = v["yo"]
        K.pb_atax(rows, n, A, v["x"], part, v["tmp"][:rows], ws=ws)  # one pass over A[R]
        L += K.last_launch_count()
        reduce_scatter_vec(v["y"][r0:r1], part, world, bounds)
    elif kernel == "bicg":  # q[R] = A[R] p ; s = sum_g A[R_g]^T r[R_g]
        part = v["yo"]
        K.pb_matvec_partial(rows, n, A, v["x"], None, v["q"][r0:r1], v["r"][r0:r1], None, part, ws=ws)
        L += K.last_launch_count()
        reduce_scatter_vec(v["s"][r0:r1], part, world, bounds)
    elif kernel == "mvt":  # x1[R] += A[R] y_1 ; x2 = x2 + sum_g A[R_g]^T y_2[R_g]
        part = v["yo"]
        x1l = v["x1"][r0:r1]
        K.pb_matvec_partial(rows, n, A, v["x"], x1l, x1l, v["y2"][r0:r1], v["x2"] if rank == 0 else None, part,
                            ws=ws)
        L += K.last_launch_count()
        reduce_scatter_vec(v["x2"][r0:r1], part, world, bounds)
    else:  # gesummv: purely row-local
        K.pb_gesummv_rows(rows, n, alpha, beta, A, v["B"], v["tmp"][:rows], v["x"], v["yo"][r0:r1], ws=ws)
        L += K.last_launch_count()
    return L
