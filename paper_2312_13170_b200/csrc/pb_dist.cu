// pb_dist.cu — the multi-GPU entry points of include/pb.h (SURVEY.md §8(b)/(e),
// DESIGN.md §9). One process per GPU, output-row-block sharding; NCCL over
// NVLink/NVSwitch carries the only exchange steps the math has: 3mm's
// all-gather of F (run on the comm's side stream, overlapped with E = A B) and
// the reduce-scatter of atax/bicg/mvt's transposed-product partial vectors.
// Every arithmetic step runs through the single-GPU entry points (the same
// kernels); this file only adds the partition and the collectives.
//
// libnccl.so.2 is resolved with dlopen on first use: libpb loads (and the CPU
// tests run) without NCCL, and inside a PyTorch process the libnccl.so.2 torch
// already loaded is reused.
#include <dlfcn.h>
#include <nccl.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <mutex>
#include <string>

#include "pb_check.h"

using namespace pb;

// Symmetric peer buffer (k_peer.cu): header (flags, acks, counters, status) + data region.
struct pb_peer {
  int nranks = 0, rank = 0, dev = -1;
  char* base = nullptr;  // own allocation: PEER_HDR + data_bytes
  size_t data_bytes = 0;
  char* mapped[PEER_MAXR] = {};  // every rank's base in this process (own = base)
  bool opened = false;
  PeerView view;
};

struct pb_comm {
  ncclComm_t nc = nullptr;  // null for a local comm (pb_comm_init_local): collectives via the peer group
  pb_peer* peer = nullptr;  // attached peer group: fused peer-memory collectives instead of NCCL
  int nranks = 0, rank = 0, dev = -1;
  cudaStream_t side = nullptr;  // collectives overlapped with compute (3mm's all-gather)
  cudaEvent_t ev_ready = nullptr, ev_done = nullptr;
};

namespace {

struct Nccl {
  std::string err;
  decltype(&ncclGetUniqueId) GetUniqueId = nullptr;
  decltype(&ncclCommInitRank) CommInitRank = nullptr;
  decltype(&ncclCommDestroy) CommDestroy = nullptr;
  decltype(&ncclAllGather) AllGather = nullptr;
  decltype(&ncclReduceScatter) ReduceScatter = nullptr;
  decltype(&ncclBroadcast) Broadcast = nullptr;
  decltype(&ncclReduce) Reduce = nullptr;
  decltype(&ncclGroupStart) GroupStart = nullptr;
  decltype(&ncclGroupEnd) GroupEnd = nullptr;
  decltype(&ncclGetErrorString) GetErrorString = nullptr;
};

const Nccl& nccl() {
  static Nccl n;
  static std::once_flag once;
  std::call_once(once, [] {
    const char* name = getenv("PB_NCCL_LIB");
    void* h = dlopen(name ? name : "libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      const char* e = dlerror();
      n.err = std::string("dlopen libnccl.so.2 failed: ") + (e ? e : "?");
      return;
    }
#define PB_SYM(f)                                                    \
  n.f = reinterpret_cast<decltype(n.f)>(dlsym(h, "nccl" #f));        \
  if (!n.f) {                                                        \
    n.err = "libnccl.so.2 lacks nccl" #f;                            \
    return;                                                          \
  }
    PB_SYM(GetUniqueId) PB_SYM(CommInitRank) PB_SYM(CommDestroy) PB_SYM(AllGather) PB_SYM(ReduceScatter)
    PB_SYM(Broadcast) PB_SYM(Reduce) PB_SYM(GroupStart) PB_SYM(GroupEnd) PB_SYM(GetErrorString)
#undef PB_SYM
  });
  return n;
}

pb_status nccl_loaded() {
  const Nccl& n = nccl();
  return n.err.empty() ? PB_OK : fail(PB_ERR_NCCL, "%s", n.err.c_str());
}

pb_status nc_check(ncclResult_t r, const char* what) {
  return r == ncclSuccess ? PB_OK : fail(PB_ERR_NCCL, "%s: %s", what, nccl().GetErrorString(r));
}
pb_status cu_check(cudaError_t e, const char* what) {
  return e == cudaSuccess ? PB_OK : fail(PB_ERR_CUDA, "%s: %s", what, cudaGetErrorString(e));
}
#define PB_TRY(expr)              \
  do {                            \
    pb_status _st = (expr);       \
    if (_st != PB_OK) return _st; \
  } while (0)
#define PB_NC(expr) PB_TRY(nc_check((expr), #expr))
#define PB_CU(expr) PB_TRY(cu_check((expr), #expr))

inline cudaStream_t S(pb_stream s) { return reinterpret_cast<cudaStream_t>(s); }

// Partition conventions (include/pb.h).
constexpr int ALIGN_MM = 128, ALIGN_SY = 256, ALIGN_MV = 4;
// covariance / correlation with the observations split: observation blocks and output row bands
constexpr int ALIGN_OBS = 32, ALIGN_ST = 32;

struct Blk {
  int b = 0, e = 0;
  int n() const { return e - b; }
};
Blk block(int rows, int nranks, int g, int mode, int align) {  // mode: pb_row_partition's `triangular`
  Blk k;
  pb_row_partition(rows, nranks, g, mode, align, &k.b, &k.e);
  return k;
}

pb_status comm_ok(const pb_comm* c) {
  if (!c || (!c->nc && !c->peer)) return fail(PB_ERR_INVALID_ARG, "comm is NULL, destroyed, or has no transport");
  int dev = -1;
  cudaGetDevice(&dev);
  if (dev != c->dev) return fail(PB_ERR_INVALID_ARG, "current device %d is not the comm's device %d", dev, c->dev);
  return PB_OK;
}

size_t ws_of(const char* k, std::initializer_list<long long> dims) {
  std::vector<long long> d(dims);
  size_t b = 0;
  if (pb_workspace_size(k, d.data(), (int)d.size(), &b) != PB_OK) return 0;
  return b;
}

// Workspace layout of a dist call: [partial vector(s)] then the local call's workspace.
struct DistWs {
  float* partial = nullptr;
  float* base = nullptr;
  void* local = nullptr;
  size_t local_bytes = 0, total = 0;
};
DistWs dist_ws(void* ws, size_t ws_bytes, long long partial_len, long long base_len, size_t local_need) {
  Carve c(ws, ws_bytes);
  DistWs w;
  if (partial_len) w.partial = c.take<float>(partial_len);
  if (base_len) w.base = c.take<float>(base_len);
  const size_t off = align_up(c.off, 256);
  w.local = ws ? static_cast<char*>(ws) + off : nullptr;
  w.local_bytes = ws_bytes > off ? ws_bytes - off : 0;
  w.total = off + local_need;
  return w;
}

// Workspace of pb_covariance_dist / pb_correlation_dist (m variables, n observations):
// every rank's column sums [G][2][m] doubles (the all-gather buffer), the centred
// transpose Yt (m x ldy, ldy = this rank's observations rounded up to 4), the partial
// Gram P (m x m), then pb_syrk_full's own workspace.
struct CovDistWs {
  double* sums = nullptr;
  float* Yt = nullptr;
  float* P = nullptr;
  void* gemm = nullptr;
  size_t gemm_bytes = 0, total = 0;
  int ldy = 0;
  static CovDistWs carve(void* ws, long long m, long long n, int G, int g) {
    CovDistWs w;
    const Blk o = block((int)n, G, g, 0, ALIGN_OBS);
    w.ldy = (o.n() + 3) / 4 * 4;
    char* base = static_cast<char*>(ws);
    size_t off = 0;
    auto take = [&](size_t bytes) -> char* {
      off = align_up(off, 256);
      char* r = base ? base + off : nullptr;
      off += bytes;
      return r;
    };
    w.sums = reinterpret_cast<double*>(take((size_t)G * 2 * m * sizeof(double)));
    if (w.ldy) {
      w.Yt = reinterpret_cast<float*>(take((size_t)m * w.ldy * sizeof(float)));
      w.P = reinterpret_cast<float*>(take((size_t)m * m * sizeof(float)));
      w.gemm_bytes = ws_of("syrk_full", {m, w.ldy});
      w.gemm = take(w.gemm_bytes);
    } else {
      w.P = reinterpret_cast<float*>(take((size_t)m * m * sizeof(float)));
    }
    w.total = align_up(off, 256);
    return w;
  }
};

size_t local_need(const std::string& k, const long long* d, int G, int g) {
  if (k == "gemm") {
    const Blk r = block(d[0], G, g, 0, ALIGN_MM);
    return r.n() ? ws_of("gemm", {r.n(), d[1], d[2]}) : 0;
  }
  if (k == "2mm") {
    const Blk r = block(d[0], G, g, 0, ALIGN_MM);
    return r.n() ? ws_of("2mm", {r.n(), d[1], d[2], d[3]}) : 0;
  }
  if (k == "3mm") {  // ni nj nk nl nm
    const Blk r = block(d[0], G, g, 0, ALIGN_MM), f = block(d[1], G, g, 0, ALIGN_MM);
    size_t b = 0;
    if (f.n()) b = std::max(b, ws_of("gemm", {f.n(), d[3], d[4]}));
    if (r.n()) b = std::max({b, ws_of("gemm", {r.n(), d[1], d[2]}), ws_of("gemm", {r.n(), d[3], d[1]})});
    return b;
  }
  if (k == "syrk" || k == "syr2k") {
    const Blk r = block(d[0], G, g, 2, ALIGN_SY);
    return r.n() ? ws_of(k == "syrk" ? "syrk_rows" : "syr2k_rows", {d[0], d[1], r.b, r.e}) : 0;
  }
  if (k == "atax") {  // m n: rows of m
    const Blk r = block(d[0], G, g, 0, ALIGN_MV);
    return r.n() ? ws_of("atax", {r.n(), d[1]}) : 0;
  }
  if (k == "bicg") {  // m n: A n x m, rows of n
    const Blk r = block(d[1], G, g, 0, ALIGN_MV);
    return r.n() ? ws_of("bicg", {d[0], r.n()}) : 0;
  }
  if (k == "mvt") {
    const Blk r = block(d[0], G, g, 0, ALIGN_MV);
    return r.n() ? ws_of("matvec_partial", {r.n(), d[0]}) : 0;
  }
  if (k == "gesummv") {
    const Blk r = block(d[0], G, g, 0, ALIGN_MV);
    return r.n() ? ws_of("gesummv_rows", {r.n(), d[0]}) : 0;
  }
  if (k == "covariance" || k == "correlation") return CovDistWs::carve(nullptr, d[0], d[1], G, g).total;
  return 0;
}

// ---- peer-memory versions (k_peer.cu): one push + one consume kernel each
pb_status peer_ready(const pb_peer* p) {
  if (!p || !p->opened) return fail(PB_ERR_INVALID_ARG, "peer group is NULL or not opened");
  int dev = -1;
  cudaGetDevice(&dev);
  if (dev != p->dev) return fail(PB_ERR_INVALID_ARG, "current device %d is not the peer group's device %d", dev, p->dev);
  return PB_OK;
}

// dst (this rank's block) <- sum over ranks of partial. The blocks are row blocks
// (partition tri 0 / align over `rows`) of a rows x cols array; vectors use cols = 1.
pb_status peer_rs(pb_peer* P, const float* partial, float* dst, int rows, int cols, int align, cudaStream_t s) {
  PB_TRY(peer_ready(P));
  long long slot = 0;
  PeerPush push;
  Blk me;
  for (int g = 0; g < P->nranks; ++g) {
    const Blk k = block(rows, P->nranks, g, 0, align);
    if (g == P->rank) me = k;
    slot = std::max<long long>(slot, (long long)k.n() * cols);
  }
  slot = (slot + 3) / 4 * 4;
  if ((size_t)slot * P->nranks * sizeof(float) > P->data_bytes)
    return fail(PB_ERR_WORKSPACE, "peer data region (%zu bytes) < %lld slots of %lld floats", P->data_bytes,
                (long long)P->nranks, slot);
  for (int g = 0; g < P->nranks; ++g) {
    const Blk k = block(rows, P->nranks, g, 0, align);
    push.src[g] = partial + (long long)k.b * cols;
    push.dst_off[g] = (long long)P->rank * slot;
    push.count[g] = (long long)k.n() * cols;
  }
  PeerConsume con;
  con.out = dst;
  con.count = (long long)me.n() * cols;
  con.slot = slot;
  con.reduce = 1;
  PB_CU(launch_peer_push(P->view, push, s));
  PB_CU(launch_peer_consume(P->view, con, s));
  return PB_OK;
}

pb_status peer_ag(pb_peer* P, const float* send_blk, float* recv, int rows, int cols, int align, cudaStream_t s) {
  PB_TRY(peer_ready(P));
  if ((size_t)rows * cols * sizeof(float) > P->data_bytes)
    return fail(PB_ERR_WORKSPACE, "peer data region (%zu bytes) < %d x %d floats", P->data_bytes, rows, cols);
  const Blk me = block(rows, P->nranks, P->rank, 0, align);
  PeerPush push;
  for (int g = 0; g < P->nranks; ++g) {
    push.src[g] = send_blk;
    push.dst_off[g] = (long long)me.b * cols;
    push.count[g] = (long long)me.n() * cols;
  }
  PeerConsume con;
  con.out = recv;
  con.count = (long long)rows * cols;
  con.slot = 0;
  con.reduce = 0;
  PB_CU(launch_peer_push(P->view, push, s));
  PB_CU(launch_peer_consume(P->view, con, s));
  return PB_OK;
}

// dst (this rank's row block, partition tri 0 / `align` over rows, of a rows x cols array)
//   <- sum over ranks of partial[0, rows x cols). Vectors: cols = 1, align 4.
pb_status reduce_scatter_rows(pb_comm* c, const float* partial, float* dst, int rows, int cols, int align,
                              cudaStream_t s) {
  if (c->peer) return peer_rs(c->peer, partial, dst, rows, cols, align, s);
  const Nccl& N = nccl();
  bool equal = true;
  const Blk me = block(rows, c->nranks, c->rank, 0, align);
  for (int g = 0; g < c->nranks; ++g)
    if (block(rows, c->nranks, g, 0, align).n() != me.n()) equal = false;
  if (equal && (long long)me.n() * c->nranks == rows) {
    PB_NC(N.ReduceScatter(partial, dst, (size_t)me.n() * cols, ncclFloat32, ncclSum, c->nc, s));
    return PB_OK;
  }
  PB_NC(N.GroupStart());  // uneven blocks: one reduce per root
  for (int g = 0; g < c->nranks; ++g) {
    const Blk k = block(rows, c->nranks, g, 0, align);
    if (!k.n()) continue;
    const float* src = partial + (long long)k.b * cols;
    float* recv = g == c->rank ? dst : const_cast<float*>(src);  // only the root's is written
    const ncclResult_t r = N.Reduce(src, recv, (size_t)k.n() * cols, ncclFloat32, ncclSum, g, c->nc, s);
    if (r != ncclSuccess) {
      N.GroupEnd();
      return nc_check(r, "ncclReduce");
    }
  }
  PB_NC(N.GroupEnd());
  return PB_OK;
}
pb_status reduce_scatter(pb_comm* c, const float* partial, float* dst, int total, cudaStream_t s) {
  return reduce_scatter_rows(c, partial, dst, total, 1, ALIGN_MV, s);
}

// Every rank's rows of F (rows x cols, partition tri 0 / align 128) -> the full F, in place.
pb_status all_gather_rows(pb_comm* c, float* F, int rows, int cols, cudaStream_t s, int align = ALIGN_MM) {
  if (c->peer) {
    const Blk me = block(rows, c->nranks, c->rank, 0, align);
    return peer_ag(c->peer, F + (size_t)me.b * cols, F, rows, cols, align, s);
  }
  const Nccl& N = nccl();
  bool equal = true;
  const Blk me = block(rows, c->nranks, c->rank, 0, align);
  for (int g = 0; g < c->nranks; ++g)
    if (block(rows, c->nranks, g, 0, align).n() != me.n()) equal = false;
  if (equal && (long long)me.n() * c->nranks == rows) {  // in place: send = recv + rank * count
    const size_t cnt = (size_t)me.n() * cols;
    PB_NC(N.AllGather(F + (size_t)me.b * cols, F, cnt, ncclFloat32, c->nc, s));
    return PB_OK;
  }
  PB_NC(N.GroupStart());  // uneven blocks: one broadcast per owner
  for (int g = 0; g < c->nranks; ++g) {
    const Blk k = block(rows, c->nranks, g, 0, align);
    if (!k.n()) continue;
    float* p = F + (size_t)k.b * cols;
    const ncclResult_t r = N.Broadcast(p, p, (size_t)k.n() * cols, ncclFloat32, g, c->nc, s);
    if (r != ncclSuccess) {
      N.GroupEnd();
      return nc_check(r, "ncclBroadcast");
    }
  }
  PB_NC(N.GroupEnd());
  return PB_OK;
}

pb_status check_dist_ws(const DistWs& w, void* ws, size_t ws_bytes) {
  if (w.total == 0) return PB_OK;
  if (!ws) return fail(PB_ERR_WORKSPACE, "workspace is NULL (need %zu bytes)", w.total);
  if (reinterpret_cast<uintptr_t>(ws) % 256) return fail(PB_ERR_WORKSPACE, "workspace not 256-byte aligned");
  if (ws_bytes < w.total) return fail(PB_ERR_WORKSPACE, "workspace has %zu bytes, need %zu", ws_bytes, w.total);
  return PB_OK;
}

}  // namespace

namespace pb {
// pb_workspace_size for "<k>_dist": the kernel's dims followed by {nranks, rank}.
pb_status dist_workspace_size(const std::string& name, const long long* d, int nd, size_t* bytes) {
  const std::string k = name.substr(0, name.size() - 5);
  const int nk = k == "gemm" ? 3 : k == "2mm" ? 4 : k == "3mm" ? 5 : (k == "syrk" || k == "syr2k") ? 2
               : (k == "atax" || k == "bicg") ? 2 : (k == "mvt" || k == "gesummv") ? 1
               : (k == "covariance" || k == "correlation") ? 2 : -1;
  if (nk < 0 || nd != nk + 2) return fail(PB_ERR_INVALID_ARG, "unknown kernel '%s' or wrong dims (%d)", name.c_str(), nd);
  for (int i = 0; i < nk; ++i)
    if (d[i] <= 0 || d[i] > (1ll << 30)) return fail(PB_ERR_INVALID_ARG, "dimension %d is %lld", i, d[i]);
  const long long G = d[nk], g = d[nk + 1];
  if (G <= 0 || g < 0 || g >= G) return fail(PB_ERR_INVALID_ARG, "bad nranks/rank %lld/%lld", G, g);
  const size_t loc = local_need(k, d, (int)G, (int)g);
  long long plen = 0, blen = 0;
  if (k == "atax") plen = d[1];
  if (k == "bicg") plen = d[0];
  if (k == "mvt") plen = blen = d[0];
  *bytes = align_up(dist_ws(nullptr, 0, plen, blen, loc).total, 256);
  return PB_OK;
}
}  // namespace pb

extern "C" {

pb_status pb_comm_unique_id(unsigned char id[128]) {
  if (!id) return fail(PB_ERR_INVALID_ARG, "id is NULL");
  PB_TRY(nccl_loaded());
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId is 128 bytes");
  ncclUniqueId u;
  PB_NC(nccl().GetUniqueId(&u));
  memcpy(id, &u, 128);
  return PB_OK;
}

pb_status pb_comm_init(int nranks, int rank, const unsigned char id[128], pb_comm** out) {
  if (!id || !out || nranks <= 0 || rank < 0 || rank >= nranks)
    return fail(PB_ERR_INVALID_ARG, "bad comm arguments (nranks %d, rank %d)", nranks, rank);
  PB_TRY(nccl_loaded());
  pb_comm* c = new pb_comm;
  c->nranks = nranks;
  c->rank = rank;
  cudaGetDevice(&c->dev);
  ncclUniqueId u;
  memcpy(&u, id, 128);
  pb_status st = nc_check(nccl().CommInitRank(&c->nc, nranks, u, rank), "ncclCommInitRank");
  if (st == PB_OK) st = cu_check(cudaStreamCreateWithFlags(&c->side, cudaStreamNonBlocking), "side stream");
  if (st == PB_OK) st = cu_check(cudaEventCreateWithFlags(&c->ev_ready, cudaEventDisableTiming), "event");
  if (st == PB_OK) st = cu_check(cudaEventCreateWithFlags(&c->ev_done, cudaEventDisableTiming), "event");
  if (st != PB_OK) {
    pb_comm_destroy(c);
    return st;
  }
  *out = c;
  return PB_OK;
}

pb_status pb_comm_destroy(pb_comm* c) {
  if (!c) return PB_OK;
  pb_status st = PB_OK;
  if (c->nc) st = nc_check(nccl().CommDestroy(c->nc), "ncclCommDestroy");
  if (c->ev_ready) cudaEventDestroy(c->ev_ready);
  if (c->ev_done) cudaEventDestroy(c->ev_done);
  if (c->side) cudaStreamDestroy(c->side);
  delete c;
  return st;
}

pb_status pb_comm_size(const pb_comm* c, int* nranks, int* rank) {
  if (!c || !nranks || !rank) return fail(PB_ERR_INVALID_ARG, "NULL argument");
  *nranks = c->nranks;
  *rank = c->rank;
  return PB_OK;
}

pb_status pb_comm_init_local(int nranks, int rank, pb_comm** out) {
  if (!out || nranks <= 0 || rank < 0 || rank >= nranks)
    return fail(PB_ERR_INVALID_ARG, "bad comm arguments (nranks %d, rank %d)", nranks, rank);
  pb_comm* c = new pb_comm;
  c->nranks = nranks;
  c->rank = rank;
  cudaGetDevice(&c->dev);
  pb_status st = cu_check(cudaStreamCreateWithFlags(&c->side, cudaStreamNonBlocking), "side stream");
  if (st == PB_OK) st = cu_check(cudaEventCreateWithFlags(&c->ev_ready, cudaEventDisableTiming), "event");
  if (st == PB_OK) st = cu_check(cudaEventCreateWithFlags(&c->ev_done, cudaEventDisableTiming), "event");
  if (st != PB_OK) {
    pb_comm_destroy(c);
    return st;
  }
  *out = c;
  return PB_OK;
}

pb_status pb_comm_attach_peer(pb_comm* c, pb_peer* p) {
  if (!c) return fail(PB_ERR_INVALID_ARG, "comm is NULL");
  if (p && (p->nranks != c->nranks || p->rank != c->rank || !p->opened))
    return fail(PB_ERR_INVALID_ARG, "peer group does not match the comm (or is not opened)");
  c->peer = p;
  return PB_OK;
}

pb_status pb_peer_create(int nranks, int rank, size_t data_bytes, pb_peer** out, unsigned char handle[64]) {
  if (!out || !handle || nranks <= 0 || nranks > PEER_MAXR || rank < 0 || rank >= nranks)
    return fail(PB_ERR_INVALID_ARG, "bad peer arguments (nranks %d (max %d), rank %d)", nranks, PEER_MAXR, rank);
  static_assert(sizeof(cudaIpcMemHandle_t) == 64, "cudaIpcMemHandle_t is 64 bytes");
  pb_peer* p = new pb_peer;
  p->nranks = nranks;
  p->rank = rank;
  p->data_bytes = (data_bytes + 255) / 256 * 256;
  cudaGetDevice(&p->dev);
  pb_status st = cu_check(cudaMalloc(&p->base, PEER_HDR + p->data_bytes), "cudaMalloc (peer buffer)");
  if (st == PB_OK) st = cu_check(cudaMemset(p->base, 0, PEER_HDR), "cudaMemset (peer header)");
  cudaIpcMemHandle_t h;
  if (st == PB_OK) st = cu_check(cudaIpcGetMemHandle(&h, p->base), "cudaIpcGetMemHandle");
  if (st != PB_OK) {
    pb_peer_destroy(p);
    return st;
  }
  memcpy(handle, &h, 64);
  *out = p;
  return PB_OK;
}

pb_status pb_peer_open(pb_peer* p, const unsigned char* handles) {
  if (!p || !handles) return fail(PB_ERR_INVALID_ARG, "NULL argument");
  if (p->opened) return fail(PB_ERR_INVALID_ARG, "peer group already opened");
  for (int g = 0; g < p->nranks; ++g) {
    if (g == p->rank) {
      p->mapped[g] = p->base;
      continue;
    }
    cudaIpcMemHandle_t h;
    memcpy(&h, handles + 64 * (size_t)g, 64);
    void* ptr = nullptr;
    PB_CU(cudaIpcOpenMemHandle(&ptr, h, cudaIpcMemLazyEnablePeerAccess));
    p->mapped[g] = static_cast<char*>(ptr);
  }
  PeerView& v = p->view;
  v.nranks = p->nranks;
  v.rank = p->rank;
  for (int g = 0; g < p->nranks; ++g) {  // header: flags @0, acks @512, counters @1024, status @1536, epoch @1600
    v.data[g] = reinterpret_cast<float*>(p->mapped[g] + PEER_HDR);
    v.flags[g] = reinterpret_cast<unsigned long long*>(p->mapped[g]);
    v.acks[g] = reinterpret_cast<unsigned long long*>(p->mapped[g] + 512);
  }
  v.flags_mine = v.flags[p->rank];
  v.acks_mine = v.acks[p->rank];
  v.counter = reinterpret_cast<unsigned*>(p->base + 1024);
  v.status = reinterpret_cast<unsigned*>(p->base + 1536);
  v.epoch = reinterpret_cast<unsigned long long*>(p->base + 1600);
  p->opened = true;
  return PB_OK;
}

pb_status pb_peer_destroy(pb_peer* p) {
  if (!p) return PB_OK;
  for (int g = 0; g < p->nranks; ++g)
    if (g != p->rank && p->mapped[g]) cudaIpcCloseMemHandle(p->mapped[g]);
  if (p->base) cudaFree(p->base);
  delete p;
  return PB_OK;
}

pb_status pb_peer_status(const pb_peer* p, unsigned* status) {
  if (!p || !status) return fail(PB_ERR_INVALID_ARG, "NULL argument");
  PB_CU(cudaMemcpy(status, p->base + 1536, sizeof(unsigned), cudaMemcpyDeviceToHost));
  return PB_OK;
}

pb_status pb_peer_reduce_scatter(pb_peer* p, const float* partial, float* out_blk, int total, pb_stream s) {
  if (total <= 0 || total % 4) return fail(PB_ERR_UNSUPPORTED, "total %d must be a positive multiple of 4", total);
  set_launches(2);
  return peer_rs(p, partial, out_blk, total, 1, ALIGN_MV, S(s));
}

pb_status pb_peer_all_gather(pb_peer* p, const float* send_blk, float* recv, int rows, int cols, pb_stream s) {
  if (rows <= 0 || cols <= 0 || cols % 4) return fail(PB_ERR_UNSUPPORTED, "rows %d, cols %d (multiple of 4)", rows, cols);
  set_launches(2);
  return peer_ag(p, send_blk, recv, rows, cols, ALIGN_MM, S(s));
}

// ---- no exchange: the local entry point on this rank's rows
pb_status pb_gemm_dist(pb_comm* c, int ni, int nj, int nk, float alpha, float beta, float* C_blk, const float* A_blk,
                       const float* B, void* ws, size_t ws_bytes, pb_stream s) {
  PB_TRY(comm_ok(c));
  if (ni <= 0) return fail(PB_ERR_INVALID_ARG, "ni %d", ni);
  const Blk r = block(ni, c->nranks, c->rank, 0, ALIGN_MM);
  set_launches(0);
  return r.n() ? pb_gemm(r.n(), nj, nk, alpha, beta, C_blk, A_blk, B, ws, ws_bytes, s) : PB_OK;
}

pb_status pb_2mm_dist(pb_comm* c, int ni, int nj, int nk, int nl, float alpha, float beta, float* tmp_blk,
                      const float* A_blk, const float* B, const float* C, float* D_blk, void* ws, size_t ws_bytes,
                      pb_stream s) {
  PB_TRY(comm_ok(c));
  if (ni <= 0) return fail(PB_ERR_INVALID_ARG, "ni %d", ni);
  const Blk r = block(ni, c->nranks, c->rank, 0, ALIGN_MM);
  set_launches(0);
  return r.n() ? pb_2mm(r.n(), nj, nk, nl, alpha, beta, tmp_blk, A_blk, B, C, D_blk, ws, ws_bytes, s) : PB_OK;
}

pb_status pb_syrk_dist(pb_comm* c, int n, int m, float alpha, float beta, float* C_blk, const float* A, void* ws,
                       size_t ws_bytes, pb_stream s) {
  PB_TRY(comm_ok(c));
  if (n <= 0) return fail(PB_ERR_INVALID_ARG, "n %d", n);
  const Blk r = block(n, c->nranks, c->rank, 2, ALIGN_SY);
  set_launches(0);
  return r.n() ? pb_syrk_rows(n, m, r.b, r.e, alpha, beta, C_blk, A, ws, ws_bytes, s) : PB_OK;
}

pb_status pb_syr2k_dist(pb_comm* c, int n, int m, float alpha, float beta, float* C_blk, const float* A,
                        const float* B, void* ws, size_t ws_bytes, pb_stream s) {
  PB_TRY(comm_ok(c));
  if (n <= 0) return fail(PB_ERR_INVALID_ARG, "n %d", n);
  const Blk r = block(n, c->nranks, c->rank, 2, ALIGN_SY);
  set_launches(0);
  return r.n() ? pb_syr2k_rows(n, m, r.b, r.e, alpha, beta, C_blk, A, B, ws, ws_bytes, s) : PB_OK;
}

pb_status pb_gesummv_dist(pb_comm* c, int n, float alpha, float beta, const float* A_blk, const float* B_blk,
                          float* tmp_blk, const float* x, float* y_blk, void* ws, size_t ws_bytes, pb_stream s) {
  PB_TRY(comm_ok(c));
  if (n <= 0) return fail(PB_ERR_INVALID_ARG, "n %d", n);
  const Blk r = block(n, c->nranks, c->rank, 0, ALIGN_MV);
  set_launches(0);
  return r.n() ? pb_gesummv_rows(r.n(), n, alpha, beta, A_blk, B_blk, tmp_blk, x, y_blk, ws, ws_bytes, s) : PB_OK;
}

// ---- 3mm: F rows -> all-gather (side stream) || E rows -> G rows
pb_status pb_3mm_dist(pb_comm* c, int ni, int nj, int nk, int nl, int nm, float* E_blk, const float* A_blk,
                      const float* B, float* F, const float* C_blk, const float* D, float* G_blk, void* ws,
                      size_t ws_bytes, pb_stream s) {
  PB_TRY(comm_ok(c));
  const Blk r = block(ni > 0 ? ni : 1, c->nranks, c->rank, 0, ALIGN_MM);
  const Blk f = block(nj > 0 ? nj : 1, c->nranks, c->rank, 0, ALIGN_MM);
  Check ck;  // everything validated before anything is enqueued
  ck.dims({ni, nj, nk, nl, nm});
  ck.cols4(nj, "B/E"); ck.cols4(nk, "A"); ck.cols4(nl, "D/F/G"); ck.cols4(nm, "C");
  ck.arr(E_blk, r.n(), nj, true, "E_blk", r.n() > 0); ck.arr(A_blk, r.n(), nk, false, "A_blk", r.n() > 0);
  ck.arr(B, nk, nj, false, "B"); ck.arr(F, nj, nl, true, "F"); ck.arr(C_blk, f.n(), nm, false, "C_blk", f.n() > 0);
  ck.arr(D, nm, nl, false, "D"); ck.arr(G_blk, r.n(), nl, true, "G_blk", r.n() > 0);
  PB_TRY(ck.finish());
  const long long dims[7] = {ni, nj, nk, nl, nm, c->nranks, c->rank};
  const DistWs w = dist_ws(ws, ws_bytes, 0, 0, local_need("3mm", dims, c->nranks, c->rank));
  PB_TRY(check_dist_ws(w, ws, ws_bytes));
  const cudaStream_t st = S(s);
  int L = 0;
  if (f.n()) {
    PB_TRY(pb_gemm(f.n(), nl, nm, 1.f, 0.f, F + (size_t)f.b * nl, C_blk, D, w.local, w.local_bytes, s));
    L += pb_last_launch_count();
  }
  PB_CU(cudaEventRecord(c->ev_ready, st));
  PB_CU(cudaStreamWaitEvent(c->side, c->ev_ready, 0));
  PB_TRY(all_gather_rows(c, F, nj, nl, c->side));
  if (c->peer) L += 2;
  PB_CU(cudaEventRecord(c->ev_done, c->side));
  if (r.n()) {  // E = A B overlaps the all-gather
    PB_TRY(pb_gemm(r.n(), nj, nk, 1.f, 0.f, E_blk, A_blk, B, w.local, w.local_bytes, s));
    L += pb_last_launch_count();
  }
  PB_CU(cudaStreamWaitEvent(st, c->ev_done, 0));
  if (r.n()) {
    PB_TRY(pb_gemm(r.n(), nl, nj, 1.f, 0.f, G_blk, E_blk, F, w.local, w.local_bytes, s));
    L += pb_last_launch_count();
  }
  set_launches(L);
  return PB_OK;
}

// ---- atax / bicg / mvt: local partial of the transposed product -> reduce-scatter
pb_status pb_atax_dist(pb_comm* c, int m, int n, const float* A_blk, const float* x, float* y_blk, float* tmp_blk,
                       void* ws, size_t ws_bytes, pb_stream s) {
  PB_TRY(comm_ok(c));
  const Blk r = block(m > 0 ? m : 1, c->nranks, c->rank, 0, ALIGN_MV);
  const Blk o = block(n > 0 ? n : 1, c->nranks, c->rank, 0, ALIGN_MV);
  Check ck;
  ck.dims({m, n});
  ck.cols4(n, "A");
  ck.arr(A_blk, r.n(), n, false, "A_blk", r.n() > 0); ck.arr(x, 1, n, false, "x");
  ck.arr(y_blk, 1, o.n(), true, "y_blk", o.n() > 0); ck.arr(tmp_blk, 1, r.n(), true, "tmp_blk", false);
  PB_TRY(ck.finish());
  const long long dims[4] = {m, n, c->nranks, c->rank};
  const DistWs w = dist_ws(ws, ws_bytes, n, 0, local_need("atax", dims, c->nranks, c->rank));
  PB_TRY(check_dist_ws(w, ws, ws_bytes));
  int L = 0;
  if (r.n()) {  // single pass over A_blk: tmp = A_blk x, partial = A_blk^T tmp
    PB_TRY(pb_atax(r.n(), n, A_blk, x, w.partial, tmp_blk, w.local, w.local_bytes, s));
    L = pb_last_launch_count();
  } else {
    PB_CU(cudaMemsetAsync(w.partial, 0, sizeof(float) * n, S(s)));
  }
  PB_TRY(reduce_scatter(c, w.partial, y_blk, n, S(s)));
  set_launches(L + (c->peer ? 2 : 0));
  return PB_OK;
}

pb_status pb_bicg_dist(pb_comm* c, int m, int n, const float* A_blk, float* s_blk, float* q_blk, const float* p,
                       const float* r_blk, void* ws, size_t ws_bytes, pb_stream s) {
  PB_TRY(comm_ok(c));
  const Blk r = block(n > 0 ? n : 1, c->nranks, c->rank, 0, ALIGN_MV);
  const Blk o = block(m > 0 ? m : 1, c->nranks, c->rank, 0, ALIGN_MV);
  Check ck;
  ck.dims({m, n});
  ck.cols4(m, "A");
  ck.arr(A_blk, r.n(), m, false, "A_blk", r.n() > 0); ck.arr(s_blk, 1, o.n(), true, "s_blk", o.n() > 0);
  ck.arr(q_blk, 1, r.n(), true, "q_blk", r.n() > 0); ck.arr(p, 1, m, false, "p");
  ck.arr(r_blk, 1, r.n(), false, "r_blk", r.n() > 0);
  PB_TRY(ck.finish());
  const long long dims[4] = {m, n, c->nranks, c->rank};
  const DistWs w = dist_ws(ws, ws_bytes, m, 0, local_need("bicg", dims, c->nranks, c->rank));
  PB_TRY(check_dist_ws(w, ws, ws_bytes));
  int L = 0;
  if (r.n()) {  // q_blk = A_blk p, partial = A_blk^T r_blk (one pass)
    PB_TRY(pb_bicg(m, r.n(), A_blk, w.partial, q_blk, p, r_blk, w.local, w.local_bytes, s));
    L = pb_last_launch_count();
  } else {
    PB_CU(cudaMemsetAsync(w.partial, 0, sizeof(float) * m, S(s)));
  }
  PB_TRY(reduce_scatter(c, w.partial, s_blk, m, S(s)));
  set_launches(L + (c->peer ? 2 : 0));
  return PB_OK;
}

pb_status pb_mvt_dist(pb_comm* c, int n, float* x1_blk, float* x2_blk, const float* y_1, const float* y_2_blk,
                      const float* A_blk, void* ws, size_t ws_bytes, pb_stream s) {
  PB_TRY(comm_ok(c));
  const Blk r = block(n > 0 ? n : 1, c->nranks, c->rank, 0, ALIGN_MV);
  Check ck;
  ck.dims({n});
  ck.cols4(n, "A");
  ck.arr(x1_blk, 1, r.n(), true, "x1_blk", r.n() > 0); ck.arr(x2_blk, 1, r.n(), true, "x2_blk", r.n() > 0);
  ck.arr(y_1, 1, n, false, "y_1"); ck.arr(y_2_blk, 1, r.n(), false, "y_2_blk", r.n() > 0);
  ck.arr(A_blk, r.n(), n, false, "A_blk", r.n() > 0);
  PB_TRY(ck.finish());
  const long long dims[3] = {n, c->nranks, c->rank};
  const DistWs w = dist_ws(ws, ws_bytes, n, n, local_need("mvt", dims, c->nranks, c->rank));
  PB_TRY(check_dist_ws(w, ws, ws_bytes));
  const cudaStream_t st = S(s);
  // base = x2's old value at this rank's rows, 0 elsewhere: the reduce-scatter then
  // yields x2 + A^T y_2 for every block.
  PB_CU(cudaMemsetAsync(w.base, 0, sizeof(float) * n, st));
  if (r.n()) PB_CU(cudaMemcpyAsync(w.base + r.b, x2_blk, sizeof(float) * r.n(), cudaMemcpyDeviceToDevice, st));
  int L = 0;
  if (r.n()) {  // x1_blk += A_blk y_1, partial = base + A_blk^T y_2_blk (one pass)
    PB_TRY(pb_matvec_partial(r.n(), n, A_blk, y_1, x1_blk, x1_blk, y_2_blk, w.base, w.partial, w.local,
                             w.local_bytes, s));
    L = pb_last_launch_count();
  } else {
    PB_CU(cudaMemsetAsync(w.partial, 0, sizeof(float) * n, st));
  }
  PB_TRY(reduce_scatter(c, w.partial, x2_blk, n, st));
  set_launches(L + (c->peer ? 2 : 0));
  return PB_OK;
}

// ---- covariance / correlation: observations split (k_covdist.cu)
// Rank g holds observations o = block(n, G, g, 0, 32) of data; it returns rows
// block(m, G, g, 0, 32) of the m x m result, plus the full mean (and stddev) vectors.
static pb_status covcorr_dist(bool corr, pb_comm* c, int m, int n, float float_n, float eps, const float* data_blk,
                              float* out_blk, float* mean, float* stddev, void* ws, size_t ws_bytes, pb_stream s) {
  PB_TRY(comm_ok(c));
  Check ck;
  ck.dims({m, n});
  if (ck.st == PB_OK && !corr && n < 2) ck.st = fail(PB_ERR_INVALID_ARG, "covariance needs n >= 2");
  if (ck.st == PB_OK && !(float_n > 0.f)) ck.st = fail(PB_ERR_INVALID_ARG, "float_n must be > 0");
  if (ck.st == PB_OK && !corr && float_n == 1.0f) ck.st = fail(PB_ERR_INVALID_ARG, "float_n - 1 == 0");
  ck.cols4(m, "data/out");
  const Blk o = block(n > 0 ? n : 1, c->nranks, c->rank, 0, ALIGN_OBS);
  const Blk r = block(m > 0 ? m : 1, c->nranks, c->rank, 0, ALIGN_ST);
  ck.arr(data_blk, o.n(), m, false, "data_blk", o.n() > 0);
  ck.arr(out_blk, r.n(), m, true, corr ? "corr_blk" : "cov_blk", r.n() > 0);
  ck.arr(mean, 1, m, true, "mean", false);
  if (corr) ck.arr(stddev, 1, m, true, "stddev", false);
  PB_TRY(ck.finish());
  const CovDistWs need = CovDistWs::carve(nullptr, m, n, c->nranks, c->rank);
  if (!ws) return fail(PB_ERR_WORKSPACE, "workspace is NULL (need %zu bytes)", need.total);
  if (reinterpret_cast<uintptr_t>(ws) % 256) return fail(PB_ERR_WORKSPACE, "workspace not 256-byte aligned");
  if (ws_bytes < need.total) return fail(PB_ERR_WORKSPACE, "workspace has %zu bytes, need %zu", ws_bytes, need.total);
  const CovDistWs w = CovDistWs::carve(ws, m, n, c->nranks, c->rank);
  const cudaStream_t st = S(s);
  int L = 0;
  // 1. this rank's column sums into its row of the gather buffer (4m floats per rank)
  double* mine = w.sums + (size_t)c->rank * 2 * m;
  if (o.n()) {
    PB_CU(launch_obs_sums(data_blk, o.n(), m, mine, st));
  } else {
    PB_CU(cudaMemsetAsync(mine, 0, (size_t)2 * m * sizeof(double), st));
  }
  ++L;
  // 2. "allreduce of column sums": gather every rank's sums (bit copies), summed in rank order
  //    by every rank in step 3, so all ranks hold the same mean / stddev bits
  PB_TRY(all_gather_rows(c, reinterpret_cast<float*>(w.sums), c->nranks, 4 * m, st, 1));
  if (c->peer) L += 2;
  // 3 + 4. statistics, centred transpose, local partial Gram P_g = Yt Yt^T (full square)
  if (o.n()) {
    PB_CU(launch_obs_center_t(corr, data_blk, o.n(), m, w.sums, c->nranks, n, (double)float_n, (double)eps, w.Yt,
                              w.ldy, mean, stddev, st));
    ++L;
    PB_TRY(pb_syrk_full(m, w.ldy, 1.f, 0.f, w.P, w.Yt, w.gemm, w.gemm_bytes, s));
    L += pb_last_launch_count();
  } else {
    // no observations here: P_g = 0; mean / stddev still come from the gathered sums
    if (mean || stddev) {
      PB_CU(launch_obs_center_t(corr, nullptr, 0, m, w.sums, c->nranks, n, (double)float_n, (double)eps, nullptr, 0,
                                mean, stddev, st));
      ++L;
    }
    PB_CU(cudaMemsetAsync(w.P, 0, (size_t)m * m * sizeof(float), st));
  }
  // 5. P = sum_g P_g, reduce-scattered into the output row bands
  PB_TRY(reduce_scatter_rows(c, w.P, out_blk, m, m, ALIGN_ST, st));
  if (c->peer) L += 2;
  // 6. 1 / (float_n - 1) (covariance) or diagonal := 1 (correlation)
  if (r.n()) {
    PB_CU(launch_obs_finish(corr, out_blk, r.n(), m, r.b, (float)(1.0 / ((double)float_n - 1.0)), st));
    ++L;
  }
  set_launches(L);
  return PB_OK;
}

pb_status pb_covariance_dist(pb_comm* c, int m, int n, float float_n, const float* data_blk, float* cov_blk,
                             float* mean, void* ws, size_t ws_bytes, pb_stream s) {
  return covcorr_dist(false, c, m, n, float_n, 0.f, data_blk, cov_blk, mean, nullptr, ws, ws_bytes, s);
}

pb_status pb_correlation_dist(pb_comm* c, int m, int n, float float_n, float eps, const float* data_blk,
                              float* corr_blk, float* mean, float* stddev, void* ws, size_t ws_bytes, pb_stream s) {
  return covcorr_dist(true, c, m, n, float_n, eps, data_blk, corr_blk, mean, stddev, ws, ws_bytes, s);
}

}  // extern "C"

