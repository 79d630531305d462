// pb_api.cu — the C ABI of libpb (include/pb.h): argument validation, alias
// checks, workspace carving and the launch sequence of each PolyBench kernel.
// Every arithmetic step runs in the kernels of k_*.cu; this file only decides
// what to launch. There is no CPU fallback: a missing/failed launch returns an
// error.
#include <stdarg.h>
#include <stdio.h>
#include <string.h>

#include <algorithm>
#include <cmath>
#include <map>
#include <string>
#include <vector>

#include "../../include/pb.h"
#include "pb_check.h"
#include "pb_internal.h"

using namespace pb;

namespace {

thread_local std::string g_err;
thread_local int g_launches = 0;

}  // namespace

namespace pb {
pb_status fail(pb_status st, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_err = std::string(pb_status_str(st)) + ": " + buf;
  return st;
}

void set_launches(int n) { g_launches = n; }
}  // namespace pb

namespace {
inline size_t fsz(long long rows, long long cols) { return (size_t)rows * (size_t)cols; }

// ---- workspace layouts (shared by pb_workspace_size and the entry points) ----
struct SplitBuf {
  float* hi;
  float* lo;
  int rows, K, ld;
  SplitOperand op() const {
    SplitOperand o;
    o.hi = hi; o.lo = lo; o.rows = rows; o.K = K; o.ld = ld;
    return o;
  }
};
// raw-hi operand: only the lo array is carved; op_raw(X) pairs it with the caller's X
struct LoBuf {
  float* lo;
  int rows, K, ld;
  SplitOperand op_raw(const float* X) const {
    SplitOperand o;
    o.hi = X; o.lo = lo; o.rows = rows; o.K = K; o.ld = ld;
    return o;
  }
};
LoBuf take_lo(Carve& c, int rows, int K) {
  LoBuf b;
  b.rows = rows;
  b.K = K;
  b.ld = round_up(K, 4);
  b.lo = c.take<float>(fsz(rows, b.ld));
  return b;
}
// MN-major B operand (B[k][n] as the caller stores it, K x N): lo of the same layout
struct LoBufMN {
  float* lo;
  int N, K;
  SplitOperand op_raw(const float* B) const {
    SplitOperand o;
    o.hi = B; o.lo = lo; o.rows = N; o.K = K; o.ld = N; o.mn = true;
    return o;
  }
};
LoBufMN take_lo_mn(Carve& c, int K, int N) {
  LoBufMN b;
  b.N = N;
  b.K = K;
  b.lo = c.take<float>(fsz(K, N));
  return b;
}
SplitBuf take_split(Carve& c, int rows, int K) {
  SplitBuf b;
  b.rows = rows;
  b.K = K;
  b.ld = round_up(K, 4);
  b.hi = c.take<float>(fsz(rows, b.ld));
  b.lo = c.take<float>(fsz(rows, b.ld));
  return b;
}

// Split-K scratch shared by the GEMMs of one call (they run in stream order).
struct SplitK {
  float* part = nullptr;
  unsigned* counters = nullptr;
  size_t part_bytes = 0, counter_bytes = 0;
  void attach(GemmDesc& d) const {
    d.part = part; d.counters = counters; d.part_cap = part_bytes; d.counter_cap = counter_bytes;
  }
};
GemmDesc shape(int M, int N, int K, int npairs = 1, uint32_t flags = EPI_OUT, int tm0 = 0, int tm1 = -1) {
  GemmDesc d;
  d.M = M; d.N = N; d.K = K; d.npairs = npairs; d.flags = flags; d.tm0 = tm0; d.tm1 = tm1;
  return d;
}
SplitK take_splitk(Carve& c, std::initializer_list<GemmDesc> gemms) {
  size_t part = 0, cnt = 0;
  for (const GemmDesc& g : gemms) {
    const UmmaPlan pl = umma_plan(g);
    part = std::max(part, pl.part_bytes);
    cnt = std::max(cnt, pl.counter_bytes);
  }
  SplitK k;
  if (part) {
    k.part = c.take<float>(part / sizeof(float));
    k.counters = c.take<unsigned>(cnt / sizeof(unsigned));
    k.part_bytes = part;
    k.counter_bytes = cnt;
  }
  return k;
}

struct WsGemm { LoBuf a; LoBufMN b; SplitK sk; };
WsGemm ws_gemm(Carve& c, int ni, int nj, int nk) {
  WsGemm w;
  w.a = take_lo(c, ni, nk); w.b = take_lo_mn(c, nk, nj);
  w.sk = take_splitk(c, {shape(ni, nj, nk)});
  return w;
}
// chain fusion (NEXT-4): each phase of the one-launch chain has its own split-K area (the
// phases' split tiles can be live at the same time) plus the readiness counters
struct ChainWs {
  unsigned* cnt = nullptr;
  size_t cnt_bytes = 0;
};
ChainWs take_chain(Carve& c, std::initializer_list<GemmDesc> gemms) {
  ChainWs w;
  w.cnt_bytes = umma_chain_cnt_bytes(gemms.begin(), (int)gemms.size());
  w.cnt = c.take<unsigned>(w.cnt_bytes / sizeof(unsigned));
  return w;
}
// raw-hi operands: A, tmp K-major (lo of the same layout), B, C MN-major (lo of B[k][n], C[k][n]);
// tmp_out holds tmp when the caller passes none (GEMM 2 reads it as its hi operand)
struct Ws2mm { LoBuf a, tmp; LoBufMN b, c; float* tmp_out; SplitK sk, sk2; ChainWs chain; };
Ws2mm ws_2mm(Carve& c, int ni, int nj, int nk, int nl) {
  Ws2mm w;
  w.a = take_lo(c, ni, nk); w.b = take_lo_mn(c, nk, nj); w.c = take_lo_mn(c, nj, nl); w.tmp = take_lo(c, ni, nj);
  w.tmp_out = c.take<float>(fsz(ni, nj));
  w.sk = take_splitk(c, {shape(ni, nj, nk), shape(ni, nl, nj)});
  w.sk2 = take_splitk(c, {shape(ni, nl, nj)});
  w.chain = take_chain(c, {shape(ni, nj, nk), shape(ni, nl, nj)});
  return w;
}
// raw-hi operands: A, C, E K-major; B, D, F MN-major (F = G's B operand as stored, no transpose)
struct Ws3mm { LoBuf a, c, e; LoBufMN b, d, f; SplitK sk, sk2, sk3; ChainWs chain; };
Ws3mm ws_3mm(Carve& c, int ni, int nj, int nk, int nl, int nm) {
  Ws3mm w;
  w.a = take_lo(c, ni, nk); w.b = take_lo_mn(c, nk, nj); w.c = take_lo(c, nj, nm);
  w.d = take_lo_mn(c, nm, nl); w.e = take_lo(c, ni, nj); w.f = take_lo_mn(c, nj, nl);
  w.sk = take_splitk(c, {shape(nj, nl, nm), shape(ni, nj, nk), shape(ni, nl, nj)});
  w.sk2 = take_splitk(c, {shape(ni, nj, nk)});
  w.sk3 = take_splitk(c, {shape(ni, nl, nj)});
  w.chain = take_chain(c, {shape(nj, nl, nm), shape(ni, nj, nk), shape(ni, nl, nj)});
  return w;
}
// covariance/correlation: n <= MAX_BANDED rows use the banded single-pass prep
// (band-centred operand + between-band scatter in the combine, reading R18);
// longer columns use the exact two-phase prep (mean first, then centre).
constexpr int MAX_BANDED = 8 * 256;
inline bool banded_stats(int n) { return n <= MAX_BANDED; }
struct WsStat { SplitBuf xt; SplitK sk; double* band_mean = nullptr; double* band_m2 = nullptr; };
WsStat ws_stat(Carve& c, int m, int n) {
  WsStat w;
  const size_t off0 = c.off;
  w.xt = take_split(c, m, n);
  const bool banded = banded_stats(n);
  // The exact-mean path (n > MAX_BANDED) switches to EPI_PARTIAL when its plan splits K
  // (stat_core), which re-plans with every tile through partials and possibly another
  // tile shape: reserve the larger of the two plans.
  if (banded)
    w.sk = take_splitk(c, {shape(m, m, n, 1, EPI_TRI | EPI_PARTIAL)});
  else
    w.sk = take_splitk(c, {shape(m, m, n, 1, EPI_TRI), shape(m, m, n, 1, EPI_TRI | EPI_PARTIAL)});
  if (banded) {
    w.band_mean = c.take<double>((size_t)band_count(n) * m);
    w.band_m2 = c.take<double>((size_t)band_count(n) * m);
  }
  // the fused one-launch path (k_gram.cu) carves the same region its own way: reserve
  // the larger of the two layouts
  if (n <= MAX_BANDED && m <= 2048) c.off = std::max(c.off, align_up(off0, 256) + gram_fused_ws_bytes(m, n));
  return w;
}
// covariance/correlation row band [r0, r1) (multi-GPU: replicated data, output row
// blocks, no exchange): exact-mean prep of all m variables + a full-width GEMM.
struct WsStatRows { SplitBuf xt; SplitK sk; };
WsStatRows ws_stat_rows(Carve& c, int m, int n, int r0, int r1) {
  WsStatRows w;
  w.xt = take_split(c, m, n);
  w.sk = take_splitk(c, {shape(r1, m, n, 1, EPI_OUT, r0 / 128, (r1 + 127) / 128)});
  return w;
}
struct WsSyrk { LoBuf a, b; SplitK sk; };
WsSyrk ws_syrk(Carve& c, int n, int m, int r0, int r1, bool two, bool full = false) {
  WsSyrk w;
  w.a = take_lo(c, r1, m);
  if (two) w.b = take_lo(c, r1, m);
  w.sk = take_splitk(c, {shape(r1, r1, m, two ? 2 : 1, full ? 0u : (uint32_t)EPI_TRI, r0 / 128, (r1 + 127) / 128)});
  return w;
}

pb_status check_ws(const Carve& need, void* ws, size_t ws_bytes) {
  if (need.off == 0) return PB_OK;
  if (ws == nullptr) return fail(PB_ERR_WORKSPACE, "workspace is NULL (%zu bytes needed)", need.off);
  if (reinterpret_cast<uintptr_t>(ws) % 256 != 0) return fail(PB_ERR_WORKSPACE, "workspace not 256-byte aligned");
  if (ws_bytes < need.off) return fail(PB_ERR_WORKSPACE, "workspace %zu bytes < %zu needed", ws_bytes, need.off);
  return PB_OK;
}

pb_status cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) return fail(PB_ERR_CUDA, "%s: %s", what, cudaGetErrorString(e));
  return PB_OK;
}

#define PB_TRY(expr)                       \
  do {                                     \
    pb_status _st = (expr);                \
    if (_st != PB_OK) return _st;          \
  } while (0)
#define PB_CUDA(expr) PB_TRY(cuda_check((expr), #expr))

inline cudaStream_t S(pb_stream s) { return reinterpret_cast<cudaStream_t>(s); }

// Side stream (per thread and device) for the memory-bound splits of operands that
// the NEXT GEMM of a chain needs: they run concurrently with the current,
// tensor-bound GEMM (a split CTA fits beside a GEMM CTA: 40 + 168 registers per
// thread, 16.6 + 193 KB smem). fork/join are events, so graph capture follows.
// PB_SIDE_SPLITS=0 keeps everything on the caller's stream.
struct Side {
  cudaStream_t s = nullptr;
  cudaEvent_t fork = nullptr, join = nullptr;
};
Side* side_stream() {
  static const bool off = getenv("PB_SIDE_SPLITS") && atoi(getenv("PB_SIDE_SPLITS")) == 0;
  if (off) return nullptr;
  thread_local std::map<int, Side> sides;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return nullptr;
  Side& x = sides[dev];
  if (!x.s) {
    if (cudaStreamCreateWithFlags(&x.s, cudaStreamNonBlocking) != cudaSuccess ||
        cudaEventCreateWithFlags(&x.fork, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&x.join, cudaEventDisableTiming) != cudaSuccess) {
      cudaGetLastError();
      x = Side();
      return nullptr;
    }
  }
  return &x;
}

// Below this many multiply-adds pb_gemm runs the single-launch SIMT kernel.
constexpr long long SMALL_GEMM_MACS = 1ll << 21;

// core sequences (validated arguments) ---------------------------------------
pb_status run_gemm(int ni, int nj, int nk, float alpha, float beta, float* C, const float* A, const float* B,
                   const WsGemm& w, cudaStream_t s, int* L) {
  // raw-hi split: A and B are the hi operands as stored (B MN-major, no transpose): lo only
  PB_CUDA(launch_split_lo(A, ni, nk, nk, w.a.lo, w.a.ld, s));
  PB_CUDA(launch_split_lo(B, nk, nj, nj, w.b.lo, nj, s));
  *L += 2;
  GemmDesc d;
  d.M = ni; d.N = nj; d.K = nk;
  d.a[0] = w.a.op_raw(A); d.b[0] = w.b.op_raw(B);
  d.flags = EPI_OUT | (beta != 0.f ? EPI_CIN : 0u);
  d.alpha = alpha; d.beta = beta;
  d.cin = C; d.ldc = nj; d.out = C; d.ldo = nj;
  w.sk.attach(d);
  PB_CUDA(launch_umma_gemm(d, s, L));
  return PB_OK;
}

}  // namespace

extern "C" {

const char* pb_status_str(pb_status s) {
  switch (s) {
    case PB_OK: return "PB_OK";
    case PB_ERR_INVALID_ARG: return "PB_ERR_INVALID_ARG";
    case PB_ERR_UNSUPPORTED: return "PB_ERR_UNSUPPORTED";
    case PB_ERR_ALIAS: return "PB_ERR_ALIAS";
    case PB_ERR_WORKSPACE: return "PB_ERR_WORKSPACE";
    case PB_ERR_CUDA: return "PB_ERR_CUDA";
    case PB_ERR_NCCL: return "PB_ERR_NCCL";
  }
  return "PB_ERR_UNKNOWN";
}

const char* pb_last_error(void) { return g_err.c_str(); }
const char* pb_version(void) { return "pb 0.1 sm_100a (3xTF32 tcgen05 + HBM-streaming matvec)"; }
int pb_last_launch_count(void) { return g_launches; }

pb_status pb_workspace_size(const char* kernel, const long long* d, int nd, size_t* bytes) {
  if (!kernel || !bytes || (nd > 0 && !d)) return fail(PB_ERR_INVALID_ARG, "NULL argument");
  const size_t kl = strlen(kernel);
  if (kl > 5 && strcmp(kernel + kl - 5, "_dist") == 0) return dist_workspace_size(kernel, d, nd, bytes);
  for (int i = 0; i < nd; ++i)
    if (d[i] <= 0 && !(strstr(kernel, "_rows") && i == 2 && d[i] == 0))
      return fail(PB_ERR_INVALID_ARG, "dimension %d is %lld", i, d[i]);
  Carve c(nullptr, 0);
  std::string k(kernel);
  auto need = [&](int n) { return nd == n; };
  if (k == "gemm" && need(3)) ws_gemm(c, d[0], d[1], d[2]);
  else if (k == "2mm" && need(4)) ws_2mm(c, d[0], d[1], d[2], d[3]);
  else if (k == "3mm" && need(5)) ws_3mm(c, d[0], d[1], d[2], d[3], d[4]);
  else if (k == "syrk" && need(2)) ws_syrk(c, d[0], d[1], 0, d[0], false);
  else if (k == "syr2k" && need(2)) ws_syrk(c, d[0], d[1], 0, d[0], true);
  else if (k == "syrk_full" && need(2)) ws_syrk(c, d[0], d[1], 0, d[0], false, true);
  else if (k == "syr2k_full" && need(2)) ws_syrk(c, d[0], d[1], 0, d[0], true, true);
  else if ((k == "covariance" || k == "correlation") && need(2)) ws_stat(c, d[0], d[1]);
  else if (k == "atax" && need(2)) c.take<char>(atax_ws_bytes(d[0], d[1]));
  else if (k == "bicg" && need(2)) c.take<char>(mvmt_ws_bytes(d[1], d[0]));
  else if (k == "mvt" && need(1)) c.take<char>(mvmt_ws_bytes(d[0], d[0]));
  else if (k == "gesummv" && need(1)) c.take<char>(gesummv_ws_bytes(d[0], d[0]));
  else if (k == "gesummv_rows" && need(2)) c.take<char>(gesummv_ws_bytes(d[0], d[1]));
  else if (k == "syrk_rows" && need(4)) ws_syrk(c, d[0], d[1], d[2], d[3], false);
  else if (k == "syr2k_rows" && need(4)) ws_syrk(c, d[0], d[1], d[2], d[3], true);
  else if (k == "matvec_partial" && need(2)) c.take<char>(mvmt_ws_bytes(d[0], d[1]));
  else if (k == "gemm_variant" && need(3)) ws_gemm(c, d[0], d[1], d[2]);
  else if (k == "conv2d" && need(2)) (void)0;
  else if (k == "conv3d" && need(3)) (void)0;
  else if (k == "fdtd_2d" && need(2)) c.take<char>(fdtd_ws_bytes(d[0], d[1]));
  else if (k == "gramschmidt" && need(2)) c.take<char>(gramschmidt_ws_bytes(d[0], d[1]));
  else if ((k == "covariance_rows" || k == "correlation_rows") && need(4)) ws_stat_rows(c, d[0], d[1], d[2], d[3]);
  else return fail(PB_ERR_INVALID_ARG, "unknown kernel '%s' or wrong number of dims (%d)", kernel, nd);
  *bytes = align_up(c.off, 256);
  return PB_OK;
}

pb_status pb_gemm(int ni, int nj, int nk, float alpha, float beta, float* C, const float* A, const float* B,
                  void* ws, size_t ws_bytes, pb_stream s) {
  Check ck;
  ck.dims({ni, nj, nk});
  ck.cols4(nj, "C/B"); ck.cols4(nk, "A");
  ck.arr(C, ni, nj, true, "C"); ck.arr(A, ni, nk, false, "A"); ck.arr(B, nk, nj, false, "B");
  PB_TRY(ck.finish());
  Carve need(nullptr, 0);
  ws_gemm(need, ni, nj, nk);
  PB_TRY(check_ws(need, ws, ws_bytes));
  if ((long long)ni * nj * nk <= SMALL_GEMM_MACS) {
    // Launch-latency regime (e.g. the N = 128 config: 2 M multiply-adds): one launch
    // of the whole-K-strip SIMT kernel (loop internalization + register accumulation,
    // exact fp32) beats split + tensor-core GEMM (3 launches). DESIGN.md §8.
    PB_CUDA(launch_gemm_small(ni, nj, nk, alpha, beta, C, A, B, S(s)));
    g_launches = 1;
    return PB_OK;
  }
  Carve c(ws, ws_bytes);
  WsGemm w = ws_gemm(c, ni, nj, nk);
  int L = 0;
  PB_TRY(run_gemm(ni, nj, nk, alpha, beta, C, A, B, w, S(s), &L));
  g_launches = L;
  return PB_OK;
}

pb_status pb_2mm(int ni, int nj, int nk, int nl, float alpha, float beta, float* tmp, const float* A,
                 const float* B, const float* C, float* D, void* ws, size_t ws_bytes, pb_stream s) {
  Check ck;
  ck.dims({ni, nj, nk, nl});
  ck.cols4(nk, "A"); ck.cols4(nj, "B/tmp"); ck.cols4(nl, "C/D");
  ck.arr(tmp, ni, nj, true, "tmp", false);
  ck.arr(A, ni, nk, false, "A"); ck.arr(B, nk, nj, false, "B"); ck.arr(C, nj, nl, false, "C");
  ck.arr(D, ni, nl, true, "D");
  PB_TRY(ck.finish());
  Carve need(nullptr, 0);
  ws_2mm(need, ni, nj, nk, nl);
  PB_TRY(check_ws(need, ws, ws_bytes));
  Carve c(ws, ws_bytes);
  Ws2mm w = ws_2mm(c, ni, nj, nk, nl);
  cudaStream_t st = S(s);
  int L = 0;
  float* tmp_eff = tmp ? tmp : w.tmp_out;  // GEMM 2's hi operand
  GemmDesc g1;  // tmp = alpha * A * B  (epilogue also emits lo of tmp: GEMM 2's A operand is (tmp, lo))
  g1.M = ni; g1.N = nj; g1.K = nk;
  g1.a[0] = w.a.op_raw(A); g1.b[0] = w.b.op_raw(B);
  g1.flags = EPI_OUT | EPI_SPLIT_LO;
  g1.alpha = alpha;
  g1.out = tmp_eff; g1.ldo = nj;
  g1.split_lo = w.tmp.lo; g1.ld_split = w.tmp.ld;
  w.sk.attach(g1);
  GemmDesc g2;  // D = tmp * C + beta * D
  g2.M = ni; g2.N = nl; g2.K = nj;
  g2.a[0] = w.tmp.op_raw(tmp_eff); g2.b[0] = w.c.op_raw(C);
  g2.flags = EPI_OUT | (beta != 0.f ? EPI_CIN : 0u);
  g2.alpha = 1.f; g2.beta = beta;
  g2.cin = D; g2.ldc = nl; g2.out = D; g2.ldo = nl;
  w.sk.attach(g2);
  {
    // NEXT-4 chain fusion (opt-in PB_CHAIN=1): both GEMMs in one persistent
    // launch; GEMM 2's tiles of row panel i start as soon as GEMM 1 has published tmp's row
    // panel i; C's lo split (GEMM 2's B operand) is done inside the launch.
    GemmDesc gs[2] = {g1, g2};
    w.sk2.attach(gs[1]);
    if (umma_chain_ok(gs, 2)) {
      ChainLink lk[2];
      lk[1].waitA = 0;
      lk[1].npre = 1;
      ChainLink::Pre& pc = lk[1].pre[0];
      pc.X = C; pc.rows = nj; pc.cols = nl; pc.ldx = nl;
      pc.lo = w.c.lo; pc.ldo = nl; pc.lo_only = true;
      PB_CUDA(launch_split_lo(A, ni, nk, nk, w.a.lo, w.a.ld, st));
      PB_CUDA(launch_split_lo(B, nk, nj, nj, w.b.lo, nj, st));
      L += 2;
      PB_CUDA(launch_umma_chain(gs, lk, 2, w.chain.cnt, w.chain.cnt_bytes, st, &L));
      g_launches = L;
      return PB_OK;
    }
  }
  Side* sd = side_stream();
  // raw-hi splits (lo only; B and C MN-major as stored, no transposes)
  PB_CUDA(launch_split_lo(A, ni, nk, nk, w.a.lo, w.a.ld, st));
  PB_CUDA(launch_split_lo(B, nk, nj, nj, w.b.lo, nj, st));
  if (sd) {  // C's lo (GEMM 2's B operand) starts with GEMM 1 and runs beside it
    PB_CUDA(cudaEventRecord(sd->fork, st));
    PB_CUDA(cudaStreamWaitEvent(sd->s, sd->fork, 0));
    PB_CUDA(launch_split_lo(C, nj, nl, nl, w.c.lo, nl, sd->s));
    PB_CUDA(cudaEventRecord(sd->join, sd->s));
  } else {
    PB_CUDA(launch_split_lo(C, nj, nl, nl, w.c.lo, nl, st));
  }
  L += 3;
  PB_CUDA(launch_umma_gemm(g1, st, &L));
  if (sd) PB_CUDA(cudaStreamWaitEvent(st, sd->join, 0));
  PB_CUDA(launch_umma_gemm(g2, st, &L));
  g_launches = L;
  return PB_OK;
}

pb_status pb_3mm(int ni, int nj, int nk, int nl, int nm, float* E, const float* A, const float* B, float* F,
                 const float* C, const float* D, float* G, void* ws, size_t ws_bytes, pb_stream s) {
  Check ck;
  ck.dims({ni, nj, nk, nl, nm});
  ck.cols4(nk, "A"); ck.cols4(nj, "B/E"); ck.cols4(nm, "C"); ck.cols4(nl, "D/F/G");
  ck.arr(E, ni, nj, true, "E"); ck.arr(A, ni, nk, false, "A"); ck.arr(B, nk, nj, false, "B");
  ck.arr(F, nj, nl, true, "F"); ck.arr(C, nj, nm, false, "C"); ck.arr(D, nm, nl, false, "D");
  ck.arr(G, ni, nl, true, "G");
  PB_TRY(ck.finish());
  Carve need(nullptr, 0);
  ws_3mm(need, ni, nj, nk, nl, nm);
  PB_TRY(check_ws(need, ws, ws_bytes));
  Carve c(ws, ws_bytes);
  Ws3mm w = ws_3mm(c, ni, nj, nk, nl, nm);
  cudaStream_t st = S(s);
  int L = 0;
  GemmDesc gf;  // F = C * D; epilogue also emits lo of F (G's B operand is (F, lo), MN-major)
  gf.M = nj; gf.N = nl; gf.K = nm;
  gf.a[0] = w.c.op_raw(C); gf.b[0] = w.d.op_raw(D);
  gf.flags = EPI_OUT | EPI_SPLIT_LO;
  gf.out = F; gf.ldo = nl;
  gf.split_lo = w.f.lo; gf.ld_split = nl;
  w.sk.attach(gf);
  GemmDesc ge;  // E = A * B; epilogue also emits lo of E (G's A operand is (E, lo))
  ge.M = ni; ge.N = nj; ge.K = nk;
  ge.a[0] = w.a.op_raw(A); ge.b[0] = w.b.op_raw(B);
  ge.flags = EPI_OUT | EPI_SPLIT_LO;
  ge.out = E; ge.ldo = nj;
  ge.split_lo = w.e.lo; ge.ld_split = w.e.ld;
  w.sk.attach(ge);
  GemmDesc gg;  // G = E * F
  gg.M = ni; gg.N = nl; gg.K = nj;
  gg.a[0] = w.e.op_raw(E); gg.b[0] = w.f.op_raw(F);
  gg.flags = EPI_OUT;
  gg.out = G; gg.ldo = nl;
  w.sk.attach(gg);
  {
    // NEXT-4 chain fusion (opt-in PB_CHAIN=1): F, E and G in one persistent
    // launch. E's operand splits (lo of A and B) are done inside the launch; G's tile (i, j)
    // starts once E's row panel i and F's column panel j are published.
    GemmDesc gs[3] = {gf, ge, gg};
    w.sk2.attach(gs[1]);
    w.sk3.attach(gs[2]);
    if (umma_chain_ok(gs, 3)) {
      ChainLink lk[3];
      lk[2].waitA = 1;
      lk[2].waitB = 0;
      lk[1].npre = 2;
      ChainLink::Pre& pa = lk[1].pre[0];
      pa.X = A; pa.rows = ni; pa.cols = nk; pa.ldx = nk;
      pa.lo = w.a.lo; pa.ldo = w.a.ld; pa.lo_only = true;
      ChainLink::Pre& pbt = lk[1].pre[1];
      pbt.X = B; pbt.rows = nk; pbt.cols = nj; pbt.ldx = nj;
      pbt.lo = w.b.lo; pbt.ldo = nj; pbt.lo_only = true;
      PB_CUDA(launch_split_lo(C, nj, nm, nm, w.c.lo, w.c.ld, st));
      PB_CUDA(launch_split_lo(D, nm, nl, nl, w.d.lo, nl, st));
      L += 2;
      PB_CUDA(launch_umma_chain(gs, lk, 3, w.chain.cnt, w.chain.cnt_bytes, st, &L));
      g_launches = L;
      return PB_OK;
    }
  }
  Side* sd = side_stream();
  cudaStream_t sab = st;
  PB_CUDA(launch_split_lo(C, nj, nm, nm, w.c.lo, w.c.ld, st));
  PB_CUDA(launch_split_lo(D, nm, nl, nl, w.d.lo, nl, st));
  if (sd) {  // E's operands (lo of A, B) are split beside GEMM F (fork: F's operands are ready)
    PB_CUDA(cudaEventRecord(sd->fork, st));
    PB_CUDA(cudaStreamWaitEvent(sd->s, sd->fork, 0));
    sab = sd->s;
  }
  PB_CUDA(launch_split_lo(A, ni, nk, nk, w.a.lo, w.a.ld, sab));
  PB_CUDA(launch_split_lo(B, nk, nj, nj, w.b.lo, nj, sab));
  if (sd) PB_CUDA(cudaEventRecord(sd->join, sd->s));
  L += 4;
  PB_CUDA(launch_umma_gemm(gf, st, &L));
  if (sd) PB_CUDA(cudaStreamWaitEvent(st, sd->join, 0));
  PB_CUDA(launch_umma_gemm(ge, st, &L));
  PB_CUDA(launch_umma_gemm(gg, st, &L));
  g_launches = L;
  return PB_OK;
}

// full == true: the SYCL-Bench / PolyBench-GPU form:
// every C[i][j] is updated, not only j <= i (the product is symmetric, C need not be).
static pb_status syrk_core(int n, int m, int r0, int r1, float alpha, float beta, float* C_blk, const float* A,
                           const float* B, void* ws, size_t ws_bytes, pb_stream s, bool full = false) {
  Check ck;
  ck.dims({n, m});
  if (ck.st == PB_OK && (r0 < 0 || r1 > n || r0 >= r1 || r0 % 128 != 0))
    ck.st = fail(PB_ERR_INVALID_ARG, "row range [%d,%d) invalid (r0 multiple of 128, r1 <= n)", r0, r1);
  ck.cols4(m, "A/B"); ck.cols4(n, "C");
  ck.arr(C_blk, r1 - r0, n, true, "C"); ck.arr(A, r1, m, false, "A");
  if (B) ck.arr(B, r1, m, false, "B");
  PB_TRY(ck.finish());
  Carve need(nullptr, 0);
  ws_syrk(need, n, m, r0, r1, B != nullptr, full);
  PB_TRY(check_ws(need, ws, ws_bytes));
  Carve c(ws, ws_bytes);
  WsSyrk w = ws_syrk(c, n, m, r0, r1, B != nullptr, full);
  cudaStream_t st = S(s);
  int L = 0;
  // raw-hi split (A and B are the hi operands, rows K-major as they are): lo only
  PB_CUDA(launch_split_lo(A, r1, m, m, w.a.lo, w.a.ld, st));
  ++L;
  if (B) { PB_CUDA(launch_split_lo(B, r1, m, m, w.b.lo, w.b.ld, st)); ++L; }
  const SplitOperand oa = w.a.op_raw(A), ob = B ? w.b.op_raw(B) : SplitOperand{};
  GemmDesc d;
  d.M = r1; d.N = r1; d.K = m;
  if (B) {  // C[i][j] += A[j].B[i] + B[j].A[i]: pair 0 = (B rows i, A rows j), pair 1 = (A rows i, B rows j)
    d.npairs = 2;
    d.a[0] = ob; d.b[0] = oa;
    d.a[1] = oa; d.b[1] = ob;
  } else {
    d.a[0] = oa; d.b[0] = oa;
  }
  d.flags = (full ? 0u : (uint32_t)EPI_TRI) | EPI_OUT | (beta != 0.f ? EPI_CIN : 0u);
  d.alpha = alpha; d.beta = beta;
  d.cin = C_blk; d.ldc = n; d.out = C_blk; d.ldo = n; d.out_row0 = r0;
  d.tm0 = r0 / 128; d.tm1 = (r1 + 127) / 128;
  w.sk.attach(d);
  PB_CUDA(launch_umma_gemm(d, st, &L));
  g_launches = L;
  return PB_OK;
}

pb_status pb_syrk(int n, int m, float alpha, float beta, float* C, const float* A, void* ws, size_t ws_bytes,
                  pb_stream s) {
  return syrk_core(n, m, 0, n, alpha, beta, C, A, nullptr, ws, ws_bytes, s);
}
pb_status pb_syr2k(int n, int m, float alpha, float beta, float* C, const float* A, const float* B, void* ws,
                   size_t ws_bytes, pb_stream s) {
  if (!B) return fail(PB_ERR_INVALID_ARG, "B is NULL");
  return syrk_core(n, m, 0, n, alpha, beta, C, A, B, ws, ws_bytes, s);
}
pb_status pb_syrk_full(int n, int m, float alpha, float beta, float* C, const float* A, void* ws, size_t ws_bytes,
                       pb_stream s) {
  return syrk_core(n, m, 0, n, alpha, beta, C, A, nullptr, ws, ws_bytes, s, true);
}
pb_status pb_syr2k_full(int n, int m, float alpha, float beta, float* C, const float* A, const float* B, void* ws,
                        size_t ws_bytes, pb_stream s) {
  if (!B) return fail(PB_ERR_INVALID_ARG, "B is NULL");
  return syrk_core(n, m, 0, n, alpha, beta, C, A, B, ws, ws_bytes, s, true);
}
pb_status pb_syrk_rows(int n, int m, int r0, int r1, float alpha, float beta, float* C_blk, const float* A, void* ws,
                       size_t ws_bytes, pb_stream s) {
  return syrk_core(n, m, r0, r1, alpha, beta, C_blk, A, nullptr, ws, ws_bytes, s);
}
pb_status pb_syr2k_rows(int n, int m, int r0, int r1, float alpha, float beta, float* C_blk, const float* A,
                        const float* B, void* ws, size_t ws_bytes, pb_stream s) {
  if (!B) return fail(PB_ERR_INVALID_ARG, "B is NULL");
  return syrk_core(n, m, r0, r1, alpha, beta, C_blk, A, B, ws, ws_bytes, s);
}

static pb_status stat_core(bool corr, int m, int n, float float_n, float eps, const float* data, float* out,
                           float* mean, float* stddev, void* ws, size_t ws_bytes, pb_stream s) {
  Check ck;
  ck.dims({m, n});
  if (ck.st == PB_OK && !corr && n < 2) ck.st = fail(PB_ERR_INVALID_ARG, "covariance needs n >= 2");
  if (ck.st == PB_OK && !(float_n > 0.f) ) ck.st = fail(PB_ERR_INVALID_ARG, "float_n must be > 0");
  if (ck.st == PB_OK && !corr && float_n == 1.0f) ck.st = fail(PB_ERR_INVALID_ARG, "float_n - 1 == 0");
  ck.cols4(m, "data/out");
  ck.arr(data, n, m, false, "data");
  ck.arr(out, m, m, true, corr ? "corr" : "cov");
  ck.arr(mean, 1, m, true, "mean", false);
  if (corr) ck.arr(stddev, 1, m, true, "stddev", false);
  PB_TRY(ck.finish());
  Carve need(nullptr, 0);
  ws_stat(need, m, n);
  PB_TRY(check_ws(need, ws, ws_bytes));
  Carve c(ws, ws_bytes);
  WsStat w = ws_stat(c, m, n);
  cudaStream_t st = S(s);
  int L = 0;
  const bool banded = banded_stats(n);
  // PB_TIMELINE (tuning only, eager calls): entry/exit of prep, Gram and combine
  static const bool tl_env = getenv("PB_TIMELINE") != nullptr;
  cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
  if (tl_env) cudaStreamIsCapturing(st, &cap);
  const bool tl = tl_env && cap == cudaStreamCaptureStatusNone;
  if (tl) {
    cudaStreamSynchronize(st);
    timeline_stats(true, nullptr);
    timeline_umma(true, nullptr);
  }
  if (banded && gram_fused_ok(m, n) && !tl) {
    // one launch: band statistics + centred split + Gram + split-K exchange + epilogue
    char* wb = static_cast<char*>(ws) + align_up(0, 256);
    PB_CUDA(launch_gram_fused(corr, m, n, (double)float_n, (double)eps, data, out, mean, corr ? stddev : nullptr, wb,
                              st, &L));
    g_launches = L;
    return PB_OK;
  }
  GramStats gs;
  if (banded) {  // one pass: band-centred split + per-band column statistics
    PB_CUDA(launch_band_prep(data, n, m, corr, w.xt.hi, w.xt.lo, w.xt.ld, w.band_mean, corr ? w.band_m2 : nullptr, st));
    gs.band_mean = w.band_mean;
    gs.band_m2 = corr ? w.band_m2 : nullptr;
    gs.nbands = band_count(n);
    gs.n = n;
    gs.float_n = (double)float_n;
    gs.eps = (double)eps;
    gs.mean_out = mean;
    gs.sd_out = corr ? stddev : nullptr;
  } else {  // exact mean first, then centre (and normalise) into the split operand
    PB_CUDA(launch_stats_split(data, n, m, (double)float_n, (double)eps, corr, w.xt.hi, w.xt.lo, w.xt.ld, mean,
                               corr ? stddev : nullptr, st));
  }
  ++L;
  GemmDesc d;  // Gram core: out[i][j] = alpha * sum_k Xt[i][k] Xt[j][k], lower tiles + mirror
  d.M = m; d.N = m; d.K = n;
  d.a[0] = w.xt.op(); d.b[0] = w.xt.op();
  d.flags = EPI_TRI | EPI_MIRROR | EPI_OUT | (corr ? EPI_DIAG_ONE : 0u) | (banded ? EPI_PARTIAL : 0u);
  d.alpha = (corr && !banded) ? 1.0f : (float)(1.0 / ((double)float_n - 1.0));
  d.out = out; d.ldo = m;
  w.sk.attach(d);
  UmmaPlan pl = umma_plan(d);
  if (!banded && pl.ksplit > 1 && w.sk.part) {  // split-K: partials + combine kernel
    d.flags |= EPI_PARTIAL;
    pl = umma_plan(d);
  }
  PB_CUDA(launch_umma_gemm(d, st, &L));
  if (d.flags & EPI_PARTIAL) PB_CUDA(launch_gram_combine(d, pl, corr, gs, st, &L));
  g_launches = L;
  if (tl) {
    cudaStreamSynchronize(st);
    unsigned long long a[2] = {0, 0}, b[4] = {0, 0, 0, 0};
    timeline_stats(false, a);
    timeline_umma(false, b);
    const double t0 = (double)a[0];
    auto us = [&](unsigned long long v) { return v == ~0ull || v == 0 ? -1.0 : ((double)v - t0) / 1e3; };
    fprintf(stderr, "[pb timeline] prep %.1f-%.1f | gram %.1f-%.1f | combine %.1f-%.1f us\n", us(a[0]), us(a[1]),
            us(b[0]), us(b[1]), us(b[2]), us(b[3]));
  }
  return PB_OK;
}

static pb_status stat_rows_core(bool corr, int m, int n, float float_n, float eps, int r0, int r1, const float* data,
                                float* out_blk, float* mean, float* stddev, void* ws, size_t ws_bytes, pb_stream s) {
  Check ck;
  ck.dims({m, n});
  if (ck.st == PB_OK && (r0 < 0 || r1 > m || r0 >= r1 || r0 % 128 != 0))
    ck.st = fail(PB_ERR_INVALID_ARG, "row range [%d,%d) invalid (r0 multiple of 128, r1 <= m)", r0, r1);
  if (ck.st == PB_OK && !corr && n < 2) ck.st = fail(PB_ERR_INVALID_ARG, "covariance needs n >= 2");
  if (ck.st == PB_OK && !(float_n > 0.f)) ck.st = fail(PB_ERR_INVALID_ARG, "float_n must be > 0");
  if (ck.st == PB_OK && !corr && float_n == 1.0f) ck.st = fail(PB_ERR_INVALID_ARG, "float_n - 1 == 0");
  ck.cols4(m, "data/out");
  ck.arr(data, n, m, false, "data");
  ck.arr(out_blk, r1 - r0, m, true, corr ? "corr" : "cov");
  ck.arr(mean, 1, m, true, "mean", false);
  if (corr) ck.arr(stddev, 1, m, true, "stddev", false);
  PB_TRY(ck.finish());
  Carve need(nullptr, 0);
  ws_stat_rows(need, m, n, r0, r1);
  PB_TRY(check_ws(need, ws, ws_bytes));
  Carve c(ws, ws_bytes);
  WsStatRows w = ws_stat_rows(c, m, n, r0, r1);
  cudaStream_t st = S(s);
  int L = 0;
  PB_CUDA(launch_stats_split(data, n, m, (double)float_n, (double)eps, corr, w.xt.hi, w.xt.lo, w.xt.ld, mean,
                             corr ? stddev : nullptr, st));
  ++L;
  GemmDesc d;  // rows [r0, r1) of X^T X over every column (both triangles: no mirror across ranks)
  d.M = r1; d.N = m; d.K = n;
  d.a[0] = w.xt.op(); d.b[0] = w.xt.op();
  d.flags = EPI_OUT | (corr ? EPI_DIAG_ONE : 0u);
  d.alpha = corr ? 1.0f : (float)(1.0 / ((double)float_n - 1.0));
  d.out = out_blk; d.ldo = m; d.out_row0 = r0;
  d.tm0 = r0 / 128; d.tm1 = (r1 + 127) / 128;
  w.sk.attach(d);
  PB_CUDA(launch_umma_gemm(d, st, &L));
  g_launches = L;
  return PB_OK;
}

pb_status pb_covariance_rows(int m, int n, float float_n, int r0, int r1, const float* data, float* cov_blk,
                             float* mean, void* ws, size_t ws_bytes, pb_stream s) {
  return stat_rows_core(false, m, n, float_n, 0.f, r0, r1, data, cov_blk, mean, nullptr, ws, ws_bytes, s);
}

pb_status pb_correlation_rows(int m, int n, float float_n, float eps, int r0, int r1, const float* data,
                              float* corr_blk, float* mean, float* stddev, void* ws, size_t ws_bytes, pb_stream s) {
  return stat_rows_core(true, m, n, float_n, eps, r0, r1, data, corr_blk, mean, stddev, ws, ws_bytes, s);
}

pb_status pb_covariance(int m, int n, float float_n, const float* data, float* cov, float* mean, void* ws,
                        size_t ws_bytes, pb_stream s) {
  return stat_core(false, m, n, float_n, 0.f, data, cov, mean, nullptr, ws, ws_bytes, s);
}
pb_status pb_correlation(int m, int n, float float_n, float eps, const float* data, float* corr, float* mean,
                         float* stddev, void* ws, size_t ws_bytes, pb_stream s) {
  return stat_core(true, m, n, float_n, eps, data, corr, mean, stddev, ws, ws_bytes, s);
}

pb_status pb_atax(int m, int n, const float* A, const float* x, float* y, float* tmp, void* ws, size_t ws_bytes,
                  pb_stream s) {
  Check ck;
  ck.dims({m, n});
  ck.cols4(n, "A");
  ck.arr(A, m, n, false, "A"); ck.arr(x, 1, n, false, "x"); ck.arr(y, 1, n, true, "y");
  ck.arr(tmp, 1, m, true, "tmp", false);
  PB_TRY(ck.finish());
  Carve need(nullptr, 0);
  need.take<char>(atax_ws_bytes(m, n));
  PB_TRY(check_ws(need, ws, ws_bytes));
  int L = 0;
  PB_CUDA(launch_atax(A, x, m, n, y, tmp, ws, S(s), &L));
  g_launches = L;
  return PB_OK;
}

pb_status pb_bicg(int m, int n, const float* A, float* s_out, float* q, const float* p, const float* r, void* ws,
                  size_t ws_bytes, pb_stream s) {
  Check ck;
  ck.dims({m, n});
  ck.cols4(m, "A");
  ck.arr(A, n, m, false, "A"); ck.arr(s_out, 1, m, true, "s"); ck.arr(q, 1, n, true, "q");
  ck.arr(p, 1, m, false, "p"); ck.arr(r, 1, n, false, "r");
  PB_TRY(ck.finish());
  Carve need(nullptr, 0);
  need.take<char>(mvmt_ws_bytes(n, m));
  PB_TRY(check_ws(need, ws, ws_bytes));
  int L = 0;
  PB_CUDA(launch_mvmt(A, n, m, p, r, nullptr, q, nullptr, s_out, ws, S(s), &L));
  g_launches = L;
  return PB_OK;
}

pb_status pb_mvt(int n, float* x1, float* x2, const float* y_1, const float* y_2, const float* A, void* ws,
                 size_t ws_bytes, pb_stream s) {
  Check ck;
  ck.dims({n});
  ck.cols4(n, "A");
  ck.arr(x1, 1, n, true, "x1"); ck.arr(x2, 1, n, true, "x2");
  ck.arr(y_1, 1, n, false, "y_1"); ck.arr(y_2, 1, n, false, "y_2"); ck.arr(A, n, n, false, "A");
  PB_TRY(ck.finish());
  Carve need(nullptr, 0);
  need.take<char>(mvmt_ws_bytes(n, n));
  PB_TRY(check_ws(need, ws, ws_bytes));
  int L = 0;
  PB_CUDA(launch_mvmt(A, n, n, y_1, y_2, x1, x1, x2, x2, ws, S(s), &L));
  g_launches = L;
  return PB_OK;
}

pb_status pb_gesummv_rows(int rows, int n, float alpha, float beta, const float* A, const float* B, float* tmp,
                          const float* x, float* y, void* ws, size_t ws_bytes, pb_stream s) {
  Check ck;
  ck.dims({rows, n});
  ck.cols4(n, "A/B");
  ck.arr(A, rows, n, false, "A"); ck.arr(B, rows, n, false, "B"); ck.arr(tmp, 1, rows, true, "tmp", false);
  ck.arr(x, 1, n, false, "x"); ck.arr(y, 1, rows, true, "y");
  PB_TRY(ck.finish());
  Carve need(nullptr, 0);
  need.take<char>(gesummv_ws_bytes(rows, n));
  PB_TRY(check_ws(need, ws, ws_bytes));
  int L = 0;
  PB_CUDA(launch_gesummv(A, B, x, rows, n, alpha, beta, y, tmp, ws, S(s), &L));
  g_launches = L;
  return PB_OK;
}

pb_status pb_gesummv(int n, float alpha, float beta, const float* A, const float* B, float* tmp, const float* x,
                     float* y, void* ws, size_t ws_bytes, pb_stream s) {
  return pb_gesummv_rows(n, n, alpha, beta, A, B, tmp, x, y, ws, ws_bytes, s);
}

pb_status pb_matvec_partial(int rows, int cols, const float* A_blk, const float* v, const float* base_row,
                            float* rowdot, const float* w, const float* base_col, float* colpart, void* ws,
                            size_t ws_bytes, pb_stream s) {
  Check ck;
  ck.dims({rows, cols});
  ck.cols4(cols, "A_blk");
  if (ck.st == PB_OK && !v && !w) ck.st = fail(PB_ERR_INVALID_ARG, "neither v nor w given");
  if (ck.st == PB_OK && ((v == nullptr) != (rowdot == nullptr) || (w == nullptr) != (colpart == nullptr)))
    ck.st = fail(PB_ERR_INVALID_ARG, "v/rowdot and w/colpart must be given together");
  ck.arr(A_blk, rows, cols, false, "A_blk");
  ck.arr(v, 1, cols, false, "v", false);
  ck.arr(w, 1, rows, false, "w", false);
  if (rowdot != base_row) ck.arr(base_row, 1, rows, false, "base_row", false);
  if (colpart != base_col) ck.arr(base_col, 1, cols, false, "base_col", false);
  ck.arr(rowdot, 1, rows, true, "rowdot", false);
  ck.arr(colpart, 1, cols, true, "colpart", false);
  PB_TRY(ck.finish());
  Carve need(nullptr, 0);
  need.take<char>(mvmt_ws_bytes(rows, cols));
  PB_TRY(check_ws(need, ws, ws_bytes));
  int L = 0;
  PB_CUDA(launch_mvmt(A_blk, rows, cols, v, w, base_row, rowdot, base_col, colpart, ws, S(s), &L));
  g_launches = L;
  return PB_OK;
}

pb_status pb_row_partition(int rows, int nranks, int rank, int triangular, int align, int* begin, int* end) {
  if (rows <= 0 || nranks <= 0 || rank < 0 || rank >= nranks || align <= 0 || !begin || !end ||
      triangular < 0 || triangular > 2)
    return fail(PB_ERR_INVALID_ARG, "bad partition arguments");
  if (triangular == 2) {
    // syrk/syr2k cost balance: rank g's cost = lower-triangle area of its rows
    // (r1^2 - r0^2)/2 + RHO * r1, the second term being the split of A[0:r1] (and
    // B) it needs. Measured on B200: 60.6 ps per triangle element (K = 8192) and
    // 16.2 ns per split row -> RHO = 267 (both scale with K: independent of m); with the
    // lo-only split (~10 ns per row) the per-rank proxy (scripts/rank_shapes.py --only-syrk,
    // PB_RHO sweep 120 / 165 / 210 / 267) is best at RHO = 210: G = 4 syrk 591 vs 660 us,
    // G = 8 equal (424 us).
    // Equal cost C per rank: r1 = sqrt(r0^2 + 2 (C - RHO r1)) solved by bisection on C.
    static const double rho_env = getenv("PB_RHO") ? atof(getenv("PB_RHO")) : 0.0;  // tuning only
    const double RHO = rho_env > 0.0 ? rho_env : 210.0, n = rows;
    auto last_bound = [&](double C, std::vector<double>* b) {
      double r0 = 0.0;
      if (b) b->assign(1, 0.0);
      for (int g = 0; g < nranks; ++g) {
        // (r1^2 - r0^2)/2 + RHO r1 = C  ->  r1 = -RHO + sqrt(RHO^2 + r0^2 + 2C)
        const double r1 = -RHO + std::sqrt(RHO * RHO + r0 * r0 + 2.0 * C);
        r0 = r1;
        if (b) b->push_back(r1);
      }
      return r0;
    };
    double lo = 0.0, hi = n * n / 2.0 + RHO * n;
    for (int it = 0; it < 100; ++it) {
      const double mid = 0.5 * (lo + hi);
      (last_bound(mid, nullptr) < n ? lo : hi) = mid;
    }
    std::vector<double> b;
    last_bound(hi, &b);
    // snap to multiples of align left to right: floor or ceil, whichever puts this
    // rank's cost closer to the balanced target (same choice on every rank)
    std::vector<long long> s(nranks + 1, 0);
    s[nranks] = rows;
    for (int g = 1; g < nranks; ++g) {
      const long long f = (long long)std::floor(b[g] / align) * align, c = f + align;
      auto dev = [&](long long e) {
        const double r0 = (double)s[g - 1], r1 = (double)e;
        return std::fabs((r1 * r1 - r0 * r0) / 2.0 + RHO * r1 - hi);
      };
      long long pick = dev(f) <= dev(c) ? f : c;
      s[g] = std::min<long long>(std::max<long long>(pick, s[g - 1]), rows);
    }
    *begin = (int)s[rank];
    *end = (int)std::max(s[rank], s[rank + 1]);
    return PB_OK;
  }
  auto bound = [&](int g) -> int {
    if (g <= 0) return 0;
    if (g >= nranks) return rows;
    double f = triangular ? std::sqrt((double)g / nranks) : (double)g / nranks;
    long long b = llround(f * rows / align) * (long long)align;
    if (b < 0) b = 0;
    if (b > rows) b = rows;
    return (int)b;
  };
  int b0 = bound(rank), b1 = bound(rank + 1);  // bound() is monotone in g
  *begin = b0;
  *end = std::max(b0, b1);
  return PB_OK;
}

pb_status pb_gemm_variant(int variant, int ni, int nj, int nk, float alpha, float beta, float* C, const float* A,
                          const float* B, void* ws, size_t ws_bytes, pb_stream s) {
  if (variant == 3) return pb_gemm(ni, nj, nk, alpha, beta, C, A, B, ws, ws_bytes, s);
  if (variant < 0 || variant > 3) return fail(PB_ERR_INVALID_ARG, "variant %d", variant);
  Check ck;
  ck.dims({ni, nj, nk});
  ck.cols4(nj, "C/B"); ck.cols4(nk, "A");
  ck.arr(C, ni, nj, true, "C"); ck.arr(A, ni, nk, false, "A"); ck.arr(B, nk, nj, false, "B");
  PB_TRY(ck.finish());
  cudaStream_t st = S(s);
  if (variant == 0) PB_CUDA(launch_gemm_listing8(ni, nj, nk, alpha, beta, C, A, B, st));
  if (variant == 1) PB_CUDA(launch_gemm_listing9(ni, nj, nk, alpha, beta, C, A, B, st));
  if (variant == 2) PB_CUDA(launch_gemm_listing9_reg(ni, nj, nk, alpha, beta, C, A, B, st));
  g_launches = 1;
  return PB_OK;
}

// ---- SYCL-Bench stencils (§VIII; readings R19-R21) -------------
pb_status pb_conv2d(int ni, int nj, const float* w, const float* A, float* B, pb_stream s) {
  Check ck;
  ck.dims({ni, nj});
  ck.cols4(nj, "A/B");
  if (ck.st == PB_OK && w == nullptr) ck.st = fail(PB_ERR_INVALID_ARG, "w is NULL");
  ck.arr(A, ni, nj, false, "A"); ck.arr(B, ni, nj, true, "B");
  PB_TRY(ck.finish());
  int L = 0;
  PB_CUDA(launch_conv2d(A, B, ni, nj, w, S(s), &L));
  g_launches = L;
  return PB_OK;
}

pb_status pb_conv2d_variant(int variant, int ni, int nj, const float* w, const float* A, float* B, pb_stream s) {
  if (variant == 1) return pb_conv2d(ni, nj, w, A, B, s);
  if (variant != 0) return fail(PB_ERR_INVALID_ARG, "variant %d (0 = naive, 1 = production)", variant);
  Check ck;
  ck.dims({ni, nj});
  ck.cols4(nj, "A/B");
  if (ck.st == PB_OK && w == nullptr) ck.st = fail(PB_ERR_INVALID_ARG, "w is NULL");
  ck.arr(A, ni, nj, false, "A"); ck.arr(B, ni, nj, true, "B");
  PB_TRY(ck.finish());
  int L = 0;
  PB_CUDA(launch_conv_naive(false, A, B, ni, nj, 1, w, S(s), &L));
  g_launches = L;
  return PB_OK;
}

pb_status pb_conv3d_variant(int variant, int ni, int nj, int nk, const float* w, const float* A, float* B,
                            pb_stream s) {
  if (variant == 1) return pb_conv3d(ni, nj, nk, w, A, B, s);
  if (variant != 0) return fail(PB_ERR_INVALID_ARG, "variant %d (0 = naive, 1 = production)", variant);
  Check ck;
  ck.dims({ni, nj, nk});
  ck.cols4(nk, "A/B");
  if (ck.st == PB_OK && w == nullptr) ck.st = fail(PB_ERR_INVALID_ARG, "w is NULL");
  ck.arr(A, (long long)ni * nj, nk, false, "A"); ck.arr(B, (long long)ni * nj, nk, true, "B");
  PB_TRY(ck.finish());
  int L = 0;
  PB_CUDA(launch_conv_naive(true, A, B, ni, nj, nk, w, S(s), &L));
  g_launches = L;
  return PB_OK;
}

pb_status pb_conv3d(int ni, int nj, int nk, const float* w, const float* A, float* B, pb_stream s) {
  Check ck;
  ck.dims({ni, nj, nk});
  ck.cols4(nk, "A/B");
  if (ck.st == PB_OK && (long long)ni * nj > (1ll << 31)) ck.st = fail(PB_ERR_INVALID_ARG, "ni*nj too large");
  if (ck.st == PB_OK && w == nullptr) ck.st = fail(PB_ERR_INVALID_ARG, "w is NULL");
  ck.arr(A, (long long)ni * nj, nk, false, "A"); ck.arr(B, (long long)ni * nj, nk, true, "B");
  PB_TRY(ck.finish());
  int L = 0;
  PB_CUDA(launch_conv3d(A, B, ni, nj, nk, w, S(s), &L));
  g_launches = L;
  return PB_OK;
}

pb_status pb_fdtd_2d(int tmax, int nx, int ny, float* ex, float* ey, float* hz, const float* fict, void* ws,
                     size_t ws_bytes, pb_stream s) {
  Check ck;
  if (tmax < 0) ck.st = fail(PB_ERR_INVALID_ARG, "tmax %d < 0", tmax);
  ck.dims({nx, ny});
  ck.cols4(ny, "ex/ey/hz");
  ck.arr(ex, nx, ny, true, "ex"); ck.arr(ey, nx, ny, true, "ey"); ck.arr(hz, nx, ny, true, "hz");
  ck.arr(fict, 1, tmax > 0 ? tmax : 1, false, "fict", tmax > 0);
  PB_TRY(ck.finish());
  Carve need(nullptr, 0);
  need.take<char>(fdtd_ws_bytes(nx, ny));
  PB_TRY(check_ws(need, ws, ws_bytes));
  int L = 0;
  PB_CUDA(launch_fdtd2d(tmax, nx, ny, ex, ey, hz, fict, ws, S(s), &L));
  g_launches = L;
  return PB_OK;
}

// ---- gramschmidt (reading R22) ---------------------------
pb_status pb_gramschmidt_variant(int variant, int m, int n, float* A, float* R, float* Q, void* ws, size_t ws_bytes,
                                 pb_stream s) {
  if (variant == 1) return pb_gramschmidt(m, n, A, R, Q, ws, ws_bytes, s);
  if (variant != 0) return fail(PB_ERR_INVALID_ARG, "variant %d (0 = naive, 1 = production)", variant);
  Check ck;
  ck.dims({m, n});
  ck.arr(A, m, n, true, "A"); ck.arr(R, n, n, true, "R"); ck.arr(Q, m, n, true, "Q");
  PB_TRY(ck.finish());
  Carve need(nullptr, 0);
  need.take<char>(gramschmidt_ws_bytes(m, n));
  PB_TRY(check_ws(need, ws, ws_bytes));
  int L = 0;
  PB_CUDA(launch_gramschmidt_naive(m, n, A, R, Q, ws, S(s), &L));
  g_launches = L;
  return PB_OK;
}

pb_status pb_gramschmidt(int m, int n, float* A, float* R, float* Q, void* ws, size_t ws_bytes, pb_stream s) {
  Check ck;
  ck.dims({m, n});
  ck.arr(A, m, n, true, "A"); ck.arr(R, n, n, true, "R"); ck.arr(Q, m, n, true, "Q");
  PB_TRY(ck.finish());
  Carve need(nullptr, 0);
  need.take<char>(gramschmidt_ws_bytes(m, n));
  PB_TRY(check_ws(need, ws, ws_bytes));
  int L = 0;
  PB_CUDA(launch_gramschmidt(m, n, A, R, Q, ws, S(s), &L));
  g_launches = L;
  return PB_OK;
}

}  // extern "C"
