// pb_internal.h — host-side interfaces between the C ABI (pb_api.cu) and the
// kernel translation units. Not installed; not part of the ABI.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <stddef.h>
#include <stdint.h>

#include <atomic>

namespace pb {

// ---- 3xTF32 tcgen05 GEMM (k_umma.cu) ---------------------------------------
// One K-major split operand: hi/lo arrays of `rows` x `K` (row pitch ld floats).
struct SplitOperand {
  const float* hi = nullptr;
  const float* lo = nullptr;
  int rows = 0;
  int K = 0;
  int ld = 0;
  // mn = true (B operands only): hi / lo are stored K x rows row-major (pitch ld), i.e.
  // MN-major (B[k][n] as the caller has it: no transpose); tiles go MN-major to the MMA.
  bool mn = false;
};

enum : uint32_t {
  EPI_TRI = 1u << 0,       // only tiles/elements with j <= i (lower triangle)
  EPI_MIRROR = 1u << 1,    // also write out[j][i] (symmetric output)
  EPI_DIAG_ONE = 1u << 2,  // out[i][i] = 1
  EPI_CIN = 1u << 3,       // v += beta * Cin[i][j]
  EPI_OUT = 1u << 4,       // write fp32 out[i][j]
  EPI_SPLIT = 1u << 5,     // write hi/lo split of v at [i][j] (next GEMM's K-major A operand)
  EPI_SPLIT_T = 1u << 6,   // write hi/lo split of v at [j][i] (next GEMM's K-major B operand)
  EPI_PARTIAL = 1u << 7,   // every tile only writes (per-split) partials; launch_gram_combine finishes
  EPI_SPLIT_LO = 1u << 8,  // write lo_of_raw(v) at [i][j] (split_lo): the next GEMM's operand is (out, lo)
};

struct GemmDesc {
  int M = 0, N = 0, K = 0;  // output rows (operand-a rows), cols (operand-b rows), contraction
  int npairs = 1;           // 1, or 2 for syr2k (acc = a0*b0^T + a1*b1^T)
  SplitOperand a[2], b[2];
  uint32_t flags = EPI_OUT;
  float alpha = 1.f, beta = 0.f;
  const float* cin = nullptr;
  int ldc = 0;
  float* out = nullptr;
  int ldo = 0;
  int out_row0 = 0;  // out/cin row index = i - out_row0
  float* split_hi = nullptr;
  float* split_lo = nullptr;
  int ld_split = 0;
  int tm0 = 0, tm1 = -1;  // tile-row range in 128-row units (default all)
  float* part = nullptr;       // split-K partials (umma_plan(d).part_bytes)
  unsigned* counters = nullptr;  // split-K counters (umma_plan(d).counter_bytes)
  size_t part_cap = 0, counter_cap = 0;  // bytes reserved at part / counters (checked at launch)
};

struct UmmaPlan {
  int cfg = 1;     // 1: 1-CTA 128x128, 2: 2-CTA 256x128, 3: 2-CTA 256x256
  int ksplit = 1;  // split-K factor of the split tiles
  long long tiles = 0;
  long long split_tiles = 0;  // tiles [0, split_tiles) are split ksplit ways
  size_t part_bytes = 0, counter_bytes = 0;
  int streamk = 0;  // 1: stream-K (every CTA group an equal share of all (tile, k-block) iterations)
  int maxseg = 1;   // stream-K: most groups sharing one tile (partial slots per tile)
};
UmmaPlan umma_plan(const GemmDesc& d);
// NEXT-4 chain fusion: phases 0..nphase-1 in ONE persistent launch (2-CTA 256x256 tiles).
// Phase q waits for the row panels of phase links[q].waitA (its A operand = that phase's
// split output, EPI_SPLIT) and/or the column panels of phase links[q].waitB (its B operand
// = that phase's transposed split output, EPI_SPLIT_T). Every phase needs its own split-K
// area (part / counters). cnt: readiness counters, umma_chain_cnt_bytes. Returns
// cudaErrorNotSupported when the shapes do not fit one launch (callers launch separately).
struct ChainLink {
  int waitA = -1;
  int waitB = -1;
  // operand splits of this phase done inside the launch (by all CTAs' epilogue warps before
  // their first epilogue): X (rows x cols, pitch ldx) -> hi/lo (transpose: of X^T), pitch ldo
  struct Pre {
    const float* X = nullptr;
    int rows = 0, cols = 0, ldx = 0;
    float* hi = nullptr;
    float* lo = nullptr;
    int ldo = 0;
    bool transpose = false;
    bool lo_only = false;  // raw-hi split: write only lo (same layout as X; hi unused)
  } pre[2];
  int npre = 0;
};
bool umma_chain_ok(const GemmDesc* d, int nphase);
size_t umma_chain_cnt_bytes(const GemmDesc* d, int nphase);
cudaError_t launch_umma_chain(const GemmDesc* d, const ChainLink* links, int nphase, unsigned* cnt, size_t cnt_cap,
                              cudaStream_t s, int* launches);
// host helpers of k_umma.cu (tensor maps, SM count)
bool make_map2d(CUtensorMap* m, const float* base, int inner, int rows, long long ld, int box_inner, int box_rows,
                bool swizzle128,
                CUtensorMapSwizzle sw_override = CU_TENSOR_MAP_SWIZZLE_NONE);
bool make_map(CUtensorMap* m, const float* base, int rows, int K, int ld, int box_rows);
bool make_map_mn_runs(CUtensorMap* m, const float* base, int inner, int rows, long long ld, int box_rows, int groups,
                      CUtensorMapSwizzle sw);
int num_sms();
cudaError_t launch_umma_gemm(const GemmDesc& d, cudaStream_t s, int* launches);
// Statistics the Gram combine needs (nullptr band_mean: the operand was centred exactly).
struct GramStats {
  const double* band_mean = nullptr;  // [nbands][m]
  const double* band_m2 = nullptr;    // [nbands][m] (correlation)
  int nbands = 0, n = 0;
  double float_n = 0.0, eps = 0.0;
  float* mean_out = nullptr;
  float* sd_out = nullptr;
};

// Gram finish for EPI_PARTIAL launches (plan pl): out[i][j] = alpha * sum_s partial_s for
// j <= i, mirrored to out[j][i]; diag_one -> out[i][i] = 1.
cudaError_t launch_gram_combine(const GemmDesc& d, const UmmaPlan& pl, bool diag_one, const GramStats& st,
                                cudaStream_t s, int* launches);

// Fused covariance / correlation (k_gram.cu): prep + Gram + split-K exchange + epilogue
// in one launch for n <= 2048, m <= 2048 (every unit co-resident).
bool gram_fused_ok(int m, int n);
size_t gram_fused_ws_bytes(int m, int n);
cudaError_t launch_gram_fused(bool corr, int m, int n, double float_n, double eps, const float* data, float* out,
                              float* mean, float* sd, void* ws, cudaStream_t s, int* launches);

// Observation-split covariance / correlation steps (k_covdist.cu, driven by pb_dist.cu).
// launch_obs_sums: out[0..m) = fp64 column sums of X (nl x m), out[m..2m) = sums of squares.
cudaError_t launch_obs_sums(const float* X, int nl, int m, double* out, cudaStream_t s);
// sums: nranks x [2][m] (rank order) -> mean / sd (optional outputs) and the centred (and for
// correlation normalised) transpose Yt (m x ldy, zero for k >= nl).
cudaError_t launch_obs_center_t(bool corr, const float* X, int nl, int m, const double* sums, int nranks, int n,
                                double float_n, double eps, float* Yt, int ldy, float* mean, float* sd, cudaStream_t s);
// in place on an output row band (rows [r0, r0 + rows)): cov *= alpha; corr: diagonal := 1.
cudaError_t launch_obs_finish(bool corr, float* out, int rows, int m, int r0, float alpha, cudaStream_t s);

// ---- split / prep (k_split.cu) ----------------------------------------------
// hi/lo split of a rows x cols matrix; same layout (ldo = ld of output).
// done != nullptr: each CTA adds 1 to *done when its part is stored (release); *ctas += grid size.
cudaError_t launch_split(const float* X, int rows, int cols, int ldx, float* hi, float* lo, int ldo,
                         cudaStream_t s, unsigned* done = nullptr, unsigned* ctas = nullptr);
// raw-hi split: only lo of X (rows x cols, same layout, pitch ldo); X itself is the hi operand.
cudaError_t launch_split_lo(const float* X, int rows, int cols, int ldx, float* lo, int ldo, cudaStream_t s);
// hi/lo split of the transpose: out (cols x rows), out pitch ldo (>= rows).
// If mean != nullptr: value = (x - mean[col]) * inv[col] computed in double first
// (inv == nullptr means 1).
cudaError_t launch_split_T(const float* X, int rows, int cols, int ldx, float* hiT, float* loT, int ldo,
                           const double* mean, const double* inv, cudaStream_t s, unsigned* done = nullptr,
                           unsigned* ctas = nullptr);


// ---- column statistics (k_stats.cu) -----------------------------------------
// Fused covariance/correlation prep: column mean (+ stddev, eps rule) and the
// centred (normalised) data written transposed as a hi/lo split (m x ldo).
cudaError_t launch_stats_split(const float* data, int n, int m, double float_n, double eps, bool corr, float* hiT,
                               float* loT, int ldo, float* mean_out, float* sd_out, cudaStream_t s);

// Banded single-pass prep (n <= 8 * 256): band-centred split + per-band column
// means (and M2 for correlation), fp64 [band_count(n)][m].
int band_count(int n);
cudaError_t launch_band_prep(const float* data, int n, int m, bool corr, float* hiT, float* loT, int ldo,
                             double* band_mean, double* band_m2, cudaStream_t s);
// ---- matrix-vector family (k_matvec.cu) -------------------------------------
// y[i] = alpha * A_i.x + beta * B_i.x (B may be null -> beta ignored); tmp[i] = A_i.x (optional).
cudaError_t launch_rowdot(const float* A, const float* B, const float* x, int rows, int cols, float alpha,
                          float beta, float* y, float* tmp, cudaStream_t s);
// Fused single pass over A (rows x cols):
//   rowpart[ct][i] = sum_{j in col tile ct} A[i][j]*v[j]        (if v)
//   colpart[rt][j] = sum_{i in row tile rt} A[i][j]*w[i]        (if w)
// then out_row[i] = base_row[i] + sum_ct rowpart, out_col[j] = base_col[j] + sum_rt colpart.
size_t mvmt_ws_bytes(int rows, int cols);
// gesummv: y = alpha*A x + beta*B x (tmp = A x, optional), A and B streamed once in
// 512 x 256 tiles (per-tile row partials in ws, then a fixed-order reduce).
size_t gesummv_ws_bytes(int rows, int cols);
cudaError_t launch_gesummv(const float* A, const float* B, const float* x, int rows, int cols, float alpha, float beta,
                           float* y, float* tmp, void* ws, cudaStream_t s, int* launches);
cudaError_t launch_mvmt(const float* A, int rows, int cols, const float* v, const float* w,
                        const float* base_row, float* out_row, const float* base_col, float* out_col,
                        void* ws, cudaStream_t s, int* launches);

// atax: single pass (2-CTA cluster, row halves staged by 1-D bulk copies, DSMEM
// partial-dot exchange) when 16384 <= n <= 32768 and A >= 96 MB (larger than L2),
// else two passes (the second from L2). ws: atax_ws_bytes(m, n).
size_t atax_ws_bytes(int m, int n);
cudaError_t launch_atax(const float* A, const float* x, int m, int n, float* y, float* tmp, void* ws,
                        cudaStream_t s, int* launches);

// ---- stencils (k_stencil.cu): SYCL-Bench 2D/3D convolution, FDTD-2D -------
// w9 / w27 are host arrays (copied into the kernel parameters).
cudaError_t launch_conv2d(const float* A, float* B, int ni, int nj, const float* w9, cudaStream_t s, int* launches);
cudaError_t launch_conv3d(const float* A, float* B, int ni, int nj, int nk, const float* w27, cudaStream_t s,
                          int* launches);
// ablation: one thread per output point, every tap a global load (SYCL-Bench shape)
cudaError_t launch_conv_naive(bool three_d, const float* A, float* B, int ni, int nj, int nk, const float* w,
                              cudaStream_t s, int* launches);
size_t fdtd_ws_bytes(int nx, int ny);
cudaError_t launch_fdtd2d(int tmax, int nx, int ny, float* ex, float* ey, float* hz, const float* fict, void* ws,
                          cudaStream_t s, int* launches);

// ---- gramschmidt (k_gramschmidt.cu): persistent modified Gram-Schmidt, fp64 state
size_t gramschmidt_ws_bytes(int m, int n);
cudaError_t launch_gramschmidt(int m, int n, float* A, float* R, float* Q, void* ws, cudaStream_t s, int* launches);
// ablation: PolyBench-GPU shape (3 launches per column; fp64 working arrays)
cudaError_t launch_gramschmidt_naive(int m, int n, float* A, float* R, float* Q, void* ws, cudaStream_t s,
                                     int* launches);

// ---- peer-memory collectives (k_peer.cu; host side in pb_dist.cu) ------------
constexpr int PEER_MAXR = 8;            // ranks per peer group
constexpr size_t PEER_HDR = 4096;       // header bytes before the data region
// Device-side view of a peer group (pointers valid in this process).
struct PeerView {
  float* data[PEER_MAXR];                // data region of rank g
  unsigned long long* flags[PEER_MAXR];  // flags array of rank g (indexed by source rank)
  unsigned long long* acks[PEER_MAXR];   // acks array of rank g (indexed by consumer rank)
  unsigned long long* flags_mine;        // == flags[rank]
  unsigned long long* acks_mine;         // == acks[rank]
  unsigned* counter;                     // this rank's grid counters [push, consume]
  unsigned* status;                      // != 0: a bounded wait timed out
  unsigned long long* epoch;             // collectives completed (this rank's header)
  int nranks = 0, rank = 0;
};
struct PeerPush {  // for every destination g: count floats from src[g] to data[g] + dst_off[g]
  const float* src[PEER_MAXR];
  long long dst_off[PEER_MAXR];
  long long count[PEER_MAXR];
};
struct PeerConsume {  // reduce: out[i] = sum_g data_mine[g * slot + i]; else out[i] = data_mine[i]
  float* out;
  long long count, slot;
  int reduce;
};
cudaError_t launch_peer_push(const PeerView& v, const PeerPush& p, cudaStream_t s);
cudaError_t launch_peer_consume(const PeerView& v, const PeerConsume& c, cudaStream_t s);

// ---- SIMT ablation kernels (k_simt.cu): PAPER.md Listing 8 / Listing 9 -------
cudaError_t launch_gemm_listing8(int ni, int nj, int nk, float alpha, float beta, float* C, const float* A,
                                 const float* B, cudaStream_t s);
cudaError_t launch_gemm_listing9(int ni, int nj, int nk, float alpha, float beta, float* C, const float* A,
                                 const float* B, cudaStream_t s);
// PB_TIMELINE (tuning only): reset the per-kernel entry/exit stamps, or read them back.
void timeline_stats(bool reset, unsigned long long* out2);
void timeline_umma(bool reset, unsigned long long* out4);
cudaError_t launch_gemm_small(int ni, int nj, int nk, float alpha, float beta, float* C, const float* A,
                              const float* B, cudaStream_t s);
cudaError_t launch_gemm_listing9_reg(int ni, int nj, int nk, float alpha, float beta, float* C, const float* A,
                                     const float* B, cudaStream_t s);

// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) once per kernel and device (the
// attribute is per device; a process may drive several GPUs from several threads).
template <auto Kernel>
cudaError_t ensure_smem(size_t bytes) {
  static std::atomic<unsigned long long> done{0};
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  const unsigned long long bit = 1ull << (dev & 63);
  if (done.load(std::memory_order_acquire) & bit) return cudaSuccess;
  e = cudaFuncSetAttribute(Kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  if (e == cudaSuccess) done.fetch_or(bit, std::memory_order_release);
  return e;
}

// Launch with programmatic stream serialization (PDL): the kernel may be scheduled
// while its predecessor drains; every kernel launched this way calls pdl_wait()
// before it touches data the predecessor produced.
template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                       Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...);
}

inline int round_up(int x, int a) { return (x + a - 1) / a * a; }
inline size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

}  // namespace pb
