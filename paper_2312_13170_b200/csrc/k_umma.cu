// k_umma.cu — the 3xTF32 tcgen05 GEMM engine behind gemm / 2mm / 3mm / syrk /
// syr2k and the Gram core of covariance / correlation.
//
// Paper mapping:
//  * Loop internalization (Listing 9 at PAPER.md:404-428):
//    the per-work-item k-loop over global memory becomes a k-block loop over
//    shared-memory tiles. Here a TMA producer warp stages 128x32 fp32 tiles of
//    the hi/lo operands into a STAGES-deep smem ring; mbarriers play the role
//    of Listing 9's two group_barriers (full = "tile loaded", empty = "tile
//    consumed"), so loads of block k+1.. overlap the math on block k.
//  * Detect reduction (Listings 4-5): C[i][j] is never
//    re-read/re-written inside the k-loop; the running sum lives in a TMEM
//    accumulator (tcgen05.mma, fp32) and is written once by the epilogue.
//  * Uniformity: every barrier/mbarrier wait sits in
//    warp-uniform control flow; tails are zero-filled by TMA, not branched.
//
// Precision: x = hi + lo with hi = tf32_rna(x), lo = tf32_rna(x - hi) (split
// done by k_split.cu); acc += a_hi*b_hi + a_hi*b_lo + a_lo*b_hi (lo*lo dropped).
//
// Two variants (template CG): CG = 1, one CTA per 128x128 tile; CG = 2, an SM
// pair (2-CTA cluster, tcgen05 cta_group::2) per 256x128 tile: each CTA stages
// its 128 rows of A and HALF of B (64 rows), the leader CTA issues M=256 MMAs
// that read both CTAs' smem, and each CTA's TMEM holds its 128 output rows.
// Per-SM operand traffic drops from 64 KiB to 48 KiB per k-block.
//
// CTA layout (192 threads, 1 CTA/SM, persistent over tiles):
//   warp 0      TMA producer (one lane)
//   warp 1      TMEM allocator + MMA issuer (one lane)
//   warps 2..5  epilogue: tcgen05.ld (warp%4 selects its 32 TMEM lanes), alpha/beta,
//               masks, fp32 / split / mirrored stores
// Tiles 128 x 128 (UMMA M=128, N=128, K=8 per instruction), BK = 32 (one 128-B
// swizzle row of fp32), 3-stage ring of {A_hi, A_lo, B_hi, B_lo} = 64 KiB/stage,
// two TMEM accumulator slots (2 x {big, small} x 128 columns = all 512) that
// alternate per 512-wide K chunk; the epilogue promotes each chunk into fp32
// registers (RN) so the tensor core's truncating accumulate cannot bias long K.
#include <math.h>
#include <stdio.h>
#include <stdlib.h>

#include <algorithm>
#include <vector>

#include "pb_device.cuh"
#include "pb_internal.h"
#include "pb_umma.cuh"

namespace pb {
// ---------------------------------------------------------------- host side (also used by k_gram.cu)
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn get_encode() {
  static EncodeTiledFn fn = nullptr;
  if (!fn) {
    void* ptr = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(ptr);
  }
  return fn;
}

// 2-D fp32 tensor map: `inner` x `rows` (row pitch ld floats), box = box_inner x box_rows,
// 128-B swizzle (box_inner == 32) or none, unless `sw_override` names another mode. Out-of-bounds boxes are zero-filled on loads
// and clipped on stores.
bool make_map2d(CUtensorMap* m, const float* base, int inner, int rows, long long ld, int box_inner, int box_rows,
                bool swizzle128, CUtensorMapSwizzle sw_override) {
  EncodeTiledFn enc = get_encode();
  if (!enc) return false;
  cuuint64_t dims[2] = {(cuuint64_t)inner, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)ld * 4};
  cuuint32_t box[2] = {(cuuint32_t)box_inner, (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(base), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE,
                   sw_override != CU_TENSOR_MAP_SWIZZLE_NONE ? sw_override
                   : swizzle128                              ? CU_TENSOR_MAP_SWIZZLE_128B
                                                             : CU_TENSOR_MAP_SWIZZLE_NONE,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

// MN-major operand tiles of a row-major fp32 matrix (`inner` columns x `rows`, pitch ld
// floats) as ONE 3-D box: {32 columns, box_rows rows, groups runs of 32 columns} lands in
// smem as [group][row][32] (runs box_rows * 128 B apart). Needs inner % 32 == 0 (the run
// dimension has no per-element bound).
bool make_map_mn_runs(CUtensorMap* m, const float* base, int inner, int rows, long long ld, int box_rows, int groups,
                      CUtensorMapSwizzle sw) {
  EncodeTiledFn enc = get_encode();
  if (!enc || inner % 32) return false;
  cuuint64_t dims[3] = {32, (cuuint64_t)rows, (cuuint64_t)(inner / 32)};
  cuuint64_t strides[2] = {(cuuint64_t)ld * 4, 128};
  cuuint32_t box[3] = {32, (cuuint32_t)box_rows, (cuuint32_t)groups};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<float*>(base), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

// K-major operand (rows x K, pitch ld floats), box = 32 (K) x box_rows, 128-B swizzle.
bool make_map(CUtensorMap* m, const float* base, int rows, int K, int ld, int box_rows) {
  return make_map2d(m, base, K, rows, ld, 32, box_rows, true);
}

int num_sms() {  // per device (cached)
  static std::atomic<int> cache[64];
  int dev = 0;
  cudaGetDevice(&dev);
  int n = cache[dev & 63].load(std::memory_order_relaxed);
  if (!n) {
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
    cache[dev & 63].store(n, std::memory_order_relaxed);
  }
  return n;
}


namespace {

__device__ int g_tl_on;                  // PB_TIMELINE (tuning only)
__device__ unsigned long long g_tl[4];   // [umma entry, exit, combine entry, exit]

constexpr int BM = 128;  // rows per CTA
constexpr int BK = 32;
constexpr int GROUP_M = 8;  // tile-rows per raster group (L2 reuse); PB_GROUP_M overrides (tuning)
constexpr uint32_t TMEM_COLS = 512;
constexpr int A_TILE = BM * BK * 4;  // 16 KiB
constexpr int EPI_COLS = 128;        // accumulator columns (fp32 registers) per epilogue thread

// Tile configurations. BN = MMA N (output columns per tile). With BN = 128 each
// slot holds separate `big` (a_hi b_hi) and `small` (cross terms) accumulators;
// with BN = 256 a slot is one 256-column accumulator (TMEM is 512 columns) and
// chunks are shorter. Smem read demand per MMA flop halves from BN=128 to 256,
// which is what bounds the tf32 SS-MMA rate.
template <int CG, int BN>
struct Cfg {
  static constexpr int B_ROWS = BN / CG;                  // B rows staged by each CTA
  static constexpr int B_TILE = B_ROWS * BK * 4;
  static constexpr int STAGE_BYTES = 2 * A_TILE + 2 * B_TILE;
  static constexpr int STAGES = (196 * 1024) / STAGE_BYTES;
  static constexpr int PAIR_M = BM * CG;                  // output rows per tile
  static constexpr bool SPLIT_ACC = BN == 128;            // separate big / small accumulators
  static constexpr int SLOT_COLS = SPLIT_ACC ? 2 * BN : BN;
  static constexpr int CHUNK_KB = 16;                     // k-blocks per TMEM partial sum (512 of K)
  static constexpr int EPI_WARPS = 4 * (BN / EPI_COLS);
  static constexpr int NUM_THREADS = 64 + 32 * EPI_WARPS;
};

struct Params {
  int M, N, K, npairs, nkb;  // nkb = k-blocks per pair
  uint32_t flags;
  float alpha, beta;
  const float* cin;
  int ldc;
  float* out;
  int ldo;
  int out_row0;
  float* split_hi;
  float* split_lo;
  int ld_split;
  int tm0, tm1, tiles_n, ratio;  // ratio = tile rows / BN (CG)
  long long num_tiles;
  int ksplit;                    // K splits of each split tile (split-K)
  long long split_tiles;         // split tiles: [split_t0, split_t0 + split_tiles)
  int group_m = GROUP_M;         // tile-rows per raster group (PB_GROUP_M)
  long long split_t0 = 0;        // 0: split tiles first (their units lead); num_tiles - split_tiles: last
  float* part;                   // split-K partial tiles [unit][CG][128][BN]
  unsigned* counters;            // split-K arrival counters [tile][CG], zero before launch
  int b_mn;                      // 1: the B operand is MN-major (B[k][n] as stored), 32-column TMA runs
  int streamk;                   // 1: stream-K schedule (pair p takes iterations [p I / P, (p+1) I / P))
  long long sk_iters;            // I = num_tiles * k-blocks per tile
  int sk_pairs;                  // P = CTA groups of the grid
  int sk_maxseg;                 // partial slots per tile (max pairs sharing one tile)
  int dbg;                       // PB_UMMA_DEBUG (tuning only): 1 = skip partial exchange
  int tma_epi;                   // 1: staged TMA-store epilogue (maps 8 = out, 9 = split_lo, 10 = cin)
  unsigned long long* tstamp;    // PB_UMMA_TIMING (tuning only): [cta][unit<16][8] globaltimer stamps
};

// A launch = one GEMM (nphase 1) or a CHAIN of up to 3 dependent GEMMs in one persistent
// grid (NEXT-4 chain fusion: 2mm's tmp -> D, 3mm's F, E -> G). Units of phase q are
// [ubase[q], ubase[q+1]); every CTA walks its units in order, so it finishes its part of a
// phase before it starts the next. A phase's epilogue publishes each finished tile on a
// readiness counter (release add after its stores); a later phase's TMA producer acquires
// the counters of the operand panels it loads (A: the row panel tm of this CTA's rank;
// B: the column panel tn, i.e. the rows of the transposed operand written by EPI_SPLIT_T)
// before its first k-block. Only earlier phases are waited on and all CTAs are resident
// (persistent grid <= SMs), so the waits cannot deadlock.
struct Chain {
  int nphase;
  long long ubase[4];
  Params ph[3];
  unsigned* cnt;           // readiness counters (zeroed before the launch)
  int sig_kind[3];         // 0 none, 1: cnt[sig_off + tm * CG + rank] += 1, 2: cnt[sig_off + tn] += 1
  int sig_off[3];
  int waitA_off[3], waitA_target[3];  // A rows: cnt[off + tm * CG + rank] >= target (off < 0: none)
  int waitB_off[3], waitB_target[3];  // B rows: cnt[off + tn] >= target
  // operand splits of a later phase done INSIDE the launch by the epilogue warps of every CTA
  // (idle during the first tile's mainloop), published on cnt[pre_off] (one add per CTA)
  struct Pre {
    const float* X;
    int rows, cols, ldx;
    float* hi;
    float* lo;
    int ldo;
    int transpose;  // 0: hi/lo of X (same layout); 1: hi/lo of X^T (cols x rows); 2: lo only (raw-hi)
  } pre[2];
  int npre, pre_phase, pre_off;
};
constexpr int PRE_STAGE = 32 * 32 * 4;  // per epilogue warp: a 32 x 32 transpose block (swizzled)
__device__ __forceinline__ int phase_of(const Chain& ch, long long u) {
  int q = 0;
  while (q + 1 < ch.nphase && u >= ch.ubase[q + 1]) ++q;
  return q;
}
__device__ __forceinline__ void wait_count(const unsigned* c, unsigned target) {
  unsigned v;
  for (;;) {
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(c) : "memory");
    if (v >= target) break;
    __nanosleep(64);
  }
}

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#define TSTAMP(unit_local, ev)                                                                         \
  do {                                                                                                 \
    if (p.tstamp && (unit_local) < 16)                                                                 \
      p.tstamp[((unsigned long long)blockIdx.x * 16 + (unit_local)) * 8 + (ev)] = gtimer();            \
  } while (0)

struct __align__(8) Ctl {
  uint64_t full[8];
  uint64_t empty[8];
  uint64_t tfull[2];
  uint64_t tempty[2];
  uint32_t tmem_base;
  uint32_t last_flag;
  uint32_t pre_warps_done;  // chain: epilogue warps that finished their share of the in-launch splits
  uint64_t cbar[16];        // TMA-store epilogue: per epilogue warp, its two C-box buffers
};

// number of column tiles in tile-row tm (lower triangle: tiles touching j <= i)
__device__ __forceinline__ int row_tiles(const Params& p, int tm) {
  if (!(p.flags & EPI_TRI)) return p.tiles_n;
  return min(p.ratio * (tm + 1), p.tiles_n);
}

// Tile t of the persistent schedule -> (tm, tn). Raster: groups of GROUP_M
// tile-rows; inside a group tn is the outer index so CTAs running together
// share B panels (and the group's A panels) in L2. In the lower-triangle mode
// column tn holds the rows tm >= tn / ratio of the group.
__device__ void tile_coords(const Params& p, long long t, int& tm, int& tn) {
  int g0 = p.tm0;
  for (;;) {
    const int g1 = min(g0 + (p.group_m > 0 ? p.group_m : GROUP_M), p.tm1);
    long long cnt = 0;
    for (int r = g0; r < g1; ++r) cnt += row_tiles(p, r);
    if (t < cnt || g1 >= p.tm1) {
      for (int c = 0;; ++c) {
        const int first = (p.flags & EPI_TRI) ? max(g0, c / p.ratio) : g0;
        const int rows = g1 - first;
        if (t < rows) {
          tn = c;
          tm = first + (int)t;
          return;
        }
        t -= rows;
      }
    }
    t -= cnt;
    g0 = g1;
  }
}

__device__ __forceinline__ void store4(float* p, float a, float b, float c, float d) {
  *reinterpret_cast<float4*>(p) = make_float4(a, b, c, d);
}

// Work unit u -> (tile, split, k-block range). Default (split_t0 = W = num_tiles -
// split_tiles): units [0, W) are the whole tiles in raster order, then the K-splits of
// the last split_tiles tiles (split-major). Every pair then runs whole tiles in lockstep
// waves — the tiles of one wave stream the same A / B panel k-blocks at nearly the same
// time, so L2 serves the re-reads (syr2k 8192: 8.3 GB of DRAM reads per launch instead of
// 15.7 GB with split units first, whose 1/S-long units shift the waves against each other;
// DESIGN.md §8) — and the split units fill the last partial wave. split_t0 = 0
// (PB_SPLIT_FIRST=1, and every EPI_PARTIAL plan) puts the split units first instead.
struct Unit {
  long long t;
  int ks, kbA, kbB;
  bool split;
  int nseg;        // units (K segments) that share tile t
  long long slot;  // this unit's partial slot
};
__device__ __forceinline__ Unit unit_of(const Params& p, long long u, int nkb_total) {
  Unit r;
  const long long rs = p.split_tiles * p.ksplit;
  const long long whole = p.num_tiles - p.split_tiles;
  const long long v = p.split_t0 == 0 ? u : u - whole;  // index among the split units (if >= 0)
  if (v >= 0 && v < rs) {
    r.t = p.split_t0 + v % p.split_tiles;
    r.ks = (int)(v / p.split_tiles);
    r.split = true;
    r.slot = v;
  } else {
    r.t = p.split_t0 == 0 ? p.split_tiles + (u - rs) : u;
    r.ks = 0;
    r.split = false;
    r.slot = u;
  }
  const int S = r.split ? p.ksplit : 1;
  r.kbA = (int)((long long)nkb_total * r.ks / S);
  r.kbB = (int)((long long)nkb_total * (r.ks + 1) / S);
  r.nseg = S;
  return r;
}
// partial slot of segment k2 of (split) tile t
__device__ __forceinline__ long long slot_of(const Params& p, long long t, int k2) {
  return p.streamk ? t * p.sk_maxseg + k2 : k2 * p.split_tiles + (t - p.split_t0);
}

// The units one CTA group works through, in order: round robin over [0, units) (every
// launch; the phases of a chain one after the other), or, in stream-K mode (one GEMM),
// the K segments covering this group's share of the flattened (tile, k-block) space:
// group g takes iterations [g I / P, (g+1) I / P); tile t is shared by the groups
// pair_of(t nkb) .. pair_of((t+1) nkb - 1), pair_of(i) = ((i + 1) P - 1) / I.
struct UnitIter {
  long long u, step, end;  // round robin
  long long it, itend;     // stream-K
  long long g;
  bool sk;
};
__device__ __forceinline__ UnitIter iter_init(const Chain& ch, long long g, long long step) {
  UnitIter r;
  const Params& p = ch.ph[0];
  r.sk = ch.nphase == 1 && p.streamk;
  r.g = g;
  r.u = g; r.step = step; r.end = ch.ubase[ch.nphase];
  r.it = g * p.sk_iters / p.sk_pairs;
  r.itend = (g + 1) * p.sk_iters / p.sk_pairs;
  return r;
}
__device__ __forceinline__ bool iter_next(const Chain& ch, UnitIter& r, int& ph, long long& ul, Unit& un) {
  if (r.sk) {
    if (r.it >= r.itend) return false;
    const Params& p = ch.ph[0];
    const long long nkb = (long long)p.nkb * p.npairs, I = p.sk_iters, P = p.sk_pairs;
    const long long t = r.it / nkb;
    const int kbA = (int)(r.it - t * nkb);
    const int kbB = (int)min(nkb, (long long)kbA + (r.itend - r.it));
    const long long lo = ((t * nkb + 1) * P - 1) / I, hi = (((t + 1) * nkb) * P - 1) / I;
    un.t = t; un.kbA = kbA; un.kbB = kbB;
    un.nseg = (int)(hi - lo + 1);
    un.ks = (int)(r.g - lo);
    un.split = un.nseg > 1;
    un.slot = t * p.sk_maxseg + un.ks;
    ph = 0;
    ul = un.slot;
    r.it += kbB - kbA;
    return true;
  }
  if (r.u >= r.end) return false;
  ph = phase_of(ch, r.u);
  const Params& p = ch.ph[ph];
  ul = r.u - ch.ubase[ph];
  un = unit_of(p, ul, p.nkb * p.npairs);
  r.u += r.step;
  return true;
}

// CHAIN = false: one GEMM (the chain machinery compiles away, keeping the epilogue's
// register budget); CHAIN = true: the phases of a Chain in one launch.
template <int CG, int BN, bool CHAIN>
__global__ void __launch_bounds__(Cfg<CG, BN>::NUM_THREADS, 1)
    umma3x_kernel(const __grid_constant__ CUtensorMap a0h, const __grid_constant__ CUtensorMap a0l,
                  const __grid_constant__ CUtensorMap b0h, const __grid_constant__ CUtensorMap b0l,
                  const __grid_constant__ CUtensorMap a1h, const __grid_constant__ CUtensorMap a1l,
                  const __grid_constant__ CUtensorMap b1h, const __grid_constant__ CUtensorMap b1l,
                  const __grid_constant__ CUtensorMap a2h, const __grid_constant__ CUtensorMap a2l,
                  const __grid_constant__ CUtensorMap b2h, const __grid_constant__ CUtensorMap b2l,
                  const __grid_constant__ Chain ch) {
  using C = Cfg<CG, BN>;
  constexpr int STAGES = C::STAGES, STAGE_BYTES = C::STAGE_BYTES, B_TILE = C::B_TILE;
  constexpr int CHUNK_KB = C::CHUNK_KB;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  Ctl* ctl = reinterpret_cast<Ctl*>(smem + STAGES * STAGE_BYTES);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const uint32_t rank = CG == 2 ? cluster_rank() : 0u;
  const bool leader = rank == 0;
  const long long tile0 = blockIdx.x / CG, tile_step = gridDim.x / CG;

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&ctl->full[s], 1);
      mbar_init(&ctl->empty[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&ctl->tfull[s], 1);
      mbar_init(&ctl->tempty[s], C::EPI_WARPS * CG);  // one arrive per epilogue warp of every CTA
    }
    ctl->pre_warps_done = 0;
    for (int w = 0; w < 2 * C::EPI_WARPS; ++w) mbar_init(&ctl->cbar[w], 1);
    fence_mbar_init();
  }
  if (warp == 0 && lane == 0) {
    tma_prefetch(&a0h); tma_prefetch(&a0l); tma_prefetch(&b0h); tma_prefetch(&b0l);
    if (ch.ph[0].npairs > 1 || ch.nphase > 1) {
      tma_prefetch(&a1h); tma_prefetch(&a1l); tma_prefetch(&b1h); tma_prefetch(&b1l);
    }
    if (ch.nphase > 2 || (!CHAIN && ch.ph[0].tma_epi)) {
      tma_prefetch(&a2h); tma_prefetch(&a2l); tma_prefetch(&b2h); tma_prefetch(&b2l);
    }
  }
  if (warp == 1) tmem_alloc_cg<CG>(&ctl->tmem_base, TMEM_COLS);
  tc_fence_before();
  if constexpr (CG == 2) cluster_sync_all(); else __syncthreads();
  tc_fence_after();
  pdl_trigger();  // dependents may start their setup once every CTA here runs
  pdl_wait();  // the setup above overlapped the producer kernel's tail (PDL)
  const int tl = g_tl_on;
  tl_enter(tl, g_tl, 0);
  const uint32_t tmem_base = ctl->tmem_base;
  const long long num_units = ch.ubase[ch.nphase];
  // operand maps: phase q (chain) or pair q (syr2k) uses maps 4q .. 4q + 3
  auto map_of = [&](int q, int which) -> const CUtensorMap* {
    switch (q * 4 + which) {
      case 0: return &a0h; case 1: return &a0l; case 2: return &b0h; case 3: return &b0l;
      case 4: return &a1h; case 5: return &a1l; case 6: return &b1h; case 7: return &b1l;
      case 8: return &a2h; case 9: return &a2l; case 10: return &b2h; default: return &b2l;
    }
  };

  if (warp == 0) {
    // ===================== TMA producer (every CTA loads its own A rows and B half)
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      UnitIter ui = iter_init(ch, tile0, tile_step);
      int ph;
      long long uph;
      Unit un;
      while (iter_next(ch, ui, ph, uph, un)) {
        const Params& p = ch.ph[ph];
        int tm, tn;
        tile_coords(p, un.t, tm, tn);
        const int arow = tm * C::PAIR_M + (int)rank * BM;
        const int brow = tn * BN + (int)rank * C::B_ROWS;
        if (CHAIN && (ch.waitA_off[ph] >= 0 || ch.waitB_off[ph] >= 0 || (ch.npre && ph == ch.pre_phase))) {  // chain
          if (ch.npre && ph == ch.pre_phase) wait_count(ch.cnt + ch.pre_off, gridDim.x);
          if (ch.waitA_off[ph] >= 0) wait_count(ch.cnt + ch.waitA_off[ph] + tm * CG + rank, ch.waitA_target[ph]);
          if (ch.waitB_off[ph] >= 0) wait_count(ch.cnt + ch.waitB_off[ph] + tn, ch.waitB_target[ph]);
          asm volatile("fence.proxy.async.global;" ::: "memory");  // generic-proxy stores -> TMA reads
        }
        for (int kb = un.kbA; kb < un.kbB; ++kb) {
          mbar_wait(&ctl->empty[stage], phase ^ 1);
          uint8_t* st = smem + stage * STAGE_BYTES;
          const int pair = kb >= p.nkb;
          const int k = (kb - pair * p.nkb) * BK;
          const int mq = ch.nphase > 1 ? ph : pair;
          if (leader) mbar_arrive_expect_tx(&ctl->full[stage], CG * STAGE_BYTES);
          tma_load_cg<CG>(map_of(mq, 0), &ctl->full[stage], st, k, arow);
          tma_load_cg<CG>(map_of(mq, 1), &ctl->full[stage], st + A_TILE, k, arow);
          if (p.b_mn) {  // B[k][n]: [32-column run][32 k rows][32] boxes, 128B_BASE32B layout
#pragma unroll
            for (int q = 0; q < C::B_ROWS / 32; ++q) {
              tma_load_cg<CG>(map_of(mq, 2), &ctl->full[stage], st + 2 * A_TILE + q * 4096, brow + 32 * q, k);
              tma_load_cg<CG>(map_of(mq, 3), &ctl->full[stage], st + 2 * A_TILE + B_TILE + q * 4096, brow + 32 * q, k);
            }
          } else {
            tma_load_cg<CG>(map_of(mq, 2), &ctl->full[stage], st + 2 * A_TILE, k, brow);
            tma_load_cg<CG>(map_of(mq, 3), &ctl->full[stage], st + 2 * A_TILE + B_TILE, k, brow);
          }
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    // ===================== MMA issuer (leader CTA) =====================
    // The k-loop of a tile is cut into chunks of CHUNK_KB k-blocks. Each chunk
    // accumulates into one of two TMEM slots; the epilogue warps drain a
    // finished slot into fp32 registers (round-to-nearest adds) while the next
    // chunk runs in the other slot. The tensor-core accumulate truncates, so
    // this bounds the truncation bias to one chunk.
    if (leader && lane == 0) {
      constexpr uint32_t idesc_k = idesc_tf32(BM * CG, BN);
      int stage = 0;
      uint32_t phase = 0;
      int chunk_it = 0;
      int ul = 0;
      UnitIter ui = iter_init(ch, tile0, tile_step);
      int ph;
      long long uph;
      Unit un;
      for (; iter_next(ch, ui, ph, uph, un); ++ul) {
        const Params& p = ch.ph[ph];
        const int kbA = un.kbA, kbB = un.kbB;
        const uint32_t idesc = idesc_k | (p.b_mn ? (1u << 16) : 0u);  // B MN-major (bit 16)
        TSTAMP(ul, 0);
        for (int kb0 = kbA; kb0 < kbB; kb0 += CHUNK_KB, ++chunk_it) {
          const int slot = chunk_it & 1;
          const uint32_t slot_phase = (chunk_it >> 1) & 1;
          if constexpr (CG == 2)  // every epilogue (both CTAs) drained this slot
            mbar_wait_cluster(&ctl->tempty[slot], slot_phase ^ 1);
          else
            mbar_wait(&ctl->tempty[slot], slot_phase ^ 1);
          tc_fence_after();
          // BN=128: `big` takes a_hi*b_hi, `small` the cross terms a_hi*b_lo +
          // a_lo*b_hi (2^-11 smaller), rounded at their own scale.
          const uint32_t d_big = tmem_base + slot * C::SLOT_COLS;
          const uint32_t d_small = C::SPLIT_ACC ? d_big + BN : d_big;
          const int kb1 = min(kb0 + CHUNK_KB, kbB);
          for (int kb = kb0; kb < kb1; ++kb) {
            mbar_wait(&ctl->full[stage], phase);
            tc_fence_after();
            const uint32_t st = smem_u32(smem + stage * STAGE_BYTES);
#pragma unroll
            for (int kk = 0; kk < BK / 8; ++kk) {
              const uint64_t ah = umma_desc_k_sw128(st + kk * 32);
              const uint64_t al = umma_desc_k_sw128(st + A_TILE + kk * 32);
              const uint64_t bh = p.b_mn ? umma_desc_mn_sw128b32(st + 2 * A_TILE + kk * 1024, 4096, 512)
                                         : umma_desc_k_sw128(st + 2 * A_TILE + kk * 32);
              const uint64_t bl = p.b_mn ? umma_desc_mn_sw128b32(st + 2 * A_TILE + B_TILE + kk * 1024, 4096, 512)
                                         : umma_desc_k_sw128(st + 2 * A_TILE + B_TILE + kk * 32);
              const uint32_t accum = (kb > kb0 || kk > 0) ? 1u : 0u;
              mma_cg<CG>(d_small, al, bh, idesc, accum);
              mma_cg<CG>(d_small, ah, bl, idesc, 1);
              mma_cg<CG>(d_big, ah, bh, idesc, C::SPLIT_ACC ? accum : 1u);
            }
            commit_cg<CG>(&ctl->empty[stage]);  // frees the stage (in both CTAs) when these MMAs finish
            if (++stage == STAGES) { stage = 0; phase ^= 1; }
          }
          commit_cg<CG>(&ctl->tfull[slot]);  // chunk partial sums ready for the epilogues
        }
        TSTAMP(ul, 1);
      }
    }
  } else {
    // ===================== epilogue (warps 2..5 of every CTA) =====================
    const int q = warp & 3;                    // TMEM lane quarter this warp may access
    const int chalf = (warp - 2) / 4;          // which EPI_COLS-wide column half of the tile
    const int cbase = chalf * EPI_COLS;
    int chunk_it = 0;
    int ul = 0;
    // ---- chain: the later phase's operand splits (hi = rna_tf32(x), lo = rna_tf32(x - hi)),
    // shared by the epilogue warps of all CTAs in 32 x 32 blocks, done one block at a time
    // while a warp would otherwise spin on an accumulator chunk (so the MMA never waits for
    // a drain); the last warp of a CTA to finish publishes the CTA's part (release add).
    const int ew = warp - 2;
    float* const stg = reinterpret_cast<float*>(smem + STAGES * STAGE_BYTES + 1024) + ew * (PRE_STAGE / 4);
    const long long gw = (long long)blockIdx.x * C::EPI_WARPS + ew, nw = (long long)gridDim.x * C::EPI_WARPS;
    int pre_k = 0;
    long long pre_blk = gw;
    bool pre_left = CHAIN && ch.npre > 0;
    auto pre_step = [&]() {  // warp-uniform: one block of task pre_k, then advance
      const Chain::Pre& t = ch.pre[pre_k];
      const int br = (t.rows + 31) / 32, bc = (t.cols + 31) / 32;
      if (pre_blk < (long long)br * bc) {
        const int r0 = (int)(pre_blk / bc) * 32, c0 = (int)(pre_blk % bc) * 32;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const int rr = i * 4 + (lane >> 3), cq = lane & 7;  // block row, 16-B chunk: 4 rows x 128 B per load
          const int r = r0 + rr, c = c0 + cq * 4;
          const bool in = r < t.rows && c < t.cols;
          const float4 v = in ? *reinterpret_cast<const float4*>(t.X + (long long)r * t.ldx + c)
                              : make_float4(0.f, 0.f, 0.f, 0.f);
          if (t.transpose == 2) {
            if (in)
              *reinterpret_cast<float4*>(t.lo + (long long)r * t.ldo + c) =
                  make_float4(lo_of_raw(v.x), lo_of_raw(v.y), lo_of_raw(v.z), lo_of_raw(v.w));
          } else if (!t.transpose) {
            if (in) {
              float4 h, l;
              split3x(v.x, h.x, l.x); split3x(v.y, h.y, l.y); split3x(v.z, h.z, l.z); split3x(v.w, h.w, l.w);
              *reinterpret_cast<float4*>(t.hi + (long long)r * t.ldo + c) = h;
              *reinterpret_cast<float4*>(t.lo + (long long)r * t.ldo + c) = l;
            }
          } else {
            *reinterpret_cast<float4*>(stg + rr * 32 + ((cq ^ (rr & 7)) << 2)) = v;  // 16-B XOR swizzle
          }
        }
        if (t.transpose == 1) {
          __syncwarp();
          for (int cc = 0; cc < 32; ++cc) {  // output row c0 + cc (input column), element r0 + lane
            const int j = c0 + cc, i2 = r0 + lane;
            const float x = stg[lane * 32 + ((((cc >> 2) ^ (lane & 7)) << 2) | (cc & 3))];
            if (j < t.cols && i2 < t.rows) {
              float h, l;
              split3x(x, h, l);
              t.hi[(long long)j * t.ldo + i2] = h;
              t.lo[(long long)j * t.ldo + i2] = l;
            }
          }
          __syncwarp();
        }
        pre_blk += nw;
      }
      if (pre_blk >= (long long)br * bc) {
        if (++pre_k < ch.npre) {
          pre_blk = gw;
        } else {
          pre_left = false;
          __threadfence();
          asm volatile("fence.proxy.async.global;" ::: "memory");  // for the later phase's TMA reads
          __syncwarp();
          if (lane == 0 && atomicAdd(&ctl->pre_warps_done, 1u) == (unsigned)C::EPI_WARPS - 1) {
            __threadfence();
            asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(ch.cnt + ch.pre_off) : "memory");
          }
        }
      }
    };
    uint32_t cpar = 0;  // TMA-store epilogue: parities of this warp's two C-box barriers (bits 0, 1)
    // (lane 0) request C box b (32 rows from brow, 16 columns) into staging buffer b & 1
    auto load_c = [&](int b, int col0, int brow) {
      uint64_t* bar = &ctl->cbar[2 * ew + (b & 1)];
      mbar_arrive_expect_tx(bar, 32 * 16 * 4);
      tma_load_2d(map_of(2, 2), bar, stg + (b & 1) * 512, col0 + cbase + b * 16, brow - ch.ph[0].out_row0);  // map 10
    };
    UnitIter ui = iter_init(ch, tile0, tile_step);
    int ph;
    long long u;  // unit index within the phase
    Unit un;
    for (; iter_next(ch, ui, ph, u, un); ++ul) {
      const Params& p = ch.ph[ph];
      const long long t = un.t;
      const uint32_t flags = p.flags;
      const int kbA = un.kbA, kbB = un.kbB;
      int tm, tn;
      tile_coords(p, t, tm, tn);
      bool cpre = false;  // TMA-store epilogue: C boxes 0 and 1 already requested
      if (!CHAIN && p.tma_epi && (flags & EPI_CIN) && !un.split) {
        const int r0 = tm * C::PAIR_M + (int)rank * BM;
        if (!((flags & EPI_TRI) && (tn * BN + BN - 1 > r0))) {  // not a diagonal tile (row stores)
          if (lane == 0) {
            bulk_wait_read0();  // the previous tile's stores have read the buffers
            if (tn * BN + cbase < p.N) load_c(0, tn * BN, r0 + q * 32);
            if (tn * BN + cbase + 16 < p.N) load_c(1, tn * BN, r0 + q * 32);
          }
          cpre = true;
        }
      }
      float acc[EPI_COLS];  // this thread's row x column-half of the tile, fp32 registers
#pragma unroll
      for (int c = 0; c < EPI_COLS; ++c) acc[c] = 0.f;
      for (int kb0 = kbA; kb0 < kbB; kb0 += CHUNK_KB, ++chunk_it) {
        const int slot = chunk_it & 1;
        const uint32_t slot_phase = (chunk_it >> 1) & 1;
        if (CHAIN && pre_left) {  // in-launch splits fill the wait for this accumulator chunk
          const uint32_t ta = smem_u32(&ctl->tfull[slot]);
          while (pre_left && !__shfl_sync(0xffffffffu, lane == 0 ? (int)mbar_try_wait(ta, slot_phase) : 0, 0)) pre_step();
        }
        mbar_wait(&ctl->tfull[slot], slot_phase);
        tc_fence_after();
        if (kb0 == kbA && warp == 2 && lane == 0) TSTAMP(ul, 2);
        __syncwarp();
        const uint32_t ta = tmem_base + ((uint32_t)(q * 32) << 16) + slot * C::SLOT_COLS + cbase;
#pragma unroll
        for (int c0 = 0; c0 < EPI_COLS; c0 += 16) {
          uint32_t r[16];
          tmem_ld16(ta + c0, r);
          if constexpr (C::SPLIT_ACC) {
            uint32_t rs[16];
            tmem_ld16(ta + BN + c0, rs);
            tmem_wait_ld();
#pragma unroll
            for (int e = 0; e < 16; ++e) acc[c0 + e] += __uint_as_float(r[e]) + __uint_as_float(rs[e]);
          } else {
            tmem_wait_ld();
#pragma unroll
            for (int e = 0; e < 16; ++e) acc[c0 + e] += __uint_as_float(r[e]);
          }
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) {
          if constexpr (CG == 2)
            mbar_arrive_cluster(map_peer(smem_u32(&ctl->tempty[slot]), 0));  // leader's barrier
          else
            mbar_arrive(&ctl->tempty[slot]);
        }
      }
      if (warp == 2 && lane == 0) TSTAMP(ul, 3);
      if (un.split && (flags & EPI_PARTIAL)) {  // partials only; launch_gram_combine finishes
        const int rl = q * 32 + lane;
        float4* mine = reinterpret_cast<float4*>(p.part) + ((un.slot * CG + rank) * (long long)BN + cbase) * (BM / 4) + rl;
#pragma unroll
        for (int c = 0; c < EPI_COLS; c += 4) mine[(c / 4) * BM] = make_float4(acc[c], acc[c + 1], acc[c + 2], acc[c + 3]);
        continue;
      }
      if (un.split && un.nseg > 1 && p.dbg != 1) {
        // Split-K: post this unit's partial tile, count arrivals; the LAST unit of
        // the tile to arrive sums all partials in split order (deterministic,
        // no waiting) and runs the epilogue; the others are done with the tile.
        // partial layout [unit][rank][col half][c/4][row 0..127][4]: lanes (rows) write
        // consecutive 16-byte pieces, every access is a coalesced 512-byte line set
        const int rl = q * 32 + lane;
        float4* mine = reinterpret_cast<float4*>(p.part) + ((un.slot * CG + rank) * (long long)BN + cbase) * (BM / 4) + rl;
#pragma unroll
        for (int c = 0; c < EPI_COLS; c += 4) mine[(c / 4) * BM] = make_float4(acc[c], acc[c + 1], acc[c + 2], acc[c + 3]);
        __threadfence();
        asm volatile("bar.sync 1, %0;" ::"r"(C::EPI_WARPS * 32) : "memory");
        if (warp == 2 && lane == 0) {
          unsigned* cnt = p.counters + (t - p.split_t0) * CG + rank;
          const unsigned prev = atomicAdd(cnt, 1u);
          const uint32_t last = prev == (unsigned)(un.nseg - 1);
          if (last) atomicExch(cnt, 0u);
          ctl->last_flag = last;
        }
        asm volatile("bar.sync 1, %0;" ::"r"(C::EPI_WARPS * 32) : "memory");
        if (!ctl->last_flag) continue;
        __threadfence();
        // sum partials 0..ksplit-1 in order (own partial re-read from L2: same order
        // whichever unit arrives last)
        for (int k2 = 0; k2 < un.nseg; ++k2) {
          const float4* o = reinterpret_cast<const float4*>(p.part) +
                            ((slot_of(p, t, k2) * CG + rank) * (long long)BN + cbase) * (BM / 4) + rl;
#pragma unroll
          for (int c = 0; c < EPI_COLS; c += 4) {
            const float4 v = __ldcg(o + (c / 4) * BM);
            if (k2 == 0) {
              acc[c] = v.x; acc[c + 1] = v.y; acc[c + 2] = v.z; acc[c + 3] = v.w;
            } else {
              acc[c] += v.x; acc[c + 1] += v.y; acc[c + 2] += v.z; acc[c + 3] += v.w;
            }
          }
        }
      }
      if (warp == 2 && lane == 0) TSTAMP(ul, 4);
      const int row0 = tm * C::PAIR_M + (int)rank * BM;  // first output row of this CTA
      const int i = row0 + q * 32 + lane;                // this thread's output row
      const bool row_ok = i < p.M;
      const bool diag_tile = (flags & EPI_TRI) && (tn * BN + BN - 1 > row0);  // tile crosses j > i
      const long long orow = (long long)(i - p.out_row0);
      if (!CHAIN && p.tma_epi && !diag_tile) {
        // Staged TMA-store epilogue (S4): this warp's 32 rows leave in 32 x 16 boxes through
        // two 2 KB staging buffers (64-B swizzle: 16-B piece c of row r at c ^ ((r >> 1) & 3),
        // conflict-free). Per box: the C box arrives by TMA (EPI_CIN; boxes 0 and 1 are
        // requested before the accumulator is drained, box b + 2 once box b's store has read
        // its buffer), every lane writes its row's 16 values, and one lane stores the box with
        // cp.async.bulk.tensor (ragged rows / columns clipped by the tensor map). EPI_SPLIT_LO
        // reuses the buffer for lo once the out store has read it.
        const int brow = row0 + q * 32;  // first row of this warp's block
        constexpr int NBOX = EPI_COLS / 16;
        if ((flags & EPI_CIN) && !cpre && lane == 0) {
          bulk_wait_read0();
          if (tn * BN + cbase < p.N) load_c(0, tn * BN, brow);
          if (tn * BN + cbase + 16 < p.N) load_c(1, tn * BN, brow);
        }
#pragma unroll
        for (int b = 0; b < NBOX; ++b) {
          const int j0 = tn * BN + cbase + b * 16;
          if (j0 >= p.N) break;
          float* const buf = stg + (b & 1) * 512;
          if (flags & EPI_CIN) {
            mbar_wait(&ctl->cbar[2 * ew + (b & 1)], (cpar >> (b & 1)) & 1u);
            cpar ^= 1u << (b & 1);
          } else {
            if (lane == 0) {  // the buffer's previous store has read it
              if (b == 0) bulk_wait_read0();
              else if (b >= 2 && (flags & EPI_SPLIT_LO)) bulk_wait_read<2>();
              else if (b >= 2) bulk_wait_read<1>();
            }
            __syncwarp();
          }
#pragma unroll
          for (int c4 = 0; c4 < 4; ++c4) {
            float4* sp = reinterpret_cast<float4*>(buf + lane * 16 + ((c4 ^ ((lane >> 1) & 3)) << 2));
            const int e = b * 16 + c4 * 4;
            float4 w = make_float4(p.alpha * acc[e], p.alpha * acc[e + 1], p.alpha * acc[e + 2], p.alpha * acc[e + 3]);
            if (flags & EPI_CIN) {
              const float4 c = *sp;
              w.x += p.beta * c.x; w.y += p.beta * c.y; w.z += p.beta * c.z; w.w += p.beta * c.w;
            }
            if (flags & EPI_DIAG_ONE) {
              const int d = i - (j0 + c4 * 4);
              if (d == 0) w.x = 1.f; else if (d == 1) w.y = 1.f; else if (d == 2) w.z = 1.f; else if (d == 3) w.w = 1.f;
            }
            *sp = w;
          }
          fence_proxy_smem();
          __syncwarp();
          if (lane == 0) {
            tma_store_2d(map_of(2, 0), buf, j0, brow - p.out_row0);  // map 8: out
            bulk_commit();
          }
          if (flags & EPI_SPLIT_LO) {
            if (lane == 0) bulk_wait_read0();
            __syncwarp();
#pragma unroll
            for (int c4 = 0; c4 < 4; ++c4) {
              float4* sp = reinterpret_cast<float4*>(buf + lane * 16 + ((c4 ^ ((lane >> 1) & 3)) << 2));
              const float4 w = *sp;
              *sp = make_float4(lo_of_raw(w.x), lo_of_raw(w.y), lo_of_raw(w.z), lo_of_raw(w.w));
            }
            fence_proxy_smem();
            __syncwarp();
            if (lane == 0) {
              tma_store_2d(map_of(2, 1), buf, j0, brow);  // map 9: split_lo (rows i, like EPI_SPLIT_LO)
              bulk_commit();
            }
          }
          if ((flags & EPI_CIN) && b + 2 < NBOX && j0 + 32 < p.N && lane == 0) {
            bulk_wait_read0();  // this box's store(s) have read the buffer
            load_c(b + 2, tn * BN, brow);
          }
        }
        if (warp == 2 && lane == 0) TSTAMP(ul, 5);
        continue;
      }
#pragma unroll
      for (int c0 = 0; c0 < EPI_COLS; c0 += 16) {
        const int j0 = tn * BN + cbase + c0;
        if (row_ok && j0 < p.N) {
          float v[16];
#pragma unroll
          for (int e = 0; e < 16; ++e) v[e] = p.alpha * acc[c0 + e];
          if (flags & EPI_CIN) {
            const float* cp = p.cin + orow * p.ldc + j0;
#pragma unroll
            for (int e = 0; e < 16; e += 4) {
              if (j0 + e < p.N) {
                float4 c = *reinterpret_cast<const float4*>(cp + e);
                v[e] += p.beta * c.x; v[e + 1] += p.beta * c.y; v[e + 2] += p.beta * c.z; v[e + 3] += p.beta * c.w;
              }
            }
          }
          if (flags & EPI_DIAG_ONE) {
#pragma unroll
            for (int e = 0; e < 16; ++e)
              if (j0 + e == i) v[e] = 1.0f;
          }
          if (!diag_tile) {
            if (flags & EPI_OUT) {
              float* op = p.out + orow * p.ldo + j0;
#pragma unroll
              for (int e = 0; e < 16; e += 4)
                if (j0 + e < p.N) store4(op + e, v[e], v[e + 1], v[e + 2], v[e + 3]);
            }
            if (flags & EPI_SPLIT_LO) {  // raw-hi split of the output: the next GEMM reads (out, lo)
              float* lp = p.split_lo + (long long)i * p.ld_split + j0;
#pragma unroll
              for (int e = 0; e < 16; e += 4)
                if (j0 + e < p.N)
                  store4(lp + e, lo_of_raw(v[e]), lo_of_raw(v[e + 1]), lo_of_raw(v[e + 2]), lo_of_raw(v[e + 3]));
            }
            if (flags & EPI_SPLIT) {
              float* hp = p.split_hi + (long long)i * p.ld_split + j0;
              float* lp = p.split_lo + (long long)i * p.ld_split + j0;
#pragma unroll
              for (int e = 0; e < 16; e += 4) {
                if (j0 + e < p.N) {
                  float h[4], l[4];
#pragma unroll
                  for (int u = 0; u < 4; ++u) split3x(v[e + u], h[u], l[u]);
                  store4(hp + e, h[0], h[1], h[2], h[3]);
                  store4(lp + e, l[0], l[1], l[2], l[3]);
                }
              }
            }
          } else {  // tile crosses the diagonal: element mask j <= i
            if (flags & EPI_OUT) {
              float* op = p.out + orow * p.ldo + j0;
#pragma unroll
              for (int e = 0; e < 16; ++e)
                if (j0 + e < p.N && j0 + e <= i) op[e] = v[e];
            }
          }
          if (flags & EPI_MIRROR) {  // out[j][i] = v for j < i
#pragma unroll
            for (int e = 0; e < 16; ++e) {
              const int j = j0 + e;
              if (j < p.N && j < i) p.out[(long long)(j - p.out_row0) * p.ldo + i] = v[e];
            }
          }
          if (flags & EPI_SPLIT_T) {
#pragma unroll
            for (int e = 0; e < 16; ++e) {
              const int j = j0 + e;
              if (j < p.N) {
                float h, l;
                split3x(v[e], h, l);
                p.split_hi[(long long)j * p.ld_split + i] = h;
                p.split_lo[(long long)j * p.ld_split + i] = l;
              }
            }
          }
        }
      }
      if (warp == 2 && lane == 0) TSTAMP(ul, 5);
      if (CHAIN && ch.sig_kind[ph]) {  // chain: publish this CTA's part of the finished tile
        __threadfence();
        asm volatile("fence.proxy.async.global;" ::: "memory");  // for the next phase's TMA reads
        asm volatile("bar.sync 1, %0;" ::"r"(C::EPI_WARPS * 32) : "memory");
        if (warp == 2 && lane == 0) {
          unsigned* c = ch.cnt + ch.sig_off[ph] + (ch.sig_kind[ph] == 1 ? tm * CG + (int)rank : tn);
          asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(c) : "memory");
        }
      }
    }
    if constexpr (CHAIN) {
      while (pre_left) pre_step();  // (a CTA with few units: the rest of its share of the splits)
    }
    if (!CHAIN && lane == 0) bulk_wait0();  // this warp's TMA stores are complete
  }

  tc_fence_before();
  if constexpr (CG == 2) cluster_sync_all(); else __syncthreads();
  tl_exit(tl, g_tl, 0);
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc_cg<CG>(tmem_base, TMEM_COLS);
  }
}

// Tile/split fields of one GEMM (phase) for the tile config <CG, BN>; false if it has no tiles.
template <int CG, int BN>
bool prep_phase(const GemmDesc& d, Params& p, int ksplit, long long split_tiles, const UmmaPlan* skp = nullptr) {
  using C = Cfg<CG, BN>;
  const int tiles_m = (d.M + C::PAIR_M - 1) / C::PAIR_M;
  p.tiles_n = (d.N + BN - 1) / BN;
  p.ratio = C::PAIR_M / BN;
  p.tm0 = d.tm0 * 128 / C::PAIR_M;  // d.tm0 is in 128-row units
  p.tm1 = d.tm1 < 0 ? tiles_m : (d.tm1 * 128 + C::PAIR_M - 1) / C::PAIR_M;
  if (p.tm1 > tiles_m) p.tm1 = tiles_m;
  if (p.tm1 <= p.tm0) return false;
  long long nt = 0;
  for (int tm = p.tm0; tm < p.tm1; ++tm)
    nt += (d.flags & EPI_TRI) ? std::min(p.ratio * (tm + 1), p.tiles_n) : p.tiles_n;
  p.num_tiles = nt;
  p.ksplit = ksplit;
  p.split_tiles = (ksplit > 1 || (d.flags & EPI_PARTIAL)) ? split_tiles : 0;
  static const bool split_first = getenv("PB_SPLIT_FIRST") && atoi(getenv("PB_SPLIT_FIRST")) != 0;
  p.split_t0 = (split_first || (d.flags & EPI_PARTIAL)) ? 0 : nt - p.split_tiles;
  static const int gm = getenv("PB_GROUP_M") ? atoi(getenv("PB_GROUP_M")) : 0;
  p.group_m = gm > 0 ? gm : GROUP_M;
  static const int dbg = getenv("PB_UMMA_DEBUG") ? atoi(getenv("PB_UMMA_DEBUG")) : 0;
  p.dbg = dbg;
  static const bool timing = getenv("PB_UMMA_TIMING") != nullptr;
  static unsigned long long* tbuf = nullptr;
  if (timing && !tbuf) cudaMalloc(&tbuf, 148 * 16 * 8 * sizeof(unsigned long long));  // debug only
  p.tstamp = timing ? tbuf : nullptr;
  p.part = d.part;
  p.counters = d.counters;
  p.b_mn = d.b[0].mn ? 1 : 0;
  p.tma_epi = 0;
  p.streamk = 0;
  p.sk_iters = 0; p.sk_pairs = 1; p.sk_maxseg = 1;
  if (skp && skp->streamk) {
    p.streamk = 1;
    p.sk_pairs = num_sms() / CG;
    p.sk_iters = nt * (long long)(p.nkb * p.npairs);
    p.sk_maxseg = skp->maxseg;
    p.split_tiles = nt;  // every tile may be split (its segment count decides)
    p.split_t0 = 0;
  }
  return true;
}
inline long long phase_units(const Params& p) {
  return p.streamk ? p.sk_pairs : p.split_tiles * p.ksplit + (p.num_tiles - p.split_tiles);
}

template <int CG, int BN>
bool phase_maps(const GemmDesc& d, CUtensorMap* maps /* 4 per operand pair */) {
  using C = Cfg<CG, BN>;
  for (int q = 0; q < d.npairs; ++q) {
    const SplitOperand& A = d.a[q];
    const SplitOperand& B = d.b[q];
    if (!make_map(&maps[4 * q + 0], A.hi, A.rows, A.K, A.ld, BM) ||
        !make_map(&maps[4 * q + 1], A.lo, A.rows, A.K, A.ld, BM))
      return false;
    if (B.mn) {  // B[k][n] (K rows x rows columns): 32-column x 32-row boxes, 128B_BASE32B swizzle
      if (!make_map2d(&maps[4 * q + 2], B.hi, B.rows, B.K, B.ld, 32, BK, true, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B) ||
          !make_map2d(&maps[4 * q + 3], B.lo, B.rows, B.K, B.ld, 32, BK, true, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B))
        return false;
    } else if (!make_map(&maps[4 * q + 2], B.hi, B.rows, B.K, B.ld, C::B_ROWS) ||
               !make_map(&maps[4 * q + 3], B.lo, B.rows, B.K, B.ld, C::B_ROWS)) {
      return false;
    }
  }
  return true;
}

template <int CG, int BN, bool CHAIN>
cudaError_t launch_chain_kernel(const Chain& ch, const CUtensorMap* maps, cudaStream_t s, int* launches);

template <int CG, int BN>
cudaError_t launch_cg(const GemmDesc& d, Params p, int ksplit, long long split_tiles, cudaStream_t s, int* launches,
                      const UmmaPlan* skp = nullptr) {
  if (!prep_phase<CG, BN>(d, p, ksplit, split_tiles, skp)) return cudaSuccess;
  if (p.tstamp) cudaMemsetAsync(p.tstamp, 0, 148 * 16 * 8 * sizeof(unsigned long long), s);
  if (p.streamk) {
    cudaError_t e = cudaMemsetAsync(d.counters, 0, (size_t)p.num_tiles * CG * sizeof(unsigned), s);
    if (e != cudaSuccess) return e;
  } else if (ksplit > 1 && !(d.flags & EPI_PARTIAL)) {
    cudaError_t e = cudaMemsetAsync(d.counters, 0, (size_t)p.split_tiles * CG * sizeof(unsigned), s);
    if (e != cudaSuccess) return e;
  }
  CUtensorMap maps[12];
  if (!phase_maps<CG, BN>(d, maps)) return cudaErrorInvalidValue;
  for (int q = 4 * d.npairs; q < 12; ++q) maps[q] = maps[q % 4];
  // staged TMA-store epilogue (maps 8 = out, 9 = split_lo, 10 = cin; free in a one-GEMM launch,
  // syr2k's second pair uses 4..7) when every output is a plain row-major store with 16-B rows
  static const bool tma_off = getenv("PB_TMA_EPI") && atoi(getenv("PB_TMA_EPI")) == 0;
  auto al16 = [](const void* x, long long ld) { return x && ((uintptr_t)x & 15) == 0 && ld % 4 == 0; };
  if (!tma_off && (d.flags & EPI_OUT) && !(d.flags & (EPI_MIRROR | EPI_SPLIT | EPI_SPLIT_T | EPI_PARTIAL)) &&
      d.M > d.out_row0 && al16(d.out, d.ldo) && (!(d.flags & EPI_CIN) || al16(d.cin, d.ldc)) &&
      (!(d.flags & EPI_SPLIT_LO) || al16(d.split_lo, d.ld_split))) {
    const CUtensorMapSwizzle sw = CU_TENSOR_MAP_SWIZZLE_64B;  // 32 x 16 boxes (64-B rows)
    const bool ok = make_map2d(&maps[8], d.out, d.N, d.M - d.out_row0, d.ldo, 16, 32, false, sw) &&
                    (!(d.flags & EPI_SPLIT_LO) || make_map2d(&maps[9], d.split_lo, d.N, d.M, d.ld_split, 16, 32, false, sw)) &&
                    (!(d.flags & EPI_CIN) || make_map2d(&maps[10], d.cin, d.N, d.M - d.out_row0, d.ldc, 16, 32, false, sw));
    if (ok)
      p.tma_epi = 1;
    else
      for (int q = 8; q < 12; ++q) maps[q] = maps[q % 4];
  }
  Chain ch{};
  ch.nphase = 1;
  ch.ph[0] = p;
  ch.ubase[0] = 0;
  ch.ubase[1] = phase_units(p);
  for (int q = 0; q < 3; ++q) { ch.waitA_off[q] = -1; ch.waitB_off[q] = -1; }
  cudaError_t e = launch_chain_kernel<CG, BN, false>(ch, maps, s, launches);
  if (e != cudaSuccess) return e;
  cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
  if (p.tstamp) cudaStreamIsCapturing(s, &cap);
  const long long units = std::min<long long>(phase_units(p), num_sms() / CG);
  if (p.tstamp && cap == cudaStreamCaptureStatusNone) {  // debug: per-phase durations (us), medians over CTAs/units
    std::vector<unsigned long long> h(148 * 16 * 8);
    cudaStreamSynchronize(s);
    cudaMemcpy(h.data(), p.tstamp, h.size() * 8, cudaMemcpyDeviceToHost);
    unsigned long long t0 = ~0ull, t1 = 0;
    std::vector<double> mma, drain_lag, split, store;
    for (int c = 0; c < (int)(units * CG); ++c)
      for (int u = 0; u < 16; ++u) {
        const unsigned long long* ev = &h[((size_t)c * 16 + u) * 8];
        for (int k = 0; k < 6; ++k)
          if (ev[k]) { t0 = std::min(t0, ev[k]); t1 = std::max(t1, ev[k]); }
        if (ev[0] && ev[1]) mma.push_back((ev[1] - ev[0]) / 1e3);
        if (ev[1] && ev[3]) drain_lag.push_back(((long long)ev[3] - (long long)ev[1]) / 1e3);
        if (ev[3] && ev[4]) split.push_back((ev[4] - ev[3]) / 1e3);
        if (ev[4] && ev[5]) store.push_back((ev[5] - ev[4]) / 1e3);
      }
    auto med = [](std::vector<double> v) { if (v.empty()) return 0.0; std::sort(v.begin(), v.end()); return v[v.size() / 2]; };
    fprintf(stderr, "[pb timing] span %.1f us | per unit median: mma %.1f, mma-end->drained %.1f, split-exchange %.1f, "
            "stores %.1f us (n=%zu)\n", (t1 - t0) / 1e3, med(mma), med(drain_lag), med(split), med(store), mma.size());
  }
  if (getenv("PB_TRACE"))
    fprintf(stderr, "[pb] umma3x<%d,%d> M=%d N=%d K=%d pairs=%d flags=0x%x tiles=%lld split %lldx%d grid=%lld\n", CG,
            BN, d.M, d.N, d.K, d.npairs, d.flags, p.num_tiles, p.split_tiles, p.ksplit, units * CG);
  return cudaSuccess;
}

template <int CG, int BN, bool CHAIN>
cudaError_t launch_chain_kernel(const Chain& ch, const CUtensorMap* maps, cudaStream_t s, int* launches) {
  using C = Cfg<CG, BN>;
  // CHAIN: + per-epilogue-warp transpose staging for the in-launch operand splits
  // + Ctl (1 KB) + per-epilogue-warp 4 KB staging: the chain's transposes, else the TMA-store boxes
  const size_t smem = C::STAGES * C::STAGE_BYTES + 1024 + 1024 + C::EPI_WARPS * PRE_STAGE;
  {
    const cudaError_t e = ensure_smem<umma3x_kernel<CG, BN, CHAIN>>(smem);
    if (e != cudaSuccess) return e;
  }
  const long long max_units = num_sms() / CG;
  const long long work = ch.ubase[ch.nphase];
  const long long units = work < max_units ? work : max_units;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(units * CG));
  cfg.blockDim = dim3(C::NUM_THREADS);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = CG; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
  at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 2;
  cudaError_t e = cudaLaunchKernelEx(&cfg, umma3x_kernel<CG, BN, CHAIN>, maps[0], maps[1], maps[2], maps[3], maps[4], maps[5],
                                     maps[6], maps[7], maps[8], maps[9], maps[10], maps[11], ch);
  if (launches) ++*launches;
  return e != cudaSuccess ? e : cudaGetLastError();
}

// Gram combine (EPI_PARTIAL): one CTA per (tile, rank, 32-row block). Partials
// (layout [unit][rank][half][c4][row][4]) are read with lanes on rows (coalesced),
// summed in split order (deterministic), staged in padded smem, then written
// row-major with lanes on columns and mirrored with lanes on rows (both coalesced).
// With band statistics (banded prep, reading R18) it adds the between-band scatter
//   sum_b n_b (mu_b - c)_i (mu_b - c)_j,   c = sum_b n_b mu_b / float_n,
// and for correlation scales by inv_i inv_j, inv = 1/(sqrt(float_n) sd), sd from
// (sum_b M2_b + sum_b n_b (mu_b - c)^2) / float_n with the eps rule (fp64).
struct CombineStats {
  const double* band_mean;
  const double* band_m2;
  int nbands, n, corr;
  double float_n, eps;
  float* mean_out;
  float* sd_out;
};
constexpr int MAXB = 8;

template <int CG, int BN>
__global__ void __launch_bounds__(256) gram_combine_kernel(const Params p, int diag_one, const CombineStats cs) {
  constexpr int PAIR_M = BM * CG, C4 = BN / 4, NCOL = 32 + BN;
  // tile: padded [32][BN+1] on the general path, XOR-swizzled [32][BN] float4 quads on the fast path
  __shared__ __align__(16) float tile_raw[32 * (BN + 1)];
  __shared__ __align__(16) float dev_s[MAXB][NCOL];  // mu_b - c (fp32 is ample: the term is summed in fp64)
  __shared__ __align__(16) float inv_s[NCOL];        // 1/(sqrt(float_n) sd) for rows, columns (1 for covariance)
  pdl_trigger();  // dependents may start their setup once every CTA here runs
  pdl_wait();
  const int tl = g_tl_on;
  tl_enter(tl, g_tl, 1);
  const int blk = blockIdx.x;
  const long long t = blk / (CG * 4);
  const int rank = (blk / 4) % CG, rb = blk % 4;
  int tm, tn;
  tile_coords(p, t, tm, tn);
  const int row_base = tm * PAIR_M + rank * BM + rb * 32;  // first output row of this block
  const int col_base = tn * BN;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;  // 8 warps
  const bool banded = cs.band_mean != nullptr;
  if (banded) {
    for (int e = threadIdx.x; e < NCOL; e += 256) {
      const int col = e < 32 ? row_base + e : col_base + (e - 32);
      // all band loads issued before any is used (unrolled over MAXB, predicated)
      double S = 0.0, M2 = 0.0, mu[MAXB], m2[MAXB];
      int nb[MAXB];
#pragma unroll
      for (int b = 0; b < MAXB; ++b) {
        const bool in = b < cs.nbands && col < p.N;
        nb[b] = b < cs.nbands ? min(256, cs.n - 256 * b) : 0;
        mu[b] = in ? cs.band_mean[(long long)b * p.N + col] : 0.0;
        m2[b] = in && cs.corr ? cs.band_m2[(long long)b * p.N + col] : 0.0;
      }
#pragma unroll
      for (int b = 0; b < MAXB; ++b) S += nb[b] * mu[b];
      const double c = S / cs.float_n;
      double between = 0.0;
#pragma unroll
      for (int b = 0; b < MAXB; ++b) {
        const double d = b < cs.nbands ? mu[b] - c : 0.0;
        dev_s[b][e] = (float)d;
        between += nb[b] * d * d;
        M2 += m2[b];
      }
      double inv = 1.0;
      double sd = 0.0;
      if (cs.corr) {
        sd = sqrt((M2 + between) / cs.float_n);
        if (sd <= cs.eps) sd = 1.0;
        inv = 1.0 / (sqrt(cs.float_n) * sd);
      }
      inv_s[e] = (float)inv;
      // column statistics outputs: written once, by the diagonal tile's first block
      if (e >= 32 && col < p.N && rank == 0 && rb == 0 && tm == tn / p.ratio) {
        if (cs.mean_out) cs.mean_out[col] = (float)c;
        if (cs.corr && cs.sd_out) cs.sd_out[col] = (float)sd;
      }
    }
    __syncthreads();
  }
  // read + sum: warp w handles c4 = w, w+8, ...; lane = row within the block. All
  // C4/8 loads of one split are issued before any is used (memory-level parallelism).
  constexpr int NC = C4 / 8;
  float4 acc[NC];
#pragma unroll
  for (int k = 0; k < NC; ++k) acc[k] = make_float4(0.f, 0.f, 0.f, 0.f);
  for (int s = 0; s < p.ksplit; ++s) {
    const float4* base = reinterpret_cast<const float4*>(p.part) +
                         (((s * p.split_tiles + t) * CG + rank) * (long long)BN) * (BM / 4) + rb * 32 + lane;
    float4 v[NC];
#pragma unroll
    for (int k = 0; k < NC; ++k) v[k] = __ldcg(base + (long long)(w + 8 * k) * BM);
#pragma unroll
    for (int k = 0; k < NC; ++k) {
      acc[k].x += v[k].x; acc[k].y += v[k].y; acc[k].z += v[k].z; acc[k].w += v[k].w;
    }
  }
  // between-band term for row `lane`: er[b] = n_b (mu_b - c)_row (registers); the column
  // factors are float4 warp-wide broadcasts from smem; 8 fp32 FMAs per element.
  float er[MAXB];
  float rinv = 1.f;
  if (banded) {
#pragma unroll
    for (int b = 0; b < MAXB; ++b) er[b] = b < cs.nbands ? (float)min(256, cs.n - 256 * b) * dev_s[b][lane] : 0.f;
    rinv = inv_s[lane];
  }
#pragma unroll
  for (int k = 0; k < NC; ++k) {
    const int c4 = w + 8 * k;
    float4 v = acc[k];
    if (banded) {
      float4 bt = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
      for (int b = 0; b < MAXB; ++b) {
        const float4 f = *reinterpret_cast<const float4*>(&dev_s[b][32 + 4 * c4]);
        bt.x = fmaf(er[b], f.x, bt.x); bt.y = fmaf(er[b], f.y, bt.y);
        bt.z = fmaf(er[b], f.z, bt.z); bt.w = fmaf(er[b], f.w, bt.w);
      }
      v.x += bt.x; v.y += bt.y; v.z += bt.z; v.w += bt.w;
      if (cs.corr) {
        const float4 ic = *reinterpret_cast<const float4*>(&inv_s[32 + 4 * c4]);
        v.x *= rinv * ic.x; v.y *= rinv * ic.y; v.z *= rinv * ic.z; v.w *= rinv * ic.w;
      } else {
        v.x *= p.alpha; v.y *= p.alpha; v.z *= p.alpha; v.w *= p.alpha;
      }
    } else {
      v.x *= p.alpha; v.y *= p.alpha; v.z *= p.alpha; v.w *= p.alpha;
    }
    acc[k] = v;
  }
  // Fast path: a full 32 x BN block strictly below the diagonal (every j < i), 16-byte
  // aligned rows. Mirror out[j][i] straight from registers (lanes = consecutive i: one
  // 128 B segment per store); direct out[i][j] through a swizzled tile (quad c4 of row r
  // at quad c4 ^ (r & 7): both the STS.128 and LDS.128 below are bank-conflict free)
  // as 16-byte stores, 512 B per warp instruction.
  const bool fast = row_base + 32 <= p.M && col_base + BN <= p.N && col_base + BN <= row_base &&
                    (p.ldo & 3) == 0 && (reinterpret_cast<uintptr_t>(p.out) & 15) == 0;
  if (fast) {
    float* mo = p.out + (long long)col_base * p.ldo + row_base + lane;
#pragma unroll
    for (int k = 0; k < NC; ++k) {
      const int c4 = w + 8 * k;
      float* q = mo + (long long)(4 * c4) * p.ldo;
      q[0] = acc[k].x;
      q[p.ldo] = acc[k].y;
      q[2 * (long long)p.ldo] = acc[k].z;
      q[3 * (long long)p.ldo] = acc[k].w;
      *reinterpret_cast<float4*>(&tile_raw[lane * BN + 4 * (c4 ^ (lane & 7))]) = acc[k];
    }
    __syncthreads();
#pragma unroll
    for (int rr = 0; rr < 4; ++rr) {
      const int r = w + 8 * rr;
      float* o = p.out + (long long)(row_base + r) * p.ldo + col_base;
#pragma unroll
      for (int h = 0; h < BN / 128; ++h) {
        const int q4 = lane + 32 * h;
        *reinterpret_cast<float4*>(o + 4 * q4) = *reinterpret_cast<const float4*>(&tile_raw[r * BN + 4 * (q4 ^ (r & 7))]);
      }
    }
    tl_exit(tl, g_tl, 1);
    return;
  }
  // General path (diagonal and ragged blocks): padded tile, per-element bounds.
#pragma unroll
  for (int k = 0; k < NC; ++k) {
    const int c4 = w + 8 * k;
    float* tr = &tile_raw[lane * (BN + 1) + 4 * c4];
    tr[0] = acc[k].x; tr[1] = acc[k].y; tr[2] = acc[k].z; tr[3] = acc[k].w;
  }
  __syncthreads();
  // direct lower part out[i][j], j <= i: lanes on columns
  for (int r = w; r < 32; r += 8) {
    const int i = row_base + r;
    if (i >= p.M) break;
    for (int c = lane; c < BN; c += 32) {
      const int j = col_base + c;
      if (j > i || j >= p.N) break;
      p.out[(long long)i * p.ldo + j] = (diag_one && j == i) ? 1.0f : tile_raw[r * (BN + 1) + c];
    }
  }
  // mirror out[j][i] = v for j < i: lanes on rows i
  const int i = row_base + lane;
  if (i < p.M) {
    for (int c = w; c < BN; c += 8) {
      const int j = col_base + c;
      if (j >= p.N) break;
      if (j < i) p.out[(long long)j * p.ldo + i] = tile_raw[lane * (BN + 1) + c];
    }
  }
  tl_exit(tl, g_tl, 1);
}

}  // namespace

void timeline_umma(bool reset, unsigned long long* out4) {
  if (reset) {
    const int on = 1;
    const unsigned long long init[4] = {~0ull, 0ull, ~0ull, 0ull};
    cudaMemcpyToSymbol(g_tl_on, &on, sizeof on);
    cudaMemcpyToSymbol(g_tl, init, sizeof init);
  } else {
    cudaMemcpyFromSymbol(out4, g_tl, 4 * sizeof(unsigned long long));
  }
}

cudaError_t launch_gram_combine(const GemmDesc& d, const UmmaPlan& pl, bool diag_one, const GramStats& st,
                                cudaStream_t s, int* launches) {
  if (pl.split_tiles <= 0) return cudaSuccess;
  if (pl.part_bytes > d.part_cap) return cudaErrorInvalidValue;
  if (st.nbands > MAXB) return cudaErrorInvalidValue;
  CombineStats cs;
  cs.band_mean = st.band_mean; cs.band_m2 = st.band_m2; cs.nbands = st.nbands; cs.n = st.n;
  cs.corr = st.band_m2 != nullptr; cs.float_n = st.float_n; cs.eps = st.eps;
  cs.mean_out = st.mean_out; cs.sd_out = st.sd_out;
  Params p{};
  p.M = d.M; p.N = d.N; p.flags = d.flags; p.alpha = d.alpha; p.out = d.out; p.ldo = d.ldo;
  p.part = d.part; p.ksplit = pl.ksplit; p.num_tiles = pl.tiles; p.split_tiles = pl.split_tiles;
  const int pm = pl.cfg == 1 ? 128 : 256, bn = pl.cfg == 3 ? 256 : 128;
  p.tm0 = 0;
  p.tm1 = (d.M + pm - 1) / pm;
  p.tiles_n = (d.N + bn - 1) / bn;
  p.ratio = pm / bn;
  const unsigned grid = (unsigned)(pl.split_tiles * (pm / 128) * 4);  // (split tile, rank, 32-row block)
  const int dg = diag_one ? 1 : 0;
  cudaError_t e;
  if (pl.cfg == 3) e = launch_pdl(gram_combine_kernel<2, 256>, dim3(grid), dim3(256), 0, s, p, dg, cs);
  else if (pl.cfg == 2) e = launch_pdl(gram_combine_kernel<2, 128>, dim3(grid), dim3(256), 0, s, p, dg, cs);
  else e = launch_pdl(gram_combine_kernel<1, 128>, dim3(grid), dim3(256), 0, s, p, dg, cs);
  if (launches) ++*launches;
  return e;
}

// ---- NEXT-4 chain fusion: up to 3 dependent GEMMs in one persistent launch (see Chain)
namespace {
Params base_params(const GemmDesc& d) {
  Params p{};
  p.M = d.M; p.N = d.N; p.K = d.K; p.npairs = d.npairs; p.nkb = (d.K + BK - 1) / BK;
  p.flags = d.flags; p.alpha = d.alpha; p.beta = d.beta; p.cin = d.cin; p.ldc = d.ldc;
  p.out = d.out; p.ldo = d.ldo; p.out_row0 = d.out_row0;
  p.split_hi = d.split_hi; p.split_lo = d.split_lo; p.ld_split = d.ld_split;
  return p;
}
}  // namespace

bool umma_chain_ok(const GemmDesc* d, int nphase) {
  // Opt-in (PB_CHAIN=1): measured on B200 at 4096 the chained launch is ~5% slower than the
  // separate launches (the in-launch operand splits cost the epilogue warps' registers and
  // time; the PDL-overlapped kernel boundary it removes is cheap). DESIGN.md §8 "chain".
  static const char* env = getenv("PB_CHAIN");
  if (!env || atoi(env) == 0) return false;
  if (nphase < 1 || nphase > 3) return false;
  for (int q = 0; q < nphase; ++q) {
    const UmmaPlan pl = umma_plan(d[q]);
    if (pl.cfg != 3 || pl.streamk || d[q].npairs != 1 || (d[q].flags & (EPI_TRI | EPI_PARTIAL | EPI_MIRROR)) || d[q].tm0 != 0 ||
        d[q].tm1 >= 0)
      return false;
  }
  return num_sms() >= 2;
}

size_t umma_chain_cnt_bytes(const GemmDesc* d, int nphase) {
  size_t n = 0;
  for (int q = 0; q < nphase; ++q) n += (size_t)((d[q].M + 255) / 256) * 2 + (size_t)((d[q].N + 255) / 256);
  return align_up((n + 1) * sizeof(unsigned), 256);  // + the in-launch split counter
}

cudaError_t launch_umma_chain(const GemmDesc* d, const ChainLink* links, int nphase, unsigned* cnt, size_t cnt_cap,
                              cudaStream_t s, int* launches) {
  if (!umma_chain_ok(d, nphase)) return cudaErrorNotSupported;
  if (umma_chain_cnt_bytes(d, nphase) > cnt_cap) return cudaErrorInvalidValue;
  constexpr int CG = 2, BN = 256;
  Chain ch{};
  ch.nphase = nphase;
  ch.cnt = cnt;
  CUtensorMap maps[12];
  int off = 0;
  int row_off[3], col_off[3];
  for (int q = 0; q < nphase; ++q) {  // counter areas: [tile rows x ranks] then [tile columns] per phase
    row_off[q] = off; off += ((d[q].M + 255) / 256) * CG;
    col_off[q] = off; off += (d[q].N + 255) / 256;
  }
  ch.ubase[0] = 0;
  for (int q = 0; q < nphase; ++q) {
    const UmmaPlan pl = umma_plan(d[q]);
    int ks = pl.ksplit;
    if (ks > 1 && (d[q].part == nullptr || d[q].counters == nullptr)) ks = 1;
    if (ks > 1 && (pl.part_bytes > d[q].part_cap || pl.counter_bytes > d[q].counter_cap)) return cudaErrorInvalidValue;
    Params p = base_params(d[q]);
    if (!prep_phase<CG, BN>(d[q], p, ks, pl.split_tiles)) return cudaErrorInvalidValue;
    if (ks > 1) {
      const cudaError_t e = cudaMemsetAsync(d[q].counters, 0, (size_t)p.split_tiles * CG * sizeof(unsigned), s);
      if (e != cudaSuccess) return e;
    }
    if (!phase_maps<CG, BN>(d[q], maps + 4 * q)) return cudaErrorInvalidValue;
    ch.ph[q] = p;
    ch.ubase[q + 1] = ch.ubase[q] + phase_units(p);
    ch.waitA_off[q] = -1;
    ch.waitB_off[q] = -1;
  }
  for (int q = nphase; q < 3; ++q) {
    for (int k = 0; k < 4; ++k) maps[4 * q + k] = maps[k];
    ch.waitA_off[q] = ch.waitB_off[q] = -1;
  }
  ch.npre = 0;
  for (int q = 0; q < nphase; ++q)
    for (int k = 0; k < links[q].npre; ++k) {
      if (ch.npre == 2 || (ch.npre && ch.pre_phase != q) || q == 0) return cudaErrorInvalidValue;
      const ChainLink::Pre& a = links[q].pre[k];
      ch.pre[ch.npre++] = Chain::Pre{a.X, a.rows, a.cols, a.ldx, a.hi, a.lo, a.ldo, a.lo_only ? 2 : a.transpose ? 1 : 0};
      ch.pre_phase = q;
    }
  for (int q = 0; q < nphase; ++q) {
    const int a = links[q].waitA, b = links[q].waitB;
    if (a >= 0) {  // this phase's A rows = phase a's output rows, panel by panel (same 256-row tiling)
      if (a >= q || d[a].M != d[q].M) return cudaErrorInvalidValue;
      ch.sig_kind[a] = 1; ch.sig_off[a] = row_off[a];
      ch.waitA_off[q] = row_off[a];
      ch.waitA_target[q] = (d[a].N + BN - 1) / BN;  // every tile of the row panel, per rank
    }
    if (b >= 0) {  // this phase's B rows = phase b's output columns (EPI_SPLIT_T), column panel by panel
      if (b >= q || d[b].N != d[q].N || !((d[b].flags & EPI_SPLIT_T) || ((d[b].flags & EPI_SPLIT_LO) && d[q].b[0].mn)))
        return cudaErrorInvalidValue;
      if (ch.sig_kind[b] == 1) return cudaErrorInvalidValue;
      ch.sig_kind[b] = 2; ch.sig_off[b] = col_off[b];
      ch.waitB_off[q] = col_off[b];
      ch.waitB_target[q] = ((d[b].M + 255) / 256) * CG;  // both ranks of every tile of the column panel
    }
  }
  ch.pre_off = off++;
  if ((size_t)off * sizeof(unsigned) > cnt_cap) return cudaErrorInvalidValue;
  cudaError_t e = cudaMemsetAsync(cnt, 0, (size_t)off * sizeof(unsigned), s);
  if (e != cudaSuccess) return e;
  e = launch_chain_kernel<CG, BN, true>(ch, maps, s, launches);
  if (getenv("PB_TRACE"))
    fprintf(stderr, "[pb] umma chain: %d phases, %lld units, grid %lld\n", nphase, ch.ubase[nphase],
            std::min<long long>(ch.ubase[nphase], num_sms() / CG) * CG);
  return e;
}

cudaError_t launch_umma_gemm(const GemmDesc& d, cudaStream_t s, int* launches) {
  Params p{};
  p.M = d.M;
  p.N = d.N;
  p.K = d.K;
  p.npairs = d.npairs;
  p.nkb = (d.K + BK - 1) / BK;
  p.flags = d.flags;
  p.alpha = d.alpha;
  p.beta = d.beta;
  p.cin = d.cin;
  p.ldc = d.ldc;
  p.out = d.out;
  p.ldo = d.ldo;
  p.out_row0 = d.out_row0;
  p.split_hi = d.split_hi;
  p.split_lo = d.split_lo;
  p.ld_split = d.ld_split;
  const UmmaPlan pl = umma_plan(d);
  int ks = pl.ksplit;
  if (ks > 1 && (d.part == nullptr || d.counters == nullptr)) ks = 1;
  if (pl.streamk && ks == 1) return launch_cg<2, 256>(d, p, 1, 0, s, launches);  // no partials workspace
  if ((d.flags & EPI_PARTIAL) && d.part == nullptr) return cudaErrorInvalidValue;
  // the workspace reserved for partials / counters must hold what this plan writes
  if ((ks > 1 || (d.flags & EPI_PARTIAL)) && (pl.part_bytes > d.part_cap || pl.counter_bytes > d.counter_cap))
    return cudaErrorInvalidValue;
  if (pl.streamk) {
    if (!d.part || !d.counters) return cudaErrorInvalidValue;
    if (pl.cfg == 3) return launch_cg<2, 256>(d, p, ks, pl.split_tiles, s, launches, &pl);
    if (pl.cfg == 2) return launch_cg<2, 128>(d, p, ks, pl.split_tiles, s, launches, &pl);
    return launch_cg<1, 128>(d, p, ks, pl.split_tiles, s, launches, &pl);
  }
  if (pl.cfg == 3) return launch_cg<2, 256>(d, p, ks, pl.split_tiles, s, launches);
  if (pl.cfg == 2) return launch_cg<2, 128>(d, p, ks, pl.split_tiles, s, launches);
  return launch_cg<1, 128>(d, p, ks, pl.split_tiles, s, launches);
}

// Tile configuration and split-K factor: a pure function of the shape (tuned
// for 148 SMs = 74 pairs) so pb_workspace_size can reserve the partials.
//   cfg 3: 2-CTA 256x256 tiles (half the smem reads per MMA flop)
//   cfg 2: 2-CTA 256x128;  cfg 1: 1-CTA 128x128 (under 256 rows / odd band start)
// ksplit in 1..4 maximises wave efficiency x (1 - 3% per extra split), keeping
// >= 8 k-blocks per split.
namespace {
// Plan for a fixed tile configuration (1: 1-CTA 128x128, 2: 2-CTA 256x128, 3: 2-CTA 256x256).
UmmaPlan plan_cfg(const GemmDesc& d, int cfg, int force_ks) {
  UmmaPlan pl;
  pl.cfg = cfg;
  const int pm = cfg == 1 ? 128 : 256, bn = cfg == 3 ? 256 : 128, cg = cfg == 1 ? 1 : 2;
  const int tm0 = d.tm0 * 128 / pm;
  const int tiles_m = (d.M + pm - 1) / pm;
  const int tm1 = d.tm1 < 0 ? tiles_m : std::min(tiles_m, (d.tm1 * 128 + pm - 1) / pm);
  const int tiles_n = (d.N + bn - 1) / bn, ratio = pm / bn;
  long long nt = 0;
  for (int tm = tm0; tm < tm1; ++tm) nt += (d.flags & EPI_TRI) ? std::min(ratio * (tm + 1), tiles_n) : tiles_n;
  pl.tiles = nt;
  const int nkb_total = ((d.K + BK - 1) / BK) * d.npairs;
  const long long units = 148 / cg;
  // Data-parallel + split-K hybrid: whole tiles fill floor(T / units) waves; the
  // R = T mod units remainder tiles are split S ways (S <= units / R, <= 4, and
  // >= 8 k-blocks per split) so the last partial wave is ~full of 1/S-size units.
  long long R = nt < units ? nt : nt % units;
  static const int smax = getenv("PB_KSPLIT_MAX") ? std::max(1, atoi(getenv("PB_KSPLIT_MAX"))) : 4;
  int S = R > 0 ? (int)std::min<long long>(smax, units / R) : 1;
  while (S > 1 && nkb_total / S < 8) --S;
  if (force_ks >= 1 && force_ks <= 8 && nkb_total / force_ks >= 1) { S = force_ks; R = nt; }
  if (S <= 1) { S = 1; R = 0; }
  if (d.flags & EPI_PARTIAL) R = nt;  // every tile through partials (the combine finishes all)
  pl.ksplit = S;
  pl.split_tiles = R;
  pl.part_bytes = R > 0 ? (size_t)R * S * cg * 128 * bn * sizeof(float) : 0;
  pl.counter_bytes = (S > 1 && !(d.flags & EPI_PARTIAL)) ? (size_t)R * cg * sizeof(unsigned) : 0;
  // Stream-K for shapes of at most two partial waves (e.g. a rank's 512 x 4096 x 4096 block
  // of 2mm at 8 GPUs: 32 tiles for 74 SM pairs): every pair gets I / P of the I = tiles x
  // k-blocks iterations, tiles shared by consecutive pairs are summed by the last arriver.
  // Opt-in (PB_STREAMK=1): measured on B200 for 512 x 4096 x 4096 the pairs' MMA time drops
  // from 74.7 to 47.5 us, but the shared tiles' partial exchange (~20 us, latency bound) and
  // the exposed single-wave epilogue make the call slower (153.6 vs 143.6 us).
  static const char* sk_env = getenv("PB_STREAMK");
  const bool sk_on = sk_env && atoi(sk_env) != 0;
  if (sk_on && cfg == 3 && !(d.flags & EPI_PARTIAL) && !force_ks && nt < 2 * units && nt % units != 0 &&
      (long long)nt * nkb_total >= 8 * units) {
    const long long I = nt * (long long)nkb_total, P = units;
    int maxseg = 1;
    for (long long t = 0; t < nt; ++t) {
      const long long lo = ((t * nkb_total + 1) * P - 1) / I, hi = (((t + 1) * nkb_total) * P - 1) / I;
      maxseg = std::max(maxseg, (int)(hi - lo + 1));
    }
    pl.streamk = 1;
    pl.maxseg = maxseg;
    pl.ksplit = maxseg;
    pl.split_tiles = nt;
    pl.part_bytes = (size_t)nt * maxseg * cg * 128 * bn * sizeof(float);
    pl.counter_bytes = (size_t)nt * cg * sizeof(unsigned);
  }
  return pl;
}
}  // namespace

UmmaPlan umma_plan(const GemmDesc& d) {
  static const int force = getenv("PB_UMMA_TILE") ? atoi(getenv("PB_UMMA_TILE")) : 0;
  static const int force_ks = getenv("PB_UMMA_KSPLIT") ? atoi(getenv("PB_UMMA_KSPLIT")) : 0;
  const int rows = d.tm1 < 0 ? d.M : (d.tm1 - d.tm0) * 128;
  const bool pair_ok = rows >= 256 && (d.tm0 % 2) == 0;
  int cfg = pair_ok ? 3 : 1;
  if (force >= 1 && force <= 3 && (force == 1 || pair_ok)) return plan_cfg(d, force, force_ks);
  UmmaPlan pl = plan_cfg(d, cfg, force_ks);
  // Single-wave shapes (fewer 256x256 tiles than SM pairs) that would need split-K:
  // 256x128 tiles without (or with less) split-K win when they still fit in one wave —
  // the split-K exchange and the 256-column epilogue cost more than the lower MMA
  // efficiency of N = 128. Measured: M x 4096 x 4096 at M = 256: 111 vs 123 us,
  // M = 512: 140 vs 147 us; gemm 1024^3: 46 vs 64 us; syrk 1024: 41 vs 67 us,
  // 2048: 68 vs 91 us; syr2k 1024: 50 vs 77 us, 2048: 119 vs 132 us. The Gram
  // (partials + combine) keeps 256x256 tiles (its 256x128 form measured slower).
  if (cfg == 3 && !force_ks && !pl.streamk && pl.ksplit > 1 && pl.tiles < 74 && !(d.flags & EPI_PARTIAL)) {
    const UmmaPlan p2 = plan_cfg(d, 2, 0);
    if (p2.tiles <= 74) pl = p2;
  }
  // Gram (partials + combine) in a single wave: compare wave fill x relative MMA
  // efficiency (1-CTA 128x128 tiles ~0.72 of 2-CTA 256x256 per SM). Measured: cov
  // 1024^2: 128x128 with split-K 4 29 us vs 37 us; at 2048^2 256x256 stays (66 us).
  if (cfg == 3 && !force_ks && (d.flags & EPI_PARTIAL)) {
    const long long u3 = pl.split_tiles * pl.ksplit + (pl.tiles - pl.split_tiles);
    const UmmaPlan p1 = plan_cfg(d, 1, 0);
    const long long u1 = p1.split_tiles * p1.ksplit + (p1.tiles - p1.split_tiles);
    if (u3 <= 74 && u1 <= 148 && 0.72 * (double)u1 / 148.0 > (double)u3 / 74.0) pl = p1;
  }
  return pl;
}

}  // namespace pb
