// k_gram.cu — covariance / correlation in ONE persistent launch (n <= 2048
// observations, m <= 2048 variables): band statistics + centred split, the
// 3xTF32 Gram core on tcgen05, the split-K reduction and the PolyBench epilogue.
//
// Paper mapping: the kernels the paper credits to detect-reduction ("array
// reduction", §VIII: Correlation 5 opportunities, Covariance 4) and
// its future-work kernel fusion (§VII-B: fusing removes launch
// overhead and the global-memory dataflow between kernels). Definitions: the
// PolyBench/C 4.2 kernel_covariance / kernel_correlation statements (readings R4-R6,
// R8, R17, R18 in DESIGN.md).
//
// One cluster of 2 CTAs (an SM pair, tcgen05 cta_group::2) per work unit
// (tile t of the lower triangle of 256 x 256 output tiles, K split ks of S);
// grid = 2 T S <= 148 CTAs, all co-resident, one CTA per SM.
//   phase 0  (every CTA, 8 compute warps): prep units (band b of 256 observations x
//            slab of 128 variables): the raw band tile is TMA-loaded into the (not yet
//            used) smem ring; exact fp64 band means (+ M2 for correlation) per
//            variable (warp-shuffle reductions); the band-centred values are written
//            split (hi/lo) and transposed (X^T, K-major) to the workspace; a release
//            flag per (band, slab) publishes them.
//   phase 1  warp 0: TMA producer — before the k-blocks of band b it acquires the
//            flags of the two slabs it loads (A rows, B rows), so the Gram starts as
//            soon as its own operands exist (no grid-wide barrier);
//            warp 1: tcgen05.mma issuer (3 MMAs per k-step, two TMEM slots, K = 512
//            chunks promoted into fp32 registers — DESIGN.md §6);
//            warps 2..9: epilogue — meanwhile they compute each row / column
//            variable's global mean, between-band deviations and 1/(sqrt(n) sd).
//   phase 2  split-K exchange: the S units of a tile split its 256 columns into S
//            chunks; each unit posts the chunks it does not own to an L2-resident
//            partial buffer (release flag) and sums the chunk it owns in split order
//            (deterministic), adds the between-band scatter (R18), scales
//            (1/(float_n-1), or inv_i inv_j and diag := 1 for correlation) and
//            stores: the direct block through swizzled smem + TMA stores
//            (cp.async.bulk.tensor), the mirrored block with coalesced row stores.
// Flags live in the workspace and are zeroed by a memset node before the launch.
#include <math.h>
#include <stdio.h>
#include <stdlib.h>

#include <algorithm>
#include <vector>

#include "pb_device.cuh"
#include "pb_internal.h"
#include "pb_umma.cuh"

namespace pb {
namespace {

constexpr int GB = 256;              // observations per band (and output tile size)
constexpr int GSLAB = 128;           // variables per prep slab (= rows per CTA)
constexpr int GBK = 32;              // k-block (observations)
constexpr int GTILE = 16 * 1024;     // 128 x 32 fp32 operand tile (= one 128-B swizzled box)
constexpr int GSTAGE = 4 * GTILE;    // A_hi, A_lo, B_hi, B_lo
constexpr int GSTAGES = 3;
constexpr int GCHUNK_KB = 32;        // k-blocks per TMEM slot (K = 1024): a unit (K <= 2048) uses <= 2 slots
constexpr int GMAXB = 8;             // bands (n <= 2048)
constexpr int GNV = 128 + 256;       // row variables + column variables of a CTA's tile part
constexpr int GTHREADS = 64 + 256;   // producer, MMA, 8 epilogue / prep warps
constexpr uint32_t GTMEM = 512;

struct GramArgs {
  int m, n, ldx, nb, nslab, T, S, nkb, corr;
  float alpha;        // covariance: 1 / (float_n - 1)
  float inv_fn;       // 1 / float_n
  float ratm1;        // n / float_n - 1 (0 when float_n == n)
  float inv_sqrt_fn;  // 1 / sqrt(float_n)
  float eps;
  float* hi;
  float* lo;        // X^T split, m x ldx
  float* band_x0;   // [nb][m] shift s_b = x0 + d (two fp32 terms, exact as a pair; phase 0)
  float* band_d;    // [nb][m]
  float* band_m2;   // [nb][m] sum over the band of (x - s_b)^2 (correlation)
  float* part;        // [T][S][2 ranks] x 128 KB: the CTA's accumulator tile in smem box layout
  unsigned* flags;    // [nb * nslab] prep done, then [T][S][2] partial posted
  float* out;
  float* mean_out;
  float* sd_out;
  unsigned long long* ts;  // PB_GRAM_TIMING (tuning only): [cta][16] %globaltimer stamps
};

struct __align__(8) GCtl {
  uint64_t full[GSTAGES];
  uint64_t empty[GSTAGES];
  uint64_t tfull;
  uint64_t xbar;  // partner partials landed
  uint64_t prep[4];
  uint32_t tmem_base;
};

struct GStats {
  float dev[GMAXB][GNV];  // s_b - c per band (e < 128: this CTA's rows; e >= 128: tile columns)
  float inv[GNV];         // 1 / (sqrt(float_n) sd) (correlation), else 1
};

__device__ __forceinline__ unsigned ld_acq(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned ld_rlx(const unsigned* p) {
  unsigned v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_rel(unsigned* p, unsigned v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void wait_flag(const unsigned* p) {
  while (ld_acq(p) == 0u) __nanosleep(32);
}
// Whole warp: lane l polls flag f (nullptr: none) until every lane's flag is set, then
// an acquire fence (relaxed polls + fence.acq_rel = acquire of all of them at once).
__device__ __forceinline__ void warp_wait_flags(const unsigned* f) {
  while (!__all_sync(0xffffffffu, f == nullptr || ld_rlx(f) != 0u)) __nanosleep(64);
  asm volatile("fence.acq_rel.gpu;" ::: "memory");
}
// generic-proxy global writes -> visible to async-proxy (TMA) reads
__device__ __forceinline__ void fence_proxy_global() { asm volatile("fence.proxy.async.global;" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void tma_store_2d(const CUtensorMap* m, const void* src, int c0, int c1) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(
                   reinterpret_cast<uint64_t>(m)),
               "r"(smem_u32(src)), "r"(c0), "r"(c1)
               : "memory");
}
// 1-D bulk copy own smem -> global (bulk group)
__device__ __forceinline__ void bulk_s2g(void* dst, const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(smem_u32(src)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait0() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read0() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
#define GTS(k)                                                                  \
  do {                                                                          \
    if (p.ts) p.ts[(unsigned long long)blockIdx.x * 16 + (k)] = gtimer_ns();    \
  } while (0)
__device__ __forceinline__ void epi_bar() { asm volatile("bar.sync 1, 256;" ::: "memory"); }

// float4 (columns 4g..4g+3 of a 32-column box) of row r in a 128-B swizzled [rows][32] fp32 box
__device__ __forceinline__ float4 ld_sw(const uint8_t* box, int r, int g) {
  return *reinterpret_cast<const float4*>(box + r * 128 + ((g ^ (r & 7)) << 4));
}
__device__ __forceinline__ void st_sw(uint8_t* box, int r, int g, float4 v) {
  *reinterpret_cast<float4*>(box + r * 128 + ((g ^ (r & 7)) << 4)) = v;
}
__device__ __forceinline__ float ld_sw1(const uint8_t* box, int r, int c) {
  return *reinterpret_cast<const float*>(box + r * 128 + ((((c >> 2) ^ (r & 7)) << 4) | ((c & 3) << 2)));
}
// tf32 round-to-nearest, ties away (== cvt.rna.tf32.f32 for finite x) on the integer pipe
__device__ __forceinline__ float rna_tf32_int(float x) {
  return __int_as_float((__float_as_int(x) + 0x1000) & (int)0xFFFFE000);
}

__device__ __forceinline__ float nbw_of(const GramArgs& p, int b) {  // observations in band b (0 past the end)
  return b < p.nb ? (float)min(GB, p.n - GB * b) : 0.f;
}

__device__ __forceinline__ void tile_of(int t, int& tm, int& tn) {
  int r = 0;
  while ((r + 1) * (r + 2) / 2 <= t) ++r;
  tm = r;
  tn = t - r * (r + 1) / 2;
}

template <bool CORR>
__global__ void __launch_bounds__(GTHREADS, 1)
    gram_fused_kernel(const __grid_constant__ CUtensorMap dmap, const __grid_constant__ CUtensorMap ah,
                      const __grid_constant__ CUtensorMap al, const __grid_constant__ CUtensorMap omap,
                      const GramArgs p) {
  extern __shared__ uint8_t smem_raw[];
  // 1024-B aligned (128-B swizzle atoms); indexing the __shared__ array keeps the pointer in
  // the shared address space, so smem loads never look aliased with the global stores
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  GCtl* ctl = reinterpret_cast<GCtl*>(smem + GSTAGES * GSTAGE);
  GStats* st = reinterpret_cast<GStats*>(smem + GSTAGES * GSTAGE + 256);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_rank();
  const bool leader = rank == 0;
  const int unit = blockIdx.x >> 1;
  const int t = unit % p.T, ks = unit / p.T;
  int tm, tn;
  tile_of(t, tm, tn);
  const int arow = tm * GB + (int)rank * GSLAB;  // this CTA's first output row (variable)
  const int brow = tn * GB + (int)rank * GSLAB;  // first B row (variable) this CTA stages

  if (threadIdx.x == 0) {
    for (int s = 0; s < GSTAGES; ++s) {
      mbar_init(&ctl->full[s], 1);
      mbar_init(&ctl->empty[s], 1);
    }
    mbar_init(&ctl->tfull, 1);
    mbar_init(&ctl->xbar, 1);
    for (int q = 0; q < 4; ++q) mbar_init(&ctl->prep[q], 1);
    fence_mbar_init();
  }
  if (warp == 0 && lane == 0) {
    tma_prefetch(&dmap); tma_prefetch(&ah); tma_prefetch(&al); tma_prefetch(&omap);
  }
  if (warp == 1) tmem_alloc_cg<2>(&ctl->tmem_base, GTMEM);
  tc_fence_before();
  cluster_sync_all();
  tc_fence_after();
  pdl_wait();  // data (and the zeroed flags) come from the preceding stream work
  if (threadIdx.x == 0) GTS(0);

  // ============================ phase 0: band shifts + centred split ============================
  // Unit (band b, slab sl). Each column is shifted by s_b = x0 + mean_b(x - x0), x0 its first
  // observation in the band: exact (0) for constant columns, within an fp32 rounding of the
  // band mean otherwise (R18's between-band scatter is taken about these s_b).
  // All arithmetic is fp32 / integer (no fp64 conversions on the per-element path).
  const int nunits0 = p.nb * p.nslab;
  for (int u = blockIdx.x, it = 0; u < nunits0; u += gridDim.x, ++it) {
    const int b = u / p.nslab, sl = u % p.nslab;
    if (warp == 0 && lane == 0) {
      for (int q = 0; q < 4; ++q) {  // always 4 boxes (fully out-of-bounds boxes are zero-filled)
        mbar_arrive_expect_tx(&ctl->prep[q], 32 * GB * 4);
        tma_load_2d(&dmap, &ctl->prep[q], smem + q * 32 * GB * 4, sl * GSLAB + 32 * q, b * GB);
      }
    }
    if (warp >= 2) {
      const int w = warp - 2, q = w >> 1, g0 = (w & 1) * 4;
      const int v0 = sl * GSLAB + 32 * q + 4 * g0;  // this warp's 16 variables v0 .. v0+15
      const int rb = b * GB, nbr = min(GB, p.n - rb);
      const uint8_t* box = smem + q * 32 * GB * 4;
      mbar_wait(&ctl->prep[q], it & 1);
      if (it == 0 && w == 0 && lane == 0) GTS(8);
      float x0[16], s[16];
#pragma unroll
      for (int g = 0; g < 4; ++g) {
        const float4 z = ld_sw(box, 0, g0 + g);
        x0[4 * g] = z.x; x0[4 * g + 1] = z.y; x0[4 * g + 2] = z.z; x0[4 * g + 3] = z.w;
      }
#pragma unroll
      for (int e = 0; e < 16; ++e) s[e] = 0.f;
#pragma unroll
      for (int i = 0; i < GB / 32; ++i) {
        const int r = lane + 32 * i;
        if (r < nbr) {
#pragma unroll
          for (int g = 0; g < 4; ++g) {
            const float4 x = ld_sw(box, r, g0 + g);
            s[4 * g] += x.x - x0[4 * g]; s[4 * g + 1] += x.y - x0[4 * g + 1];
            s[4 * g + 2] += x.z - x0[4 * g + 2]; s[4 * g + 3] += x.w - x0[4 * g + 3];
          }
        }
      }
      if (it == 0 && w == 0 && lane == 0) GTS(12);
#pragma unroll
      for (int e = 0; e < 16; ++e) s[e] = warp_sum(s[e]) / (float)nbr;  // identical in every lane
      if (it == 0 && w == 0 && lane == 0) GTS(13);
#pragma unroll
      for (int e = 0; e < 16; ++e)
        if (lane == e && v0 + e < p.m) {
          p.band_x0[(long long)b * p.m + v0 + e] = x0[e];
          p.band_d[(long long)b * p.m + v0 + e] = s[e];
        }
      float q2[16];
#pragma unroll
      for (int e = 0; e < 16; ++e) q2[e] = 0.f;
      if (it == 0 && w == 0 && lane == 0) GTS(9);
      // y = (x - x0) - mean_b(x - x0); X^T[v][rb + 4 rq .. +3] = split(y): each thread owns 4
      // consecutive observations (two quads rq = lane, lane + 32), so the stores are 16-byte
      // vectors and a warp writes 512 contiguous bytes of an X^T row per instruction
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int r0 = 4 * (lane + 32 * h);
        if (r0 < nbr) {
#pragma unroll
          for (int g = 0; g < 4; ++g) {
            float4 x[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) x[u] = ld_sw(box, r0 + u, g0 + g);
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              const int k = 4 * g + e, v = v0 + k;
              float y[4], hh[4], ll[4];
#pragma unroll
              for (int u = 0; u < 4; ++u) {
                const float xe = e == 0 ? x[u].x : e == 1 ? x[u].y : e == 2 ? x[u].z : x[u].w;
                y[u] = (r0 + u < nbr) ? (xe - x0[k]) - s[k] : 0.f;
                if (CORR) q2[k] = fmaf(y[u], y[u], q2[k]);
                hh[u] = rna_tf32_int(y[u]);
                ll[u] = rna_tf32_int(y[u] - hh[u]);
              }
              if (v < p.m) {
                const long long o = (long long)v * p.ldx + rb + r0;
                __stcg(reinterpret_cast<float4*>(p.hi + o), make_float4(hh[0], hh[1], hh[2], hh[3]));
                __stcg(reinterpret_cast<float4*>(p.lo + o), make_float4(ll[0], ll[1], ll[2], ll[3]));
              }
            }
          }
        }
      }
      if (CORR) {
#pragma unroll
        for (int e = 0; e < 16; ++e) q2[e] = warp_sum(q2[e]);
#pragma unroll
        for (int e = 0; e < 16; ++e)
          if (lane == e && v0 + e < p.m) p.band_m2[(long long)b * p.m + v0 + e] = q2[e];
      }
      if (it == 0 && w == 0 && lane == 0) GTS(10);
      __threadfence();
      fence_proxy_global();
    }
    fence_proxy_smem();  // generic reads of the tile before the next async-proxy (TMA) writes
    __syncthreads();     // every store of this unit issued + fenced; the smem tile is free again
    if (threadIdx.x == 0) st_rel(p.flags + u, 1u);
  }
  if (threadIdx.x == 0) GTS(1);

  // ============================ phase 1: Gram core ============================
  const int kbA = (int)((long long)p.nkb * ks / p.S), kbB = (int)((long long)p.nkb * (ks + 1) / p.S);
  const int nchunks = (kbB - kbA + GCHUNK_KB - 1) / GCHUNK_KB;  // 1 or 2 TMEM slots
  const int slabA = arow / GSLAB, slabB = brow / GSLAB;
  if (warp == 0) {
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      int ready_band = -1;
      for (int kb = kbA; kb < kbB; ++kb) {
        const int b = kb * GBK / GB;
        if (b != ready_band) {  // this band's operand rows published by their prep units
          const unsigned* fa = slabA < p.nslab ? p.flags + b * p.nslab + slabA : nullptr;
          const unsigned* fb = slabB < p.nslab ? p.flags + b * p.nslab + slabB : nullptr;
          while ((fa && ld_rlx(fa) == 0u) || (fb && ld_rlx(fb) == 0u)) __nanosleep(32);
          asm volatile("fence.acq_rel.gpu;" ::: "memory");
          fence_proxy_global();
          if (ready_band < 0) GTS(2);
          ready_band = b;
        }
        mbar_wait(&ctl->empty[stage], phase ^ 1);
        uint8_t* sp = smem + stage * GSTAGE;
        const int k = kb * GBK;
        if (leader) mbar_arrive_expect_tx(&ctl->full[stage], 2 * GSTAGE);
        tma_load_cg<2>(&ah, &ctl->full[stage], sp, k, arow);
        tma_load_cg<2>(&al, &ctl->full[stage], sp + GTILE, k, arow);
        tma_load_cg<2>(&ah, &ctl->full[stage], sp + 2 * GTILE, k, brow);
        tma_load_cg<2>(&al, &ctl->full[stage], sp + 3 * GTILE, k, brow);
        if (++stage == GSTAGES) { stage = 0; phase ^= 1; }
      }
    }
  } else if (warp == 1) {
    // Each K = 1024 chunk accumulates into its own TMEM slot (the tensor-core accumulate
    // truncates: chunks bound the bias); the epilogue adds the slots with
    // round-to-nearest fp32 adds.
    if (leader && lane == 0) {
      constexpr uint32_t idesc = idesc_tf32(256, 256);
      const uint32_t tmem_base = ctl->tmem_base;
      int stage = 0;
      uint32_t phase = 0;
      for (int kb = kbA; kb < kbB; ++kb) {
        const int slot = (kb - kbA) / GCHUNK_KB;
        const uint32_t d = tmem_base + slot * 256;
        mbar_wait(&ctl->full[stage], phase);
        tc_fence_after();
        const uint32_t sa = smem_u32(smem + stage * GSTAGE);
#pragma unroll
        for (int kk = 0; kk < GBK / 8; ++kk) {
          const uint64_t dah = umma_desc_k_sw128(sa + kk * 32);
          const uint64_t dal = umma_desc_k_sw128(sa + GTILE + kk * 32);
          const uint64_t dbh = umma_desc_k_sw128(sa + 2 * GTILE + kk * 32);
          const uint64_t dbl = umma_desc_k_sw128(sa + 3 * GTILE + kk * 32);
          const uint32_t acc = ((kb - kbA) % GCHUNK_KB > 0 || kk > 0) ? 1u : 0u;
          mma_cg<2>(d, dal, dbh, idesc, acc);
          mma_cg<2>(d, dah, dbl, idesc, 1);
          mma_cg<2>(d, dah, dbh, idesc, 1);
        }
        commit_cg<2>(&ctl->empty[stage]);
        if (++stage == GSTAGES) { stage = 0; phase ^= 1; }
      }
      commit_cg<2>(&ctl->tfull);  // every MMA of the unit has completed
    }
  } else {
    // ============================ epilogue warps ============================
    const int et = threadIdx.x - 64;  // 0..255
    const int q = warp & 3, ch = (warp - 2) >> 2;
    const int cbase = ch * 128, row = q * 32 + lane;
    // (a) per-variable statistics of this CTA's rows and the tile's columns (overlaps the MMA)
    if (warp == 2) {  // lane l polls (band l % 8, slab l / 8 of {row slab, 2 column slabs})
      const int b = lane & 7, which = lane >> 3;
      const int slab = which == 0 ? slabA : 2 * tn + which - 1;
      warp_wait_flags((which < 3 && b < p.nb && slab < p.nslab) ? p.flags + b * p.nslab + slab : nullptr);
    }
    epi_bar();
    // fp32 only: e_b = s_b - s_0 and every later difference are small numbers (differences of
    // band shifts), so no catastrophic cancellation against the mean's magnitude; and no fp64
    // while the tensor pipe runs the MMA (measured: fp64 here stalled until the MMA finished).
    for (int e = et; e < GNV; e += 256) {
      const int var = e < 128 ? arow + e : tn * GB + (e - 128);
      const bool in = var < p.m;
      float eb[GMAXB], nbw[GMAXB];
      float x00 = 0.f, d00 = 0.f, M2 = 0.f, se = 0.f;
#pragma unroll
      for (int b = 0; b < GMAXB; ++b) {
        const bool ok = in && b < p.nb;
        const float xb = ok ? __ldcg(p.band_x0 + (long long)b * p.m + var) : 0.f;
        const float db = ok ? __ldcg(p.band_d + (long long)b * p.m + var) : 0.f;
        if (CORR) M2 += ok ? __ldcg(p.band_m2 + (long long)b * p.m + var) : 0.f;
        if (b == 0) { x00 = xb; d00 = db; }
        eb[b] = ok ? (xb - x00) + (db - d00) : 0.f;  // s_b - s_0
        nbw[b] = b < p.nb ? (float)min(GB, p.n - GB * b) : 0.f;
        se = fmaf(nbw[b], eb[b], se);
      }
      // c - s_0 = sum_b n_b (s_b - s_0) / float_n + s_0 (n / float_n - 1)
      const float cz = se * p.inv_fn + (x00 + d00) * p.ratm1;
      float between = 0.f;
#pragma unroll
      for (int b = 0; b < GMAXB; ++b) {
        const float dd = b < p.nb ? eb[b] - cz : 0.f;  // s_b - c
        st->dev[b][e] = dd;
        between = fmaf(nbw[b] * dd, dd, between);
      }
      float inv = 1.f, sd = 0.f;
      if (CORR) {
        sd = sqrtf((M2 + between) * p.inv_fn);
        if (sd <= p.eps) sd = 1.f;
        inv = p.inv_sqrt_fn / sd;
      }
      st->inv[e] = inv;
      if (e >= 128 && in && tm == tn && rank == 0 && ks == 0) {  // column outputs, written once
        if (p.mean_out) p.mean_out[var] = x00 + (d00 + cz);
        if (CORR && p.sd_out) p.sd_out[var] = sd;
      }
    }
    if (et == 0) GTS(6);
    // (b) accumulators (1 or 2 TMEM slots, summed RN) -> the smem tile: 8 boxes of
    // [128 rows][32 columns], 128-B swizzled (the ring is idle once every MMA completed)
    mbar_wait(&ctl->tfull, 0);
    tc_fence_after();
    if (et == 0) GTS(3);
    {
      const uint32_t ta = ctl->tmem_base + ((uint32_t)(q * 32) << 16) + cbase;
#pragma unroll 2
      for (int c0 = 0; c0 < 128; c0 += 16) {
        uint32_t r0[16], r1[16];
        tmem_ld16(ta + c0, r0);
        if (nchunks > 1) tmem_ld16(ta + 256 + c0, r1);
        tmem_wait_ld();
        float v[16];
#pragma unroll
        for (int e = 0; e < 16; ++e) v[e] = __uint_as_float(r0[e]) + (nchunks > 1 ? __uint_as_float(r1[e]) : 0.f);
        const int col = cbase + c0;
        uint8_t* bx = smem + (col >> 5) * GTILE;
#pragma unroll
        for (int qd = 0; qd < 4; ++qd)
          st_sw(bx, row, ((col & 31) >> 2) + qd, make_float4(v[4 * qd], v[4 * qd + 1], v[4 * qd + 2], v[4 * qd + 3]));
      }
    }
    tc_fence_before();
    fence_proxy_smem();
    epi_bar();  // the smem tile (and st->dev / st->inv) complete
    // (c) split-K exchange: chunk c (CW columns = CW / 32 boxes) of the tile is finalised by
    // unit ks == c. The other chunks go to L2 as 1-D bulk copies of whole boxes; the
    // partners' copies of chunk ks come back into the (now free) smem of their chunks.
    const int CW = GB / p.S, CB = CW * 128 * 4;  // chunk width, chunk bytes in smem
    if (p.S > 1) {
      if (warp == 2) {
        uint8_t* mine = reinterpret_cast<uint8_t*>(p.part) + (((long long)t * p.S + ks) * 2 + rank) * (256 * 128 * 4);
        if (lane == 0) {
          for (int c = 0; c < p.S; ++c)
            if (c != ks) bulk_s2g(mine + c * CB, smem + c * CB, CB);
          bulk_commit();
          bulk_wait0();  // writes complete (and the smem of those chunks free)
          fence_proxy_global();
          __threadfence();
          st_rel(p.flags + p.nb * p.nslab + (t * p.S + ks) * 2 + rank, 1u);
        }
        __syncwarp();
        warp_wait_flags(lane < p.S && lane != ks ? p.flags + p.nb * p.nslab + (t * p.S + lane) * 2 + rank : nullptr);
        if (et == 0) GTS(4);
        if (lane == 0) {
          fence_proxy_global();
          mbar_arrive_expect_tx(&ctl->xbar, (uint32_t)(p.S - 1) * CB);
          for (int k = 0; k < p.S; ++k)
            if (k != ks) {
              const uint8_t* theirs =
                  reinterpret_cast<const uint8_t*>(p.part) + (((long long)t * p.S + k) * 2 + rank) * (256 * 128 * 4);
              bulk_g2s(smem + k * CB, theirs + ks * CB, CB, &ctl->xbar);
            }
        }
      }
      mbar_wait(&ctl->xbar, 0);
    }
    // (d) finalise chunk ks with all 8 warps (the tile lives in smem): thread (row, ch) takes
    // half of the chunk's columns. own + partners (ascending k: a fixed order per chunk, so
    // runs are bitwise reproducible), between-band scatter sum_b n_b (s_b - c)_i (s_b - c)_j,
    // normalisation, written back in place; mirror out[j][i] as coalesced row stores (lanes on i)
    const int hw = CW / 2;
    const int f0 = ks * CW + ch * hw, f1 = f0 + hw;  // this thread's columns of the tile
    const bool diag_tile = tm == tn;
    const int i = arow + row;  // output row (variable)
    {
      float er[GMAXB];
#pragma unroll
      for (int b = 0; b < GMAXB; ++b) er[b] = nbw_of(p, b) * st->dev[b][row];
      const float rinv = st->inv[row];
#pragma unroll 2
      for (int col = f0; col < f1; col += 4) {
        const int rc = col - ks * CW;  // column within the chunk
        uint8_t* ob = smem + (col >> 5) * GTILE;
        const int gq = (col & 31) >> 2;
        const float4 own = ld_sw(ob, row, gq);
        float v[4] = {own.x, own.y, own.z, own.w};
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          if (k >= p.S || k == ks) continue;
          const float4 pv = ld_sw(smem + ((k * CW + rc) >> 5) * GTILE, row, gq);
          v[0] += pv.x; v[1] += pv.y; v[2] += pv.z; v[3] += pv.w;
        }
        float bt[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
        for (int b = 0; b < GMAXB; ++b) {
          const float4 f = *reinterpret_cast<const float4*>(&st->dev[b][128 + col]);
          bt[0] = fmaf(er[b], f.x, bt[0]); bt[1] = fmaf(er[b], f.y, bt[1]);
          bt[2] = fmaf(er[b], f.z, bt[2]); bt[3] = fmaf(er[b], f.w, bt[3]);
        }
        const float4 ic = *reinterpret_cast<const float4*>(&st->inv[128 + col]);
        const float icv[4] = {ic.x, ic.y, ic.z, ic.w};
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          v[u] += bt[u];
          v[u] = CORR ? v[u] * (rinv * icv[u]) : v[u] * p.alpha;
        }
        if (CORR && diag_tile) {
#pragma unroll
          for (int u = 0; u < 4; ++u)
            if (tn * GB + col + u == i) v[u] = 1.0f;
        }
        st_sw(ob, row, gq, make_float4(v[0], v[1], v[2], v[3]));  // in place (this thread's row)
        const int j0 = tn * GB + col;
        if (i < p.m) {
#pragma unroll
          for (int u = 0; u < 4; ++u)
            if (j0 + u < i && j0 + u < p.m) __stcg(p.out + (long long)(j0 + u) * p.m + i, v[u]);  // mirror (j < i)
        }
      }
    }
    if (et == 0) GTS(11);
    // (e) direct block out[i][j], j <= i: TMA stores of the chunk's boxes (off-diagonal tiles),
    // or coalesced masked row stores (lanes on j) on diagonal tiles
    fence_proxy_smem();
    epi_bar();
    if (!diag_tile) {
      if (et == 0) {
        for (int bx = (ks * CW) >> 5; bx < ((ks + 1) * CW) >> 5; ++bx)
          tma_store_2d(&omap, smem + bx * GTILE, tn * GB + 32 * bx, arow);
        bulk_commit();
        bulk_wait_read0();
      }
    } else {
      for (int r = et >> 5; r < 128; r += 8) {
        const int ii = arow + r;
        if (ii >= p.m) break;
#pragma unroll 4
        for (int col = ks * CW + lane; col < (ks + 1) * CW; col += 32) {
          const int j = tn * GB + col;
          const float val = ld_sw1(smem + (col >> 5) * GTILE, r, col & 31);
          if (j <= ii && j < p.m) __stcg(p.out + (long long)ii * p.m + j, val);
        }
      }
    }
  }

  if (threadIdx.x == 64) GTS(5);
  pdl_trigger();
  tc_fence_before();
  cluster_sync_all();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc_cg<2>(ctl->tmem_base, GTMEM);
  }
}

struct FusedPlan {
  int T, S, nb, nslab, nkb;
};
FusedPlan fused_plan(int m, int n) {
  FusedPlan f;
  const int tiles = (m + GB - 1) / GB;
  f.T = tiles * (tiles + 1) / 2;
  f.nb = (n + GB - 1) / GB;
  f.nslab = (m + GSLAB - 1) / GSLAB;
  f.nkb = (n + GBK - 1) / GBK;
  const int pairs = num_sms() / 2;
  f.S = 1;
  for (int s : {4, 2})
    if (f.T * s <= pairs && f.nkb / s >= 8) { f.S = s; break; }
  return f;
}

}  // namespace

bool gram_fused_ok(int m, int n) {
  static const char* env = getenv("PB_GRAM_FUSED");
  if (env && atoi(env) == 0) return false;
  if (m > 2048 || n > GMAXB * GB || m < 1 || n < 2) return false;
  const int tiles = (m + GB - 1) / GB;
  return tiles * (tiles + 1) / 2 <= 74 && num_sms() >= 2 * tiles * (tiles + 1) / 2;
}

size_t gram_fused_ws_bytes(int m, int n) {
  const int tiles = (m + GB - 1) / GB, T = tiles * (tiles + 1) / 2;
  const int nb = (n + GB - 1) / GB, nslab = (m + GSLAB - 1) / GSLAB;
  const int ldx = (n + 3) / 4 * 4;
  size_t o = 0;
  auto take = [&](size_t bytes) { o = align_up(o, 256) + bytes; };
  take((size_t)m * ldx * 4);                 // hi
  take((size_t)m * ldx * 4);                 // lo
  take((size_t)nb * m * 4);                  // band_x0
  take((size_t)nb * m * 4);                  // band_d
  take((size_t)nb * m * 4);                  // band_m2
  take((size_t)T * 4 * 2 * 128 * 256 * 4);   // partials (S <= 4)
  take((size_t)(nb * nslab + T * 4 * 2) * 4);  // flags
  return align_up(o, 256);
}

cudaError_t launch_gram_fused(bool corr, int m, int n, double float_n, double eps, const float* data, float* out,
                              float* mean, float* sd, void* ws, cudaStream_t s, int* launches) {
  const FusedPlan f = fused_plan(m, n);
  GramArgs a{};
  a.m = m; a.n = n; a.ldx = (n + 3) / 4 * 4; a.nb = f.nb; a.nslab = f.nslab; a.T = f.T; a.S = f.S; a.nkb = f.nkb;
  a.corr = corr ? 1 : 0;
  a.alpha = (float)(1.0 / (float_n - 1.0));
  a.inv_fn = (float)(1.0 / float_n);
  a.ratm1 = (float)((double)n / float_n - 1.0);
  a.inv_sqrt_fn = (float)(1.0 / sqrt(float_n));
  a.eps = (float)eps;
  char* base = static_cast<char*>(ws);
  size_t o = 0;
  auto take = [&](size_t bytes) { o = align_up(o, 256); char* r = base + o; o += bytes; return r; };
  const int tiles = (m + GB - 1) / GB, Tmax = tiles * (tiles + 1) / 2;
  a.hi = reinterpret_cast<float*>(take((size_t)m * a.ldx * 4));
  a.lo = reinterpret_cast<float*>(take((size_t)m * a.ldx * 4));
  a.band_x0 = reinterpret_cast<float*>(take((size_t)f.nb * m * 4));
  a.band_d = reinterpret_cast<float*>(take((size_t)f.nb * m * 4));
  a.band_m2 = reinterpret_cast<float*>(take((size_t)f.nb * m * 4));
  a.part = reinterpret_cast<float*>(take((size_t)Tmax * 4 * 2 * 128 * 256 * 4));
  const size_t nflags = (size_t)(f.nb * f.nslab + f.T * f.S * 2);
  a.flags = reinterpret_cast<unsigned*>(take((size_t)(f.nb * f.nslab + Tmax * 4 * 2) * 4));
  a.out = out; a.mean_out = mean; a.sd_out = sd;
  static const bool timing = getenv("PB_GRAM_TIMING") != nullptr;
  static unsigned long long* tbuf = nullptr;
  cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
  if (timing) cudaStreamIsCapturing(s, &cap);
  const bool tm_on = timing && cap == cudaStreamCaptureStatusNone;
  if (tm_on && !tbuf) cudaMalloc(&tbuf, 148 * 16 * sizeof(unsigned long long));  // tuning only
  if (tm_on) cudaMemsetAsync(tbuf, 0, 148 * 16 * sizeof(unsigned long long), s);
  a.ts = tm_on ? tbuf : nullptr;
  CUtensorMap dmap, ah, al, omap;
  if (!make_map2d(&dmap, data, m, n, m, 32, GB, true) || !make_map(&ah, a.hi, m, n, a.ldx, GSLAB) ||
      !make_map(&al, a.lo, m, n, a.ldx, GSLAB) || !make_map2d(&omap, out, m, m, m, 32, 128, true))
    return cudaErrorInvalidValue;
  cudaError_t e = cudaMemsetAsync(a.flags, 0, nflags * 4, s);
  if (e != cudaSuccess) return e;
  const size_t smem = 1024 + GSTAGES * GSTAGE + 256 + sizeof(GStats);
  e = corr ? ensure_smem<gram_fused_kernel<true>>(smem) : ensure_smem<gram_fused_kernel<false>>(smem);
  if (e != cudaSuccess) return e;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(2 * f.T * f.S));
  cfg.blockDim = dim3(GTHREADS);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = 2; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
  at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 2;
  e = corr ? cudaLaunchKernelEx(&cfg, gram_fused_kernel<true>, dmap, ah, al, omap, a)
           : cudaLaunchKernelEx(&cfg, gram_fused_kernel<false>, dmap, ah, al, omap, a);
  if (launches) ++*launches;
  if (tm_on) {  // per-phase stamps: min / median / max over CTAs, us after the first entry
    std::vector<unsigned long long> h(148 * 16);
    cudaStreamSynchronize(s);
    cudaMemcpy(h.data(), tbuf, h.size() * 8, cudaMemcpyDeviceToHost);
    const int G = 2 * f.T * f.S;
    unsigned long long t0 = ~0ull;
    for (int c = 0; c < G; ++c) if (h[c * 16]) t0 = std::min(t0, h[c * 16]);
    const char* names[14] = {"entry", "prep done", "first band ready", "MMA done", "partials ready", "end",
                             "stats ready", "-", "prep box landed", "prep shifts", "prep stores", "finalised",
                             "prep sums", "prep reduced"};
    for (int k = 0; k < 14; ++k) {
      std::vector<double> v;
      for (int c = 0; c < G; ++c) if (h[c * 16 + k]) v.push_back((h[c * 16 + k] - t0) / 1e3);
      if (v.empty()) continue;
      std::sort(v.begin(), v.end());
      fprintf(stderr, "[pb gram timing] %-16s min %7.1f  med %7.1f  max %7.1f us (n=%zu)\n", names[k], v.front(),
              v[v.size() / 2], v.back(), v.size());
    }
  }
  if (getenv("PB_TRACE"))
    fprintf(stderr, "[pb] gram_fused<%d> m=%d n=%d tiles=%d S=%d grid=%d\n", corr ? 1 : 0, m, n, f.T, f.S,
            2 * f.T * f.S);
  return e != cudaSuccess ? e : cudaGetLastError();
}

}  // namespace pb
