// k_gram.cu — covariance / correlation in ONE persistent launch (n <= 2048
// observations, m <= 2048 variables): band statistics, the 3xTF32 Gram core on
// tcgen05 with the centring shift and hi/lo split done on load, the split-K
// reduction and the PolyBench epilogue.
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
//   phase 0  (8 converter / epilogue warps): band statistics only — unit (band b of 256
//            observations, slab of 128 variables): x0 = the band's first observation,
//            d = mean_b(x - x0) and (correlation) M2 = sum_b((x - x0) - d)^2, read
//            straight from `data` (coalesced rows, no staging); a release flag per unit.
//   phase 1  warp 0 (every CTA): TMA producer — raw [32 observations][32 variables] boxes
//            of `data` itself (MN-major operand tiles, 128-B swizzle; no split copy of
//            the data exists anywhere) into a 3-stage ring, from the first cycle on;
//            warps 2..9: converters — per stage, y = (x - x0_b) - d_b (the band shift of
//            R18), hi = rna_tf32(y) written in place, lo = rna_tf32(y - hi) into the
//            stage's lo tile; one arrive per warp on the leader's `conv` barrier;
//            warp 1 (leader CTA): tcgen05.mma issuer, 3 MMAs per k-step (MN-major
//            descriptors), K = 1024 chunks in separate TMEM slots.
//   phase 2  the converters compute each row / column variable's global mean,
//            between-band deviations and 1/(sqrt(float_n) sd) while the MMA drains; then
//            split-K exchange: the non-owned column chunks go to L2 as 1-D bulk copies,
//            the partners' copies of the owned chunk come back into smem; finalise (sum in
//            split order, between-band scatter (R18), 1/(float_n-1) or inv_i inv_j and
//            diag := 1) into swizzled smem boxes for the direct block and, transposed, for
//            the mirrored block; both leave as TMA tensor stores (cp.async.bulk.tensor).
// Flags live in the workspace and are zeroed by a one-CTA kernel that lets this one launch early (PDL).
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
constexpr int GBOX = GBK * 32 * 4;   // [32 observations][32 variables] fp32 box, 4 KB
constexpr int GTILE = 4 * GBOX;      // 128 variables x 32 observations, MN-major: one 3-D TMA box
constexpr int GSTAGE = 4 * GTILE;    // A_hi, A_lo, B_hi, B_lo: 64 KB
constexpr int GSTAGES = 3;
constexpr int GRING = GSTAGES * GSTAGE;  // 192 KB (reused by the epilogue)
constexpr int GZ = 16 * 1024;        // scatter rows: {A, B} x {hi, lo} x 4 groups x [8 bands][32 variables]
constexpr int GEBOX = 128 * 32 * 4;  // epilogue box: [128 rows][32 columns], 16 KB
constexpr int GMBOX = 32 * 32 * 4;   // epilogue mirror box: [32 rows j][32 columns i], 4 KB
constexpr int GCHUNK_KB = 1024 / GBK;  // k-blocks per TMEM slot (K = 1024): a unit (K <= 2048) uses <= 2 slots
constexpr int GMAXB = 8;             // bands (n <= 2048)
constexpr int GNV = 128 + 256;       // row variables + column variables of a CTA's tile part
constexpr int GTHREADS = 64 + 256;   // producer, MMA, 8 converter / epilogue warps
constexpr uint32_t GTMEM = 512;

struct GramArgs {
  const float* data;
  int m, n, nb, nslab, T, S, nkb, corr;
  float alpha;        // covariance: 1 / (float_n - 1)
  float inv_fn;       // 1 / float_n
  float ratm1;        // n / float_n - 1 (0 when float_n == n)
  float inv_sqrt_fn;  // 1 / sqrt(float_n)
  float eps;
  float fn;           // float_n
  int xbulk;          // split-K partner values by bulk copy into smem (PB_GRAM_XBULK, default 1)
  uint32_t lbo, sbo;  // MN-major UMMA descriptor strides (bytes)
  int mp;             // row pitch of xh / xl (floats, m rounded up to 32)
  float* xh;          // n x mp: hi of the band-shifted data y = (x - x0_b) - d_b (row-major, like data)
  float* xl;          // n x mp: lo = rna(y - hi)
  float* band_x0;     // [nb][m] band shift s_b = x0 + d (two fp32 terms; phase 0)
  float* band_d;      // [nb][m]
  float* band_m2;     // [nb][m] sum over the band of ((x - x0) - d)^2 (correlation)
  float* part;        // [T][S][2 ranks] x 128 KB: posted column chunks, smem box layout
  unsigned* flags;    // [nb * nslab] band statistics (1: shift, 2: + M2), then [T][S][2] partial posted
  float* out;
  float* mean_out;
  float* sd_out;
  unsigned long long* ts;  // PB_GRAM_TIMING (tuning only): [cta][16] %globaltimer stamps
};

struct __align__(8) GCtl {
  uint64_t full[GSTAGES];   // leader: both CTAs' operand boxes landed (cta_group::2 TMA)
  uint64_t empty[GSTAGES];  // the MMAs reading the stage completed (multicast commit)
  uint64_t tfull;
  uint64_t zbar;  // leader: both CTAs' scatter rows written (last K split only)
  uint64_t xbar;  // partner partials landed
  uint32_t tmem_base;
};

struct GStats {
  float inv[GNV];         // 1 / (sqrt(float_n) sd) (correlation), else 1 (e < 128: rows; else tile columns)
  float red[2 * 8 * 8 * 4];  // phase-0 reduction scratch
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
// Whole warp: lane l polls flag f (nullptr: none) until every lane's flag is >= want, then
// an acquire fence (relaxed polls + fence.acq_rel = acquire of all of them at once).
__device__ __forceinline__ void warp_wait_flags(const unsigned* f, unsigned want) {
  while (!__all_sync(0xffffffffu, f == nullptr || ld_rlx(f) >= want)) __nanosleep(64);
  asm volatile("fence.acq_rel.gpu;" ::: "memory");
}
// generic-proxy global writes -> visible to async-proxy (TMA) reads
__device__ __forceinline__ void fence_proxy_global() { asm volatile("fence.proxy.async.global;" ::: "memory"); }
// 3-D tiled load, cta_group::2: completion counted on the LEADER CTA's barrier
__device__ __forceinline__ void tma_load_3d_cg2(const CUtensorMap* m, uint64_t* bar, void* dst, int c0, int c1, int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, "
      "%5}], [%2];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(smem_u32(bar) & 0xFEFFFFFFu), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}
// 1-D bulk copy own smem -> global (bulk group)
__device__ __forceinline__ void bulk_s2g(void* dst, const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(smem_u32(src)),
               "r"(bytes)
               : "memory");
}
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
__device__ __forceinline__ void st_sw1(uint8_t* box, int r, int c, float v) {
  *reinterpret_cast<float*>(box + r * 128 + ((((c >> 2) ^ (r & 7)) << 4) | ((c & 3) << 2))) = v;
}
// tf32 round-to-nearest, ties away (== cvt.rna.tf32.f32 for finite x) on the integer pipe
__device__ __forceinline__ float rna_tf32_int(float x) {
  return __int_as_float((__float_as_int(x) + 0x1000) & (int)0xFFFFE000);
}
__device__ __forceinline__ float4 f4sub(float4 a, float4 b) { return make_float4(a.x - b.x, a.y - b.y, a.z - b.z, a.w - b.w); }
__device__ __forceinline__ float4 f4add(float4 a, float4 b) { return make_float4(a.x + b.x, a.y + b.y, a.z + b.z, a.w + b.w); }

// byte offset of 16-B chunk c (0..7) of row r in that layout
__device__ __forceinline__ uint32_t sw32_off(int r, int c) {
  return (uint32_t)(r * 128 + (((((c >> 1) ^ (r & 3)) << 1) | (c & 1)) << 4));
}


__device__ __forceinline__ void tile_of(int t, int& tm, int& tn) {
  int r = 0;
  while ((r + 1) * (r + 2) / 2 <= t) ++r;
  tm = r;
  tn = t - r * (r + 1) / 2;
}

// Zeroes the fused kernel's flags. It lets its dependent (the fused kernel, launched with
// programmatic stream serialization) start right away: the fused kernel's prologue (TMEM
// allocation, barrier setup) overlaps this, and its griddepcontrol.wait returns once these
// stores are complete and visible. Replaces a memset node (which cannot trigger early).
__global__ void __launch_bounds__(256) gram_zero_flags(unsigned* flags, int n) {
  pdl_trigger();
  for (int k = threadIdx.x; k < n; k += blockDim.x) flags[k] = 0u;
}

template <bool CORR>
__global__ void __launch_bounds__(GTHREADS, 1)
    gram_fused_kernel(const __grid_constant__ CUtensorMap hmap, const __grid_constant__ CUtensorMap lmap,
                      const __grid_constant__ CUtensorMap omap, const __grid_constant__ CUtensorMap mmap,
                      const GramArgs p) {
  extern __shared__ uint8_t smem_raw[];
  // 1024-B aligned (128-B swizzle atoms); indexing the __shared__ array keeps the pointer in
  // the shared address space, so smem loads never look aliased with the global stores
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* const zb = smem + GRING;  // scatter rows (MN-major, 1024-B aligned)
  GCtl* ctl = reinterpret_cast<GCtl*>(smem + GRING + GZ);
  GStats* st = reinterpret_cast<GStats*>(smem + GRING + GZ + 256);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_rank();
  const bool leader = rank == 0;
  const int unit = blockIdx.x >> 1;
  const int t = unit % p.T, ks = unit / p.T;
  const bool zlast = ks == p.S - 1;  // this unit adds the between-band scatter
  int tm, tn;
  tile_of(t, tm, tn);
  const int arow = tm * GB + (int)rank * GSLAB;  // this CTA's first output row (variable)
  const int brow = tn * GB + (int)rank * GSLAB;  // first B row (variable) this CTA stages
  const int slabA = arow / GSLAB, slabB = brow / GSLAB;
  const int kbA = (int)((long long)p.nkb * ks / p.S), kbB = (int)((long long)p.nkb * (ks + 1) / p.S);
  const int nchunks = (kbB - kbA + GCHUNK_KB - 1) / GCHUNK_KB;  // 1 or 2 TMEM slots

  if (threadIdx.x == 0) {
    for (int s = 0; s < GSTAGES; ++s) {
      mbar_init(&ctl->full[s], 1);
      mbar_init(&ctl->empty[s], 1);
    }
    mbar_init(&ctl->tfull, 1);
    mbar_init(&ctl->zbar, 2);
    mbar_init(&ctl->xbar, 1);
    fence_mbar_init();
  }
  if (warp == 0 && lane == 0) {
    tma_prefetch(&hmap); tma_prefetch(&lmap); tma_prefetch(&omap); tma_prefetch(&mmap);
  }
  if (warp == 1) tmem_alloc_cg<2>(&ctl->tmem_base, GTMEM);
  tc_fence_before();
  // Cluster barrier split in arrive / wait: the producer and MMA warps wait here (barriers
  // and TMEM of both CTAs ready); the epilogue warps start phase 0 at once (it touches no
  // mbarrier, no TMEM and nothing of the peer CTA) and wait before phase 2.
  asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
  if (warp < 2) {
    asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
    tc_fence_after();
  }
  pdl_wait();  // data (and the zeroed flags) come from the preceding stream work
  const int slabA_ok = slabA < p.nslab, slabB_ok = slabB < p.nslab;
  if (threadIdx.x == 0) {
    GTS(0);
    if (p.ts) p.ts[(unsigned long long)blockIdx.x * 16 + 14] = clock64();
  }

  if (warp == 0) {
    // ============================ TMA producer (both CTAs) ============================
    // Before the k-blocks of band b: acquire the phase-0 flags of the 8 variable groups this
    // CTA loads (4 of its A rows, 4 of its B half), so the Gram starts as soon as its own
    // operands exist.
    {
      const int ng = p.mp / 32;
      int stage = 0;
      uint32_t phase = 0;
      int ready = -1;
      for (int kb = kbA; kb < kbB; ++kb) {
        const int b = kb * GBK / GB;
        if (b != ready) {
          const int g = lane < 4 ? arow / 32 + lane : brow / 32 + (lane - 4);
          warp_wait_flags(lane < 8 && g < ng ? p.flags + b * ng + g : nullptr, 1u);
          fence_proxy_global();
          if (ready < 0 && lane == 0) GTS(2);
          ready = b;
        }
        if (lane == 0) {
          mbar_wait(&ctl->empty[stage], phase ^ 1);
          uint8_t* sp = smem + stage * GSTAGE;
          const int k = kb * GBK;
          if (leader) mbar_arrive_expect_tx(&ctl->full[stage], 2 * GSTAGE);
          tma_load_3d_cg2(&hmap, &ctl->full[stage], sp, 0, k, arow / 32);
          tma_load_3d_cg2(&lmap, &ctl->full[stage], sp + GTILE, 0, k, arow / 32);
          tma_load_3d_cg2(&hmap, &ctl->full[stage], sp + 2 * GTILE, 0, k, brow / 32);
          tma_load_3d_cg2(&lmap, &ctl->full[stage], sp + 3 * GTILE, 0, k, brow / 32);
        }
        __syncwarp();
        if (++stage == GSTAGES) { stage = 0; phase ^= 1; }
      }
    }
  } else if (warp == 1) {
    // ============================ MMA issuer (leader CTA) ============================
    // Each K = 1024 chunk accumulates into its own TMEM slot (the tensor-core accumulate
    // truncates: chunks bound the bias); the epilogue adds the slots with
    // round-to-nearest fp32 adds.
    if (leader && lane == 0) {
      constexpr uint32_t idesc = idesc_tf32(256, 256) | (1u << 15) | (1u << 16);  // A, B MN-major
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
          const uint64_t dah = umma_desc_mn_sw128b32(sa + kk * 1024, p.lbo, p.sbo);
          const uint64_t dal = umma_desc_mn_sw128b32(sa + GTILE + kk * 1024, p.lbo, p.sbo);
          const uint64_t dbh = umma_desc_mn_sw128b32(sa + 2 * GTILE + kk * 1024, p.lbo, p.sbo);
          const uint64_t dbl = umma_desc_mn_sw128b32(sa + 3 * GTILE + kk * 1024, p.lbo, p.sbo);
          const uint32_t acc = ((kb - kbA) % GCHUNK_KB > 0 || kk > 0) ? 1u : 0u;
          mma_cg<2>(d, dal, dbh, idesc, acc);
          mma_cg<2>(d, dah, dbl, idesc, 1);
          mma_cg<2>(d, dah, dbh, idesc, 1);
        }
        commit_cg<2>(&ctl->empty[stage]);
        if (++stage == GSTAGES) { stage = 0; phase ^= 1; }
      }
      if (zlast) {
        // between-band scatter sum_b n_b (s_b - c)_i (s_b - c)_j (R18) as 8 more observations
        // z_b = sqrt(n_b) (s_b - c), written by the epilogue warps of both CTAs: one K = 8 step
        mbar_wait_cluster(&ctl->zbar, 0);
        tc_fence_after();
        const uint32_t d = tmem_base + ((kbB - 1 - kbA) / GCHUNK_KB) * 256;
        const uint32_t za = smem_u32(zb);
        const uint64_t dah = umma_desc_mn_sw128b32(za, 1024, 512), dal = umma_desc_mn_sw128b32(za + 4096, 1024, 512);
        const uint64_t dbh = umma_desc_mn_sw128b32(za + 8192, 1024, 512);
        const uint64_t dbl = umma_desc_mn_sw128b32(za + 12288, 1024, 512);
        mma_cg<2>(d, dal, dbh, idesc, 1);
        mma_cg<2>(d, dah, dbl, idesc, 1);
        mma_cg<2>(d, dah, dbh, idesc, 1);
      }
      commit_cg<2>(&ctl->tfull);  // every MMA of the unit has completed
    }
  } else {
    const int et = threadIdx.x - 64;  // 0..255
    // ============================ phase 0: band shift + split ============================
    // Unit (band b, group g of 32 variables), in "first needed" band order (the first band of
    // every K split first, then the second, ...), spread over all CTAs, one release flag per
    // unit: the Gram's producers start as soon as their first band is published, and the
    // later bands are prepared while the MMAs run. Thread (variable quad vq, row group rg)
    // holds rows rg, rg + 32, .. of the band (8 x 16 B loads in flight; a warp reads 4
    // rows x 128 B per load). Shift s_b = x0 + d: x0 the band's first observation,
    // d = mean_b(x - x0) in fp32 (exact for constant columns; R18's between-band scatter is
    // taken about these s_b); y = (x - x0) - d is split hi = rna_tf32(y), lo = rna_tf32(y - hi)
    // and stored row-major like the data (n x mp), zero for padded variables. Sums run in a
    // fixed order (per thread, lanes, then warps ascending): bitwise reproducible.
    {
      const int vq = et & 7, rg = et >> 3;
      float4* red = reinterpret_cast<float4*>(st->red);  // [8 warps][8 quads]
      const int ng = p.mp / 32, bps = (p.nb + p.S - 1) / p.S;
      // unit -> (band b, first row rb, rows nbr, variable v of this thread, column pointer)
      auto unit_at = [&](int u, int& b, int& rb, int& nbr, int& v, const float*& col) {
        const int ord = u / ng, g = u % ng;
        b = 0;  // the ord-th band of the order (split 0's first band, split 1's first band, ...)
        for (int j = 0, cnt = 0; j < bps * p.S; ++j) {
          const int bb = (j % p.S) * bps + j / p.S;
          if (bb < p.nb) {
            if (cnt == ord) { b = bb; break; }
            ++cnt;
          }
        }
        rb = b * GB;
        nbr = min(GB, p.n - rb);
        v = g * 32 + 4 * vq;
        col = p.data + (v < p.m ? v : 0);
      };
      // software pipeline: the next unit's loads are in flight while this unit's stores drain
      float4 xn[GB / 32], x0n = make_float4(0.f, 0.f, 0.f, 0.f);
      auto load_unit = [&](int u) {
        int b, rb, nbr, v;
        const float* col;
        unit_at(u, b, rb, nbr, v, col);
#pragma unroll
        for (int i = 0; i < GB / 32; ++i) {
          const int r = min(rg + 32 * i, nbr - 1);
          xn[i] = __ldg(reinterpret_cast<const float4*>(col + (long long)(rb + r) * p.m));
        }
        x0n = __ldg(reinterpret_cast<const float4*>(col + (long long)rb * p.m));
      };
      if ((int)blockIdx.x < p.nb * ng) load_unit(blockIdx.x);
      for (int u = blockIdx.x; u < p.nb * ng; u += gridDim.x) {
        int b, rb, nbr, v;
        const float* col;
        unit_at(u, b, rb, nbr, v, col);
        const int g = u % ng;
        const bool vin = v < p.m;
        float4 x[GB / 32];
#pragma unroll
        for (int i = 0; i < GB / 32; ++i) x[i] = xn[i];
        const float4 x0 = x0n;
        float4 s = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
        for (int i = 0; i < GB / 32; ++i)
          if (rg + 32 * i < nbr) s = f4add(s, f4sub(x[i], x0));
        if (et == 0 && u == (int)blockIdx.x) GTS(7);
#pragma unroll
        for (int o = 8; o < 32; o <<= 1)
          s = make_float4(s.x + __shfl_xor_sync(0xffffffffu, s.x, o), s.y + __shfl_xor_sync(0xffffffffu, s.y, o),
                          s.z + __shfl_xor_sync(0xffffffffu, s.z, o), s.w + __shfl_xor_sync(0xffffffffu, s.w, o));
        if (lane < 8) red[(warp - 2) * 8 + lane] = s;
        epi_bar();
        float4 d = red[vq];
#pragma unroll
        for (int w = 1; w < 8; ++w) d = f4add(d, red[w * 8 + vq]);
        const float rn = (float)nbr;
        const float rinv_n = 1.0f / rn;  // any shift close to the band mean serves (R18): no IEEE divide per lane
        d = make_float4(d.x * rinv_n, d.y * rinv_n, d.z * rinv_n, d.w * rinv_n);
        if (rg == 0 && vin) {
          *reinterpret_cast<float4*>(p.band_x0 + (long long)b * p.m + v) = x0;
          *reinterpret_cast<float4*>(p.band_d + (long long)b * p.m + v) = d;
        }
        if (et == 0 && u == (int)blockIdx.x) GTS(8);
        float4 q2 = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
        for (int i = 0; i < GB / 32; ++i) {
          const int r = rg + 32 * i;
          if (r < nbr) {
            const float4 y4 = f4sub(f4sub(x[i], x0), d);
            float y[4] = {y4.x, y4.y, y4.z, y4.w}, h[4], l[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              y[e] = vin ? y[e] : 0.f;
              h[e] = rna_tf32_int(y[e]);
              l[e] = rna_tf32_int(y[e] - h[e]);
            }
            if (CORR) {
              q2.x = fmaf(y[0], y[0], q2.x); q2.y = fmaf(y[1], y[1], q2.y);
              q2.z = fmaf(y[2], y[2], q2.z); q2.w = fmaf(y[3], y[3], q2.w);
            }
            const long long o = (long long)(rb + r) * p.mp + v;
            __stcg(reinterpret_cast<float4*>(p.xh + o), make_float4(h[0], h[1], h[2], h[3]));
            __stcg(reinterpret_cast<float4*>(p.xl + o), make_float4(l[0], l[1], l[2], l[3]));
          }
        }
        if (CORR) {  // M2 = sum_b y^2 (y about the band mean: no cancellation)
#pragma unroll
          for (int o = 8; o < 32; o <<= 1)
            q2 = make_float4(q2.x + __shfl_xor_sync(0xffffffffu, q2.x, o), q2.y + __shfl_xor_sync(0xffffffffu, q2.y, o),
                             q2.z + __shfl_xor_sync(0xffffffffu, q2.z, o), q2.w + __shfl_xor_sync(0xffffffffu, q2.w, o));
          epi_bar();  // red[] (shift sums) consumed by everyone
          if (lane < 8) red[(warp - 2) * 8 + lane] = q2;
          epi_bar();
          if (rg == 0) {
            float4 m2 = red[vq];
#pragma unroll
            for (int w = 1; w < 8; ++w) m2 = f4add(m2, red[w * 8 + vq]);
            if (vin) *reinterpret_cast<float4*>(p.band_m2 + (long long)b * p.m + v) = m2;
          }
        }
        if (et == 0 && u == (int)blockIdx.x) GTS(9);
        __threadfence();       // (waits for this unit's stores only: the next unit's loads come after)
        fence_proxy_global();  // generic-proxy stores -> the Gram's TMA (async-proxy) reads
        epi_bar();             // every store of the unit fenced; red[] free again
        if (et == 0) st_rel(p.flags + b * ng + g, 1u);
        if (et == 0 && u == (int)blockIdx.x) GTS(10);
        if (u + (int)gridDim.x < p.nb * ng) load_unit(u + gridDim.x);
      }
    }
    if (et == 0) GTS(1);
    asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");  // (arrived before phase 0)
    tc_fence_after();

    // ============================ phase 2: epilogue ============================
    const int q = warp & 3, ch = (warp - 2) >> 2;
    const int rl = q * 32 + lane;  // this thread's row of the CTA's 128
    const int i = arow + rl;       // output row (variable)
    // (a) per-variable statistics of this CTA's rows and the tile's columns (overlaps the
    // MMAs still in flight). fp32 only: e_b = s_b - s_0 and every later difference are small
    // numbers (differences of band shifts), so no cancellation against the mean's magnitude.
    if (warp == 2) {  // every band's flags of the 4 row groups and 8 column groups of this CTA's part
      const int ng = p.mp / 32;
      for (int f0 = 0; f0 < p.nb * 12; f0 += 32) {  // warp-uniform trip count
        const int f = f0 + lane, b = f / 12, j = f % 12;
        const int g = j < 4 ? arow / 32 + j : tn * (GB / 32) + (j - 4);
        warp_wait_flags(f < p.nb * 12 && g < ng ? p.flags + b * ng + g : nullptr, 1u);
      }
    }
    epi_bar();
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
      // this CTA's A rows and B half: scatter rows z_b = sqrt(n_b) (s_b - c), split, MN-major
      const int vl = e < 128 ? e : e - 128 - (int)rank * 128;
      const bool zw = zlast && (e < 128 || (vl >= 0 && vl < 128));
      uint8_t* zp = zb + (e < 128 ? 0 : 8192) + (vl >> 5) * 1024 + ((vl & 3) << 2);
#pragma unroll
      for (int b = 0; b < GMAXB; ++b) {
        const float dv = b < p.nb ? eb[b] - cz : 0.f;  // s_b - c
        between = fmaf(nbw[b] * dv, dv, between);
        if (zw) {
          const float z = sqrtf(nbw[b]) * dv;
          const float zh = rna_tf32_int(z);
          const uint32_t off = sw32_off(b, (vl & 31) >> 2);
          *reinterpret_cast<float*>(zp + off) = zh;
          *reinterpret_cast<float*>(zp + 4096 + off) = rna_tf32_int(z - zh);
        }
      }
      float inv = 1.f, sd = 0.f;
      if (CORR) {
        sd = sqrtf((M2 + between) * p.inv_fn);
        if (sd <= p.eps) sd = 1.f;
        inv = p.inv_sqrt_fn / sd;
      }
      st->inv[e] = inv;
      if (e >= 128 && in && tm == tn && rank == 0 && ks == 0) {  // column outputs, written once
        // mean = sum_b n_b s_b / float_n, summed from s_0's two terms (no cancellation against
        // (n / float_n - 1) when float_n != n, e.g. PolyBench-GPU's 3214212.01)
        if (p.mean_out) p.mean_out[var] = (se + (float)p.n * x00 + (float)p.n * d00) / p.fn;
        if (CORR && p.sd_out) p.sd_out[var] = sd;
      }
    }
    if (et == 0) GTS(6);
    fence_proxy_smem();  // scatter rows -> the tensor core (async proxy)
    epi_bar();  // st->inv and the scatter rows complete
    if (zlast && et == 0) {
      if (leader) mbar_arrive(&ctl->zbar);
      else mbar_arrive_cluster(map_peer(smem_u32(&ctl->zbar), 0));
    }
    const int CW = GB / p.S, CB = CW * 128 * 4;  // chunk width (columns), chunk bytes in smem
    mbar_wait(&ctl->tfull, 0);
    tc_fence_after();
    if (et == 0) GTS(3);
    const uint32_t ta = ctl->tmem_base + ((uint32_t)(q * 32) << 16);
    // (b) split-K exchange: chunk c (CW columns) of the tile is finalised by unit ks == c.
    // Each thread stores its row's part of the chunks it does not own straight from TMEM to
    // an L2-resident partial tile ([column quad][128 rows] float4: a warp store covers 512
    // contiguous bytes), loads its own chunk part from TMEM into registers, and after the
    // partners' release flags adds their parts (ascending split index: a fixed order, so runs
    // are bitwise reproducible) with coalesced loads. No smem staging, no bulk-copy round trip.
    float acc[64];  // S > 1: this thread's own-chunk values (CW / 2 <= 64 columns), partners added
    if (p.S > 1) {
      const int hw = CW / 2;
      float4* const part4 = reinterpret_cast<float4*>(p.part);
      const long long tile_f4 = 256 * 128 / 4;
      float4* mine = part4 + (((long long)t * p.S + ks) * 2 + rank) * tile_f4;
      for (int cc = 0; cc < p.S; ++cc) {
        if (cc == ks) continue;
        for (int c0 = cc * CW + ch * hw; c0 < cc * CW + ch * hw + hw; c0 += 16) {
          uint32_t r0[16];
          tmem_ld16(ta + c0, r0);
          tmem_wait_ld();
#pragma unroll
          for (int qd = 0; qd < 4; ++qd)
            __stcg(mine + ((c0 >> 2) + qd) * 128 + rl,
                   make_float4(__uint_as_float(r0[4 * qd]), __uint_as_float(r0[4 * qd + 1]),
                               __uint_as_float(r0[4 * qd + 2]), __uint_as_float(r0[4 * qd + 3])));
        }
      }
      const int fo = ks * CW + ch * hw;  // this thread's own columns [fo, fo + hw)
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        if (16 * j < hw) {
          uint32_t r0[16];
          tmem_ld16(ta + fo + 16 * j, r0);
          tmem_wait_ld();
#pragma unroll
          for (int e = 0; e < 16; ++e) acc[16 * j + e] = __uint_as_float(r0[e]);
        }
      }
      __threadfence();
      epi_bar();
      if (et == 0) st_rel(p.flags + p.nb * (p.mp / 32) + (t * p.S + ks) * 2 + rank, 1u);
      if (warp == 2)
        warp_wait_flags(lane < p.S && lane != ks ? p.flags + p.nb * (p.mp / 32) + (t * p.S + lane) * 2 + rank : nullptr,
                        1u);
      epi_bar();
      if (et == 0) GTS(4);
      if (p.xbulk) {
        // the partners' posts of this unit's chunk (S - 1 contiguous [CW / 4 quads][128 rows]
        // float4 runs) come in as bulk copies (TMA engine) into the free ring space behind the
        // direct boxes, then every thread reads its values from shared memory; the sum order
        // (own, then partners in ascending split index) is the same as the direct loads'.
        const uint32_t run = (uint32_t)CW * 128u * 4u;
        float4* xs = reinterpret_cast<float4*>(smem + (CW < 128 ? CW : 128) / 32 * GEBOX);
        if (et == 0) {
          fence_proxy_global();  // the partners' generic-proxy stores -> these async-proxy reads
          mbar_arrive_expect_tx(&ctl->xbar, run * (uint32_t)(p.S - 1));
          for (int k = 0, slot = 0; k < p.S; ++k) {
            if (k == ks) continue;
            const float4* theirs = part4 + (((long long)t * p.S + k) * 2 + rank) * tile_f4 + (ks * CW / 4) * 128;
            bulk_g2s(xs + (size_t)slot * (CW / 4) * 128, theirs, run, &ctl->xbar);
            ++slot;
          }
        }
        mbar_wait(&ctl->xbar, 0);
        for (int k = 0, slot = 0; k < p.S; ++k) {
          if (k == ks) continue;
          const float4* theirs = xs + (size_t)slot * (CW / 4) * 128;
#pragma unroll
          for (int j = 0; j < 16; ++j) {
            if (4 * j < hw) {
              const float4 pv = theirs[((fo - ks * CW) >> 2) * 128 + j * 128 + rl];
              acc[4 * j] += pv.x; acc[4 * j + 1] += pv.y; acc[4 * j + 2] += pv.z; acc[4 * j + 3] += pv.w;
            }
          }
          ++slot;
        }
      } else {
        for (int k = 0; k < p.S; ++k) {
          if (k == ks) continue;
          const float4* theirs = part4 + (((long long)t * p.S + k) * 2 + rank) * tile_f4;
#pragma unroll
          for (int j = 0; j < 16; ++j) {
            if (4 * j < hw) {
              const float4 pv = __ldcg(theirs + ((fo >> 2) + j) * 128 + rl);
              acc[4 * j] += pv.x; acc[4 * j + 1] += pv.y; acc[4 * j + 2] += pv.z; acc[4 * j + 3] += pv.w;
            }
          }
        }
      }
      if (et == 0) GTS(12);
    }
    // (c) finalise chunk ks in sub-chunks of <= 128 columns: thread (row rl, half ch) takes
    // half of each sub-chunk's columns: own (TMEM) + partners (ascending k: a fixed order per
    // chunk, so runs are bitwise reproducible), then 1/(float_n - 1), or inv_i inv_j and
    // diag := 1. The values go to the chunk's own slot (direct boxes) and, transposed, to the
    // mirror boxes at 128 KB; both leave as TMA tensor stores. Relative to the diagonal a
    // sub-chunk (rows R of this CTA, columns C) is: below (max C < min R, every off-diagonal
    // tile): direct + mirror; symmetric (C == R): its upper triangle is overwritten with the
    // transposed lower one in smem, then stored once (PolyBench's cov[j][i] = cov[i][j]
    // bitwise); above (min C > max R): written by the block that mirrors into it, skipped;
    // mixed (S = 4 only): masked element stores.
    const float rinv = st->inv[rl];
    const int SW = min(CW, 128);
    uint8_t* mir = smem + 2 * 64 * 1024;  // [SW/32 j-boxes][4 i-boxes] of [32 j][32 i]
    for (int col0 = ks * CW; col0 < (ks + 1) * CW; col0 += SW) {
      const int r0c = (int)rank * GSLAB;  // this CTA's rows within the tile
      const int kind = tm != tn || col0 + SW <= r0c ? 0 : col0 >= r0c + GSLAB ? 3 : (col0 == r0c && SW == GSLAB) ? 1 : 2;
      if (kind == 3) continue;  // above the diagonal: another block's mirror covers it
      const int hw = SW / 2, f0 = col0 + ch * hw;
#pragma unroll
      for (int jj = 0; jj < 4; ++jj) {
        const int c0 = f0 + 16 * jj;
        if (16 * jj >= hw) break;
        float vals[16];
        if (p.S > 1) {
#pragma unroll
          for (int e = 0; e < 16; ++e) vals[e] = acc[16 * jj + e];
        } else {
          uint32_t r0[16], r1[16];
          tmem_ld16(ta + c0, r0);
          if (nchunks > 1) tmem_ld16(ta + 256 + c0, r1);
          tmem_wait_ld();
#pragma unroll
          for (int e = 0; e < 16; ++e) vals[e] = __uint_as_float(r0[e]) + (nchunks > 1 ? __uint_as_float(r1[e]) : 0.f);
        }
#pragma unroll
        for (int qd = 0; qd < 4; ++qd) {
          const int col = c0 + 4 * qd;
          const int gq = (col & 31) >> 2;
          float v[4] = {vals[4 * qd], vals[4 * qd + 1], vals[4 * qd + 2], vals[4 * qd + 3]};
          const float4 ic = *reinterpret_cast<const float4*>(&st->inv[128 + col]);
          const float icv[4] = {ic.x, ic.y, ic.z, ic.w};
#pragma unroll
          for (int u = 0; u < 4; ++u) v[u] = CORR ? v[u] * (rinv * icv[u]) : v[u] * p.alpha;
          if (CORR && kind != 0) {
#pragma unroll
            for (int u = 0; u < 4; ++u)
              if (tn * GB + col + u == i) v[u] = 1.0f;
          }
          st_sw(smem + (col >> 5) * GEBOX, rl, gq, make_float4(v[0], v[1], v[2], v[3]));  // direct (own slot)
          if (kind == 0) {
            const int jl = col - col0;  // mirror: element (j, i) at box (jl / 32, q), row j % 32, column lane
            uint8_t* mb = mir + ((jl >> 5) * 4 + q) * GMBOX;
#pragma unroll
            for (int u = 0; u < 4; ++u) st_sw1(mb, (jl + u) & 31, lane, v[u]);
          } else if (kind == 2) {
            const int j0 = tn * GB + col;
            if (i < p.m) {
#pragma unroll
              for (int u = 0; u < 4; ++u)
                if (j0 + u < i && j0 + u < p.m) __stcg(p.out + (long long)(j0 + u) * p.m + i, v[u]);  // mirror
            }
          }
        }
      }
      if (et == 0 && col0 == ks * CW) GTS(11);
      if (kind == 1) {  // upper triangle := transposed lower triangle (element (a, b), b > a, takes (b, a))
        epi_bar();
        for (int bcol = ch * 64; bcol < ch * 64 + 64; ++bcol) {
          if (bcol > rl) {
            const float t = ld_sw1(smem + ((col0 + rl) >> 5) * GEBOX, bcol, (col0 + rl) & 31);
            st_sw1(smem + ((col0 + bcol) >> 5) * GEBOX, rl, (col0 + bcol) & 31, t);
          }
        }
      }
      fence_proxy_smem();
      epi_bar();
      if (kind != 2) {
        if (et == 0) {
          for (int bx = col0 >> 5; bx < (col0 + SW) >> 5; ++bx) tma_store_2d(&omap, smem + bx * GEBOX, tn * GB + 32 * bx, arow);
          if (kind == 0)
            for (int jb = 0; jb < SW / 32; ++jb)
              for (int ib = 0; ib < 4; ++ib)
                tma_store_2d(&mmap, mir + (jb * 4 + ib) * GMBOX, arow + 32 * ib, tn * GB + col0 + 32 * jb);
          bulk_commit();
          bulk_wait_read0();
        }
        epi_bar();  // the mirror boxes are free for the next sub-chunk
      } else {
        for (int r = et >> 5; r < 128; r += 8) {
          const int ii = arow + r;
          if (ii >= p.m) break;
          for (int col = col0 + lane; col < col0 + SW; col += 32) {
            const int j = tn * GB + col;
            const float val = ld_sw1(smem + (col >> 5) * GEBOX, r, col & 31);
            if (j <= ii && j < p.m) __stcg(p.out + (long long)ii * p.m + j, val);
          }
        }
      }
    }
  }

  if (threadIdx.x == 64) {
    GTS(5);
    if (p.ts) p.ts[(unsigned long long)blockIdx.x * 16 + 15] = clock64();
  }
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

size_t gram_smem_bytes() { return 1024 + GRING + GZ + 256 + sizeof(GStats); }

// The kernel's flags need every CTA of the grid resident at once: the launch is only
// taken when the device can hold T * S clusters of 2 CTAs with this footprint.
int gram_max_clusters() {
  static std::atomic<int> cache[64];
  int dev = 0;
  cudaGetDevice(&dev);
  int v = cache[dev & 63].load(std::memory_order_relaxed);
  if (v) return v;
  const size_t smem = gram_smem_bytes();
  if (ensure_smem<gram_fused_kernel<true>>(smem) != cudaSuccess ||
      ensure_smem<gram_fused_kernel<false>>(smem) != cudaSuccess)
    return -1;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(2 * 74);
  cfg.blockDim = dim3(GTHREADS);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = 2; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  int n1 = 0, n2 = 0;
  if (cudaOccupancyMaxActiveClusters(&n1, gram_fused_kernel<true>, &cfg) != cudaSuccess ||
      cudaOccupancyMaxActiveClusters(&n2, gram_fused_kernel<false>, &cfg) != cudaSuccess) {
    cudaGetLastError();
    return -1;
  }
  v = std::max(1, std::min(n1, n2));
  cache[dev & 63].store(v, std::memory_order_relaxed);
  if (getenv("PB_TRACE")) {  // tuning aid: how many 4-CTA clusters of this footprint fit
    at[0].val.clusterDim.x = 4;
    cfg.gridDim = dim3(4 * 36);
    int n4 = 0;
    cudaOccupancyMaxActiveClusters(&n4, gram_fused_kernel<false>, &cfg);
    cudaGetLastError();
    fprintf(stderr, "[pb] gram: max active clusters: %d of 2 CTAs, %d of 4 CTAs (smem %zu)\n", v, n4, smem);
  }
  return v;
}

}  // namespace

bool gram_fused_ok(int m, int n) {
  static const char* env = getenv("PB_GRAM_FUSED");
  if (env && atoi(env) == 0) return false;
  if (m > 2048 || n > GMAXB * GB || m < 1 || n < 2) return false;
  const FusedPlan f = fused_plan(m, n);
  return f.T * f.S <= gram_max_clusters();
}

size_t gram_fused_ws_bytes(int m, int n) {
  const int tiles = (m + GB - 1) / GB, T = tiles * (tiles + 1) / 2;
  const int nb = (n + GB - 1) / GB, nslab = (m + GSLAB - 1) / GSLAB;
  const size_t mp = (m + 31) / 32 * 32;
  size_t o = 0;
  auto take = [&](size_t bytes) { o = align_up(o, 256) + bytes; };
  take((size_t)n * mp * 4);                  // xh
  take((size_t)n * mp * 4);                  // xl
  take((size_t)nb * m * 4);                  // band_x0
  take((size_t)nb * m * 4);                  // band_d
  take((size_t)nb * m * 4);                  // band_m2
  take((size_t)T * 4 * 2 * 128 * 256 * 4);   // posted chunks (S <= 4)
  take((size_t)(nb * (mp / 32) + T * 4 * 2) * 4);  // flags
  return align_up(o, 256);
}

cudaError_t launch_gram_fused(bool corr, int m, int n, double float_n, double eps, const float* data, float* out,
                              float* mean, float* sd, void* ws, cudaStream_t s, int* launches) {
  const FusedPlan f = fused_plan(m, n);
  GramArgs a{};
  a.data = data;
  a.m = m; a.n = n; a.nb = f.nb; a.nslab = f.nslab; a.T = f.T; a.S = f.S; a.nkb = f.nkb;
  a.corr = corr ? 1 : 0;
  a.alpha = (float)(1.0 / (float_n - 1.0));
  a.inv_fn = (float)(1.0 / float_n);
  a.ratm1 = (float)((double)n / float_n - 1.0);
  a.inv_sqrt_fn = (float)(1.0 / sqrt(float_n));
  a.eps = (float)eps;
  a.fn = (float)float_n;
  static const int xbulk = getenv("PB_GRAM_XBULK") ? atoi(getenv("PB_GRAM_XBULK")) : 1;
  a.xbulk = xbulk != 0;
  // MN-major operand boxes: 32-variable runs GBOX apart, 4-observation groups 512 B apart
  static const bool swap = getenv("PB_GRAM_MNSWAP") != nullptr;  // tuning / bring-up only
  a.lbo = swap ? 512u : (uint32_t)GBOX;
  a.sbo = swap ? (uint32_t)GBOX : 512u;
  char* base = static_cast<char*>(ws);
  size_t o = 0;
  auto take = [&](size_t bytes) { o = align_up(o, 256); char* r = base + o; o += bytes; return r; };
  const int tiles = (m + GB - 1) / GB, Tmax = tiles * (tiles + 1) / 2;
  a.mp = (m + 31) / 32 * 32;
  a.xh = reinterpret_cast<float*>(take((size_t)n * a.mp * 4));
  a.xl = reinterpret_cast<float*>(take((size_t)n * a.mp * 4));
  a.band_x0 = reinterpret_cast<float*>(take((size_t)f.nb * m * 4));
  a.band_d = reinterpret_cast<float*>(take((size_t)f.nb * m * 4));
  a.band_m2 = reinterpret_cast<float*>(take((size_t)f.nb * m * 4));
  a.part = reinterpret_cast<float*>(take((size_t)Tmax * 4 * 2 * 128 * 256 * 4));
  const size_t nflags = (size_t)(f.nb * (a.mp / 32) + f.T * f.S * 2);
  a.flags = reinterpret_cast<unsigned*>(take((size_t)(f.nb * (a.mp / 32) + Tmax * 4 * 2) * 4));
  a.out = out; a.mean_out = mean; a.sd_out = sd;
  static const bool timing = getenv("PB_GRAM_TIMING") != nullptr;
  static unsigned long long* tbuf = nullptr;
  cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
  if (timing) cudaStreamIsCapturing(s, &cap);
  const bool tm_on = timing && cap == cudaStreamCaptureStatusNone;
  if (tm_on && !tbuf) cudaMalloc(&tbuf, 148 * 16 * sizeof(unsigned long long));  // tuning only
  if (tm_on) cudaMemsetAsync(tbuf, 0, 148 * 16 * sizeof(unsigned long long), s);
  a.ts = tm_on ? tbuf : nullptr;
  CUtensorMap hmap, lmap, omap, mmap;
  const bool dm_ok = make_map_mn_runs(&hmap, a.xh, a.mp, n, a.mp, GBK, 4, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B) &&
                     make_map_mn_runs(&lmap, a.xl, a.mp, n, a.mp, GBK, 4, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B);
  if (!dm_ok || !make_map2d(&omap, out, m, m, m, 32, 128, true) ||
      !make_map2d(&mmap, out, m, m, m, 32, 32, true))
    return cudaErrorInvalidValue;
  gram_zero_flags<<<1, 256, 0, s>>>(a.flags, (int)nflags);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  if (launches) ++*launches;
  const size_t smem = gram_smem_bytes();
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
  e = corr ? cudaLaunchKernelEx(&cfg, gram_fused_kernel<true>, hmap, lmap, omap, mmap, a)
           : cudaLaunchKernelEx(&cfg, gram_fused_kernel<false>, hmap, lmap, omap, mmap, a);
  if (launches) ++*launches;
  if (tm_on) {  // per-phase stamps: min / median / max over CTAs, us after the first entry
    std::vector<unsigned long long> h(148 * 16);
    cudaStreamSynchronize(s);
    cudaMemcpy(h.data(), tbuf, h.size() * 8, cudaMemcpyDeviceToHost);
    const int G = 2 * f.T * f.S;
    unsigned long long t0 = ~0ull;
    for (int c = 0; c < G; ++c) if (h[c * 16]) t0 = std::min(t0, h[c * 16]);
    const char* names[14] = {"entry", "prep done", "first band ready", "MMA done", "partials in", "end",
                             "var stats ready", "u0 loads in", "u0 shift", "u0 stores issued", "u0 published",
                             "finalised", "partner values in", "-"};
    {  // effective SM clock over [entry, end] (clock64 of threads 0 and 64 of one SM)
      std::vector<double> mhz;
      for (int c = 0; c < G; ++c)
        if (h[c * 16 + 5] > h[c * 16] && h[c * 16 + 15] > h[c * 16 + 14])
          mhz.push_back((double)(h[c * 16 + 15] - h[c * 16 + 14]) * 1e3 / (double)(h[c * 16 + 5] - h[c * 16]));
      if (!mhz.empty()) {
        std::sort(mhz.begin(), mhz.end());
        fprintf(stderr, "[pb gram timing] SM clock        med %7.0f MHz\n", mhz[mhz.size() / 2]);
      }
    }
    for (int k = 0; k < 13; ++k) {
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
