// k_stencil.cu — the SYCL-Bench polybench stencils (§VIII lists
// "2D Convolution", "3D Convolution" and "FDTD2D"; SURVEY.md §8(f) NEXT-3;
// definitions = readings R19-R21 in DESIGN.md).
//
// No contraction here, so no tensor cores: the convolutions are HBM streams and
// FDTD at the paper's 1024^2 is an L2/shared-memory-resident time loop. Loop
// internalization's role (stage what neighbouring work-items
// re-read through local memory) is played by
//   conv2d / conv3d: one "march" kernel. A CTA owns a tile of output columns (2-D:
//           1024 columns of a row; 3-D: 8 or 16 rows x 128 columns of a plane) and
//           marches along the slowest axis. A producer warp stages each plane (2-D:
//           row) tile plus its halo by 1-D bulk copies (the TMA engine) into a
//           shared-memory ring STAGES ahead (full / empty mbarriers, no CTA barrier
//           in the march), so the bytes in flight do not depend on registers. Every
//           staged plane contributes to three output planes held in registers
//           (register pipelining), so each tile is read from shared memory once.
//           The FMAs are packed (fma.rn.f32x2: two outputs per instruction), and
//           the zero pattern of the weights can be a compile-time template argument
//           (the paper's host-to-device constant propagation: a
//           filter known on the host specialises the device code); the weights'
//           values stay runtime arguments.
//   fdtd2d: a persistent cooperative kernel when every 64x128 tile fits on the GPU
//           at once: each tile keeps its core plus an 8-wide halo of the three
//           fields in shared memory, advances 8 steps, and exchanges only its
//           outer band with its 8 neighbours through L2 (release/acquire epoch
//           flags). Otherwise one fused launch per step, state ping-ponging through
//           the workspace. In both, the hz update's two neighbour values
//           (ex'[i][j+1], ey'[i+1][j]) are recomputed with the identical fp32
//           operations, so the result equals the sequential sweeps bitwise.
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>

#include <algorithm>
#include <cmath>

#include "pb_device.cuh"
#include "pb_internal.h"

namespace pb {
namespace {

int sm_count() {
  static int cache[64] = {0};
  int dev = 0;
  cudaGetDevice(&dev);
  int& n = cache[dev & 63];
  if (!n) {
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

// ============================================================== conv2d / conv3d
struct W27x2 {
  float2 w[27];  // (w, w): the weight broadcast to both lanes of a packed FMA
};

__device__ __forceinline__ float2 ffma2(float2 a, float2 b, float2 c) {  // a*b + c, two RN FMAs
  unsigned long long d;
  asm volatile("fma.rn.f32x2 %0, %1, %2, %3;"
      : "=l"(d)
      : "l"(*reinterpret_cast<unsigned long long*>(&a)), "l"(*reinterpret_cast<unsigned long long*>(&b)),
        "l"(*reinterpret_cast<unsigned long long*>(&c)));
  return *reinterpret_cast<float2*>(&d);
}


// 1-D bulk copy with an L2 eviction-priority hint (policy from createpolicy).
__device__ __forceinline__ void bulk_g2s_hint(void* dst, const void* src, uint32_t bytes, uint64_t* bar,
                                              uint64_t policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}
__device__ __forceinline__ uint64_t l2_policy(int kind) {
  uint64_t p = 0;
  if (kind == 2)
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  else
    asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(p));
  return p;
}

template <int NJT, int OROWS, int WPR, int RPW = 1>
struct March {
  // planes in flight (Little's law: ~100+ KB per SM at the resident CTA count)
  static constexpr int STAGES = NJT == 1 ? 6 : (OROWS / RPW == 8 && RPW == 1 ? 12 : 8);
  static constexpr int TC = 128 * WPR;               // tile columns
  static constexpr int TROWS = OROWS + NJT - 1;      // staged rows per plane
  static constexpr int PITCH = TC + 8;               // [3] left halo, [4, 4+TC) values, [4+TC] right halo
  static constexpr int TILE = TROWS * PITCH;         // floats per stage
  static constexpr int CW = OROWS / RPW * WPR;             // compute warps (RPW output rows each)
  static constexpr int THREADS = 32 * (CW + 1);            // + one producer warp
  static constexpr size_t SMEM = (size_t)STAGES * TILE * sizeof(float) + 2 * STAGES * sizeof(uint64_t);
};

// One plane q of the march (rows j0-(NJT>1) .. +TROWS, columns c0-4 .. c0+TC+4,
// clipped to the array) -> ring buffer `buf`, tx bytes on `bar`. Called by the whole
// producer warp: lane 0 posts the byte count, lane r copies tile row r.
template <int NJT, int OROWS, int WPR, int RPW>
__device__ __forceinline__ void march_issue(const float* A, float* buf, uint64_t* bar, int q, int j0, int c0,
                                            int nrow, int ncol, int hint, uint64_t pol, int lane) {
  using M = March<NJT, OROWS, WPR, RPW>;
  const int ka = max(c0 - 4, 0);
  const int kb = min(c0 + M::TC + 4, ncol);
  const int jb = j0 - (NJT > 1 ? 1 : 0);  // global row of tile row 0
  const int jlo = max(jb, 0);
  const int jhi = min(jb + M::TROWS, nrow);
  const uint32_t row_bytes = (uint32_t)(kb - ka) * 4u;
  if (lane == 0) mbar_arrive_expect_tx(bar, row_bytes * (uint32_t)(jhi - jlo));
  __syncwarp();
  const int jj = jb + lane;
  if (lane < M::TROWS && jj >= jlo && jj < jhi) {
    float* dst = buf + lane * M::PITCH + 4 + (ka - c0);
    const float* src = A + ((size_t)q * nrow + jj) * ncol + ka;
    if (hint)
      bulk_g2s_hint(dst, src, row_bytes, bar, pol);
    else
      bulk_g2s(dst, src, row_bytes, bar);
  }
}

// The 5 input pairs a thread's 4 outputs need from one staged row: (l,a) (a,b) (b,c) (c,d) (d,r).
struct Pairs {
  float2 p[5];
};
__device__ __forceinline__ Pairs read_pairs(const float* t) {  // t = row base + 4 + column offset
  const float4 v = *reinterpret_cast<const float4*>(t);
  const float l = t[-1], r = t[4];
  Pairs o;
  o.p[0] = make_float2(l, v.x);
  o.p[1] = make_float2(v.x, v.y);
  o.p[2] = make_float2(v.y, v.z);
  o.p[3] = make_float2(v.z, v.w);
  o.p[4] = make_float2(v.w, r);
  return o;
}

// Stores the interior part of 4 outputs (cols k..k+3, row base dst): float4 when all
// four are interior columns, else element-wise (border columns untouched).
__device__ __forceinline__ void store4_interior(float* dst, int k, int klo, int khi, float2 lo, float2 hi) {
  if (k >= klo && k + 3 <= khi) {
    __stcs(reinterpret_cast<float4*>(dst + k), make_float4(lo.x, lo.y, hi.x, hi.y));
  } else {
    const float o[4] = {lo.x, lo.y, hi.x, hi.y};
#pragma unroll
    for (int e = 0; e < 4; ++e)
      if (k + e >= klo && k + e <= khi) dst[k + e] = o[e];
  }
}

// MASK bit (di+1)*NJT*3 + dj*3 + (dk+1) set <=> that weight may be nonzero.
template <int NJT, uint32_t MASK>
__device__ __forceinline__ void march_taps(float2 (&am)[2], float2 (&a0)[2], float2 (&ap)[2], const Pairs* rows,
                                           const W27x2& w) {
#pragma unroll
  for (int dj = 0; dj < NJT; ++dj) {
#pragma unroll
    for (int dk = 0; dk < 3; ++dk) {
      const float2 xlo = rows[dj].p[dk], xhi = rows[dj].p[dk + 2];
      constexpr int PLANE = NJT * 3;
      const int tm = 2 * PLANE + dj * 3 + dk;  // di = +1 -> output plane q-1
      const int t0 = PLANE + dj * 3 + dk;      // di =  0 -> output plane q
      const int tp = dj * 3 + dk;              // di = -1 -> output plane q+1
      if (MASK & (1u << tm)) { am[0] = ffma2(w.w[tm], xlo, am[0]); am[1] = ffma2(w.w[tm], xhi, am[1]); }
      if (MASK & (1u << t0)) { a0[0] = ffma2(w.w[t0], xlo, a0[0]); a0[1] = ffma2(w.w[t0], xhi, a0[1]); }
      if (MASK & (1u << tp)) { ap[0] = ffma2(w.w[tp], xlo, ap[0]); ap[1] = ffma2(w.w[tp], xhi, ap[1]); }
    }
  }
}

// Work unit = (column chunk cc, row group rg, segment sg of output planes [o0, o1)).
// nrow = 1 for 2-D (the march axis is the row index; columns are the stencil's j).
// Warps 0..OROWS*WPR-1 compute; the last warp only issues the bulk copies. Stage s is
// handed over by full[s] (tx bytes) and released by empty[s] (one arrive per compute
// warp): no CTA-wide barrier inside the march.
template <int NJT, int OROWS, int WPR, int RPW, uint32_t MASK>
__global__ void __launch_bounds__(March<NJT, OROWS, WPR, RPW>::THREADS) march_kernel(const float* __restrict__ A,
                                                                       float* __restrict__ B, int ni, int nrow,
                                                                       int ncol, int seg, int ncc, int nrg, int hint,
                                                                       int order, const __grid_constant__ W27x2 w) {
  using M = March<NJT, OROWS, WPR, RPW>;
  constexpr int CW = M::CW;  // compute warps
  extern __shared__ __align__(128) float st_smem[];
  float* tiles = st_smem;
  uint64_t* full = reinterpret_cast<uint64_t*>(st_smem + M::STAGES * M::TILE);
  uint64_t* empty = full + M::STAGES;
  const int lane = threadIdx.x & 31, wp = threadIdx.x >> 5;
  // order 0: column chunks fastest; 1: row groups fastest (vertical neighbours, which
  // share a halo row, are adjacent in launch order)
  const int cc = order ? (blockIdx.x / nrg) % ncc : blockIdx.x % ncc;
  const int rg = order ? blockIdx.x % nrg : (blockIdx.x / ncc) % nrg;
  const int sg = blockIdx.x / (ncc * nrg);
  const int c0 = cc * M::TC, j0 = rg * OROWS;
  const int o0 = 1 + sg * seg;
  const int o1 = min(o0 + seg, ni - 1);  // output planes [o0, o1)
  if (o0 >= o1) return;
  const int q0 = o0 - 1;
  const int nplanes = o1 + 1 - q0;  // planes [o0-1, o1]
  if (threadIdx.x == 0) {
    for (int s = 0; s < M::STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], CW);
    }
    fence_mbar_init();
  }
  __syncthreads();
  pdl_wait();
  if (wp == CW) {  // producer warp
    const uint64_t pol = hint ? l2_policy(hint) : 0;
#pragma unroll 1
    for (int p = 0; p < nplanes; ++p) {
      const int s = p % M::STAGES;
      if (p >= M::STAGES) mbar_wait(&empty[s], (uint32_t)(((p / M::STAGES) - 1) & 1));
      march_issue<NJT, OROWS, WPR, RPW>(A, tiles + s * M::TILE, &full[s], q0 + p, j0, c0, nrow, ncol, hint, pol, lane);
    }
    return;
  }
  const int tr = (wp / WPR) * RPW;                 // first output row of this warp within the tile
  const int col = (wp % WPR) * 128 + 4 * lane;     // column offset within the tile
  const int k = c0 + col;
  bool store_ok[RPW];
#pragma unroll
  for (int r = 0; r < RPW; ++r) {
    const int j = j0 + tr + r;
    store_ok[r] = (NJT == 1 || (j >= 1 && j <= nrow - 2)) && k < ncol;
  }
  float2 acc[3][RPW][2];
#pragma unroll
  for (int a = 0; a < 3; ++a)
#pragma unroll
    for (int r = 0; r < RPW; ++r) acc[a][r][0] = acc[a][r][1] = make_float2(0.f, 0.f);

  auto step = [&](int p, float2(&am)[RPW][2], float2(&a0)[RPW][2], float2(&ap)[RPW][2]) {
    const int s = p % M::STAGES;
    mbar_wait(&full[s], (uint32_t)((p / M::STAGES) & 1));
    const float* t = tiles + s * M::TILE + tr * M::PITCH + 4 + col;
    Pairs rows[NJT + RPW - 1];
#pragma unroll
    for (int dj = 0; dj < NJT + RPW - 1; ++dj) rows[dj] = read_pairs(t + dj * M::PITCH);
#pragma unroll
    for (int r = 0; r < RPW; ++r) march_taps<NJT, MASK>(am[r], a0[r], ap[r], rows + r, w);
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);  // this warp is done reading stage s
#pragma unroll
    for (int r = 0; r < RPW; ++r) {
      if (p >= 2 && store_ok[r])  // output plane q-1 is complete
        store4_interior(B + ((size_t)(q0 + p - 1) * nrow + (NJT > 1 ? j0 + tr + r : 0)) * ncol, k, 1, ncol - 2,
                        am[r][0], am[r][1]);
      am[r][0] = am[r][1] = make_float2(0.f, 0.f);  // becomes the next plane's q+1 accumulator
    }
  };
#pragma unroll 1
  for (int p = 0; p < nplanes; p += 3) {  // roles rotate statically: (m, 0, p) = (0,1,2), (1,2,0), (2,0,1)
    step(p, acc[0], acc[1], acc[2]);
    if (p + 1 < nplanes) step(p + 1, acc[1], acc[2], acc[0]);
    if (p + 2 < nplanes) step(p + 2, acc[2], acc[0], acc[1]);
  }
}

// Zero patterns compiled as specialisations (bit t <=> weight t may be nonzero).
constexpr uint32_t MASK_DENSE = (1u << 27) - 1;
constexpr uint32_t MASK_DENSE9 = (1u << 9) - 1;

uint32_t weight_mask(const float* w, int n) {
  uint32_t m = 0;
  for (int t = 0; t < n; ++t)
    if (w[t] != 0.f) m |= 1u << t;
  return m;
}

// PolyBench-GPU 3DConvolution's 11 nonzero taps (R20): (di,dj,dk) =
// (-1,-1,-1) (-1,-1,+1) (-1,0,+1) (-1,+1,+1) (0,-1,0) (0,0,0) (0,+1,0)
// (+1,-1,-1) (+1,-1,+1) (+1,0,+1) (+1,+1,+1).
constexpr uint32_t tap3(int di, int dj, int dk) { return 1u << ((di + 1) * 9 + (dj + 1) * 3 + (dk + 1)); }
constexpr uint32_t MASK_PBGPU3D = tap3(-1, -1, -1) | tap3(-1, -1, 1) | tap3(-1, 0, 1) | tap3(-1, 1, 1) |
                                  tap3(0, -1, 0) | tap3(0, 0, 0) | tap3(0, 1, 0) | tap3(1, -1, -1) |
                                  tap3(1, -1, 1) | tap3(1, 0, 1) | tap3(1, 1, 1);

template <int NJT, int OROWS, int WPR, int RPW, uint32_t MASK>
cudaError_t launch_march(const float* A, float* B, int ni, int nrow, int ncol, const W27x2& w, cudaStream_t s) {
  using M = March<NJT, OROWS, WPR, RPW>;
  auto kern = march_kernel<NJT, OROWS, WPR, RPW, MASK>;
  cudaError_t e = ensure_smem<march_kernel<NJT, OROWS, WPR, RPW, MASK>>(M::SMEM);
  if (e != cudaSuccess) return e;
  static int per_sm = 0;  // resident CTAs per SM (same on every B200)
  if (!per_sm && (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, M::THREADS, M::SMEM) != cudaSuccess ||
                  per_sm <= 0))
    per_sm = 4;
  const int ncc = (ncol + M::TC - 1) / M::TC;
  const int nrg = (nrow + OROWS - 1) / OROWS;
  const long long tiles = (long long)ncc * nrg;
  const int interior = ni - 2;
  // Segments of the march: the CTA count tiles*nseg should fill whole waves of the
  // resident slots (a last wave 30% full costs a third of the run), and each segment
  // re-reads 2 halo planes. Score = wave efficiency x seg / (seg + 2).
  // (2-D: measured best with ~2 waves of long segments; the HBM stream, not the wave
  // tail, bounds it there.)
  const long long slots = (long long)sm_count() * per_sm;
  long long nseg = 1;
  double best = -1.0;
  for (long long c = 1; NJT > 1 && c <= 2048 && c <= interior; ++c) {
    const int sgl = (int)((interior + c - 1) / c);
    const long long cnt = tiles * ((interior + sgl - 1) / sgl);
    const double waves = (double)cnt / (double)slots;
    const double eff = waves / std::ceil(waves);
    const double score = eff * sgl / (sgl + 2.0);
    if (score > best + 1e-9) { best = score; nseg = c; }
  }
  if (NJT == 1) nseg = std::max(1ll, std::min<long long>(interior, (2 * slots + tiles - 1) / tiles));
  const int seg = (int)((interior + nseg - 1) / nseg);
  nseg = (interior + seg - 1) / seg;
  static const int hint = getenv("PB_ST_L2") ? atoi(getenv("PB_ST_L2")) : 0;        // tuning aid
  static const int order = getenv("PB_ST_ORDER") ? atoi(getenv("PB_ST_ORDER")) : 0;  // tuning aid
  return launch_pdl(kern, dim3((unsigned)(tiles * nseg)), dim3(M::THREADS), M::SMEM, s, A, B, ni, nrow, ncol, seg,
                    ncc, nrg, hint, order, w);
}

// ============================================================== fdtd-2d
// One time step t: (exo, eyo, hzo) = step(exi, eyi, hzi). Thread = 4 consecutive
// columns of one row. Every operation is the PolyBench statement's fp32 op in C
// order (no contraction: explicit _rn intrinsics), so the result is bitwise the
// sequential sweeps'.
__device__ __forceinline__ float ey_upd(float ey, float hz, float hz_up) {
  return __fsub_rn(ey, __fmul_rn(0.5f, __fsub_rn(hz, hz_up)));
}
__device__ __forceinline__ float ex_upd(float ex, float hz, float hz_left) {
  return __fsub_rn(ex, __fmul_rn(0.5f, __fsub_rn(hz, hz_left)));
}
__device__ __forceinline__ float hz_upd(float hz, float ex_r, float ex_c, float ey_d, float ey_c) {
  const float s = __fsub_rn(__fadd_rn(__fsub_rn(ex_r, ex_c), ey_d), ey_c);
  return __fsub_rn(hz, __fmul_rn(0.7f, s));
}

__global__ void __launch_bounds__(256) fdtd_step_kernel(const float* __restrict__ exi, const float* __restrict__ eyi,
                                                        const float* __restrict__ hzi, float* __restrict__ exo,
                                                        float* __restrict__ eyo, float* __restrict__ hzo,
                                                        const float* __restrict__ fict, int t, int nx, int ny) {
  pdl_wait();
  const int q = ny >> 2;  // float4 groups per row
  const long long g = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (g < (long long)nx * q) {
    const int i = (int)(g / q);
    const int j = (int)(g - (long long)i * q) * 4;
    const size_t e = (size_t)i * ny + j;
    const float4 h = *reinterpret_cast<const float4*>(hzi + e);
    const float4 x = *reinterpret_cast<const float4*>(exi + e);
    const float4 y = *reinterpret_cast<const float4*>(eyi + e);
    const float hl = (j > 0) ? hzi[e - 1] : 0.f;
    const bool last_col = (j + 4 >= ny);
    const float hr = last_col ? 0.f : hzi[e + 4];
    const float xr = last_col ? 0.f : exi[e + 4];
    // ey' (row i)
    float4 yn;
    if (i == 0) {
      const float f = fict[t];
      yn = make_float4(f, f, f, f);
    } else {
      const float4 hu = *reinterpret_cast<const float4*>(hzi + e - ny);
      yn = make_float4(ey_upd(y.x, h.x, hu.x), ey_upd(y.y, h.y, hu.y), ey_upd(y.z, h.z, hu.z), ey_upd(y.w, h.w, hu.w));
    }
    // ex' (row i): column 0 unchanged
    float4 xn;
    xn.x = (j == 0) ? x.x : ex_upd(x.x, h.x, hl);
    xn.y = ex_upd(x.y, h.y, h.x);
    xn.z = ex_upd(x.z, h.z, h.y);
    xn.w = ex_upd(x.w, h.w, h.z);
    float4 hn = h;
    if (i < nx - 1) {
      // ey'[i+1][j..] and ex'[i][j+4] recomputed with the owner's exact operations
      const float4 yd = *reinterpret_cast<const float4*>(eyi + e + ny);
      const float4 hd = *reinterpret_cast<const float4*>(hzi + e + ny);
      const float4 ydn = make_float4(ey_upd(yd.x, hd.x, h.x), ey_upd(yd.y, hd.y, h.y), ey_upd(yd.z, hd.z, h.z),
                                     ey_upd(yd.w, hd.w, h.w));
      const float xrn = last_col ? 0.f : ex_upd(xr, hr, h.w);
      hn.x = hz_upd(h.x, xn.y, xn.x, ydn.x, yn.x);
      hn.y = hz_upd(h.y, xn.z, xn.y, ydn.y, yn.y);
      hn.z = hz_upd(h.z, xn.w, xn.z, ydn.z, yn.z);
      if (!last_col) hn.w = hz_upd(h.w, xrn, xn.w, ydn.w, yn.w);  // j+3 = ny-1 is outside the hz sweep
    }
    *reinterpret_cast<float4*>(exo + e) = xn;
    *reinterpret_cast<float4*>(eyo + e) = yn;
    *reinterpret_cast<float4*>(hzo + e) = hn;
  }
  pdl_trigger();
}


// ---- persistent, temporally blocked variant ------------------------------------
// One CTA per FT_I x FT_J core tile (cooperative launch: every tile co-resident).
// A tile keeps its core plus an FT_H-wide halo of all three fields in shared memory
// and advances FT_H steps on that region without talking to anyone: values near
// the region's edge go stale (each step reads old neighbours one row/column out),
// but the staleness moves inward one point per step, so after FT_H steps the core
// is still exact. Then the tiles exchange: each publishes its core into a
// parity-double-buffered copy of the grid in global memory (L2-resident), releases
// its epoch flag, acquires its 8 neighbours' flags and reloads its halo ring (only
// the core's FT_H-wide outer band is published, only the ring is read back). HBM sees
// the state once in and once out; one neighbour round trip through L2 per FT_H steps
// replaces FT_H kernel launches. Every update is the PolyBench statement's fp32
// operations, so the result is bitwise the sequential sweeps'.
constexpr int FT_I = 64, FT_J = 128, FT_THREADS = 512;  // core tile; halo width FT_H is a template argument

__device__ __forceinline__ unsigned ld_acq(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_rel(unsigned* p, unsigned v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// Waits until every existing neighbour (8-neighbourhood) has flag >= v.
__device__ __forceinline__ void ft_wait_neighbours(const unsigned* flags, int ti, int tj, int tiles_i, int tiles_j,
                                                   unsigned v) {
  const int tid = threadIdx.x;
  if (tid < 9 && tid != 4) {
    const int ni = ti + tid / 3 - 1, nj = tj + tid % 3 - 1;
    if (ni >= 0 && ni < tiles_i && nj >= 0 && nj < tiles_j) {
      unsigned long long spins = 0;
      while (ld_acq(&flags[ni * tiles_j + nj]) < v) {
        if (++spins > (1ull << 30)) asm volatile("trap;");
      }
    }
  }
  __syncthreads();
}

template <int FT_H>
__global__ void __launch_bounds__(FT_THREADS, 1) fdtd_persist_kernel(float* __restrict__ ex, float* __restrict__ ey,
                                                                     float* __restrict__ hz,
                                                                     const float* __restrict__ fict, int tmax, int nx,
                                                                     int ny, int tiles_j, float* __restrict__ grid2,
                                                                     unsigned* __restrict__ flags) {
  constexpr int FT_RI = FT_I + 2 * FT_H, FT_RJ = FT_J + 2 * FT_H;  // region (H = 8: 80 x 144)
  constexpr int FT_GROUPS = FT_RI * FT_RJ / 4;
  constexpr int FT_G = (FT_GROUPS + FT_THREADS - 1) / FT_THREADS;  // float4 groups per thread
  extern __shared__ __align__(16) float ft_smem[];
  float* sx = ft_smem;                  // ex [FT_RI][FT_RJ]
  float* sy = sx + FT_RI * FT_RJ;       // ey
  float* sh = sy + FT_RI * FT_RJ;       // hz
  const int tiles_i = gridDim.x / tiles_j;
  const int ti = blockIdx.x / tiles_j, tj = blockIdx.x % tiles_j;
  const int i0 = ti * FT_I, j0 = tj * FT_J;  // core origin; region origin (i0 - H, j0 - H)
  const int tid = threadIdx.x;
  const size_t N = (size_t)nx * ny;
  pdl_wait();
  const int nep = (tmax + FT_H - 1) / FT_H;
  for (int e = 0; e < nep; ++e) {
    // 1. region <- the state after e*H steps (epoch 0: the caller's arrays)
    const float* gx = e == 0 ? ex : grid2 + (size_t)(e & 1) * 3 * N;
    const float* gy = e == 0 ? ey : gx + N;
    const float* gh = e == 0 ? hz : gx + 2 * N;
    if (e > 0) ft_wait_neighbours(flags, ti, tj, tiles_i, tiles_j, (unsigned)e);
    // epoch 0 loads the whole region; later epochs only the halo ring (the core in
    // shared memory is exact: it is this tile's own state)
    for (int g = tid; g < FT_GROUPS; g += FT_THREADS) {
      const int r = g / (FT_RJ / 4), c = (g % (FT_RJ / 4)) * 4;
      if (e > 0 && r >= FT_H && r < FT_H + FT_I && c >= FT_H && c < FT_H + FT_J) continue;
      const int i = i0 - FT_H + r, j = j0 - FT_H + c;
      float4 x = make_float4(0.f, 0.f, 0.f, 0.f), y = x, h = x;
      if (i >= 0 && i < nx && j >= 0 && j < ny) {
        const size_t o = (size_t)i * ny + j;
        x = __ldcg(reinterpret_cast<const float4*>(gx + o));
        y = __ldcg(reinterpret_cast<const float4*>(gy + o));
        h = __ldcg(reinterpret_cast<const float4*>(gh + o));
      }
      *reinterpret_cast<float4*>(sx + r * FT_RJ + c) = x;
      *reinterpret_cast<float4*>(sy + r * FT_RJ + c) = y;
      *reinterpret_cast<float4*>(sh + r * FT_RJ + c) = h;
    }
    __syncthreads();
    // 2. up to H steps on the region
    const int t_end = min(tmax, (e + 1) * FT_H);
    for (int t = e * FT_H; t < t_end; ++t) {
      float4 nxv[FT_G], nyv[FT_G], nhv[FT_G];
      const float f = __ldg(fict + t);
#pragma unroll
      for (int u = 0; u < FT_G; ++u) {
        const int g = tid + u * FT_THREADS;
        if (g >= FT_GROUPS) continue;
        const int r = g / (FT_RJ / 4), c = (g % (FT_RJ / 4)) * 4;
        const int i = i0 - FT_H + r, j = j0 - FT_H + c;
        const float4 h = *reinterpret_cast<const float4*>(sh + r * FT_RJ + c);
        const float4 x = *reinterpret_cast<const float4*>(sx + r * FT_RJ + c);
        const float4 y = *reinterpret_cast<const float4*>(sy + r * FT_RJ + c);
        nxv[u] = x;
        nyv[u] = y;
        nhv[u] = h;
        if (i < 0 || i >= nx || j < 0 || j >= ny) continue;  // outside the grid: never read by grid points
        // neighbours one out (clamped at the region edge: stale there, see above)
        const int ru = max(r - 1, 0), rd = min(r + 1, FT_RI - 1);
        const float hl = sh[r * FT_RJ + max(c - 1, 0)];
        const bool last_col = (j + 4 >= ny);
        const int cr = min(c + 4, FT_RJ - 1);
        const float hr = sh[r * FT_RJ + cr];
        const float xr = sx[r * FT_RJ + cr];
        float4 yn;
        if (i == 0) {
          yn = make_float4(f, f, f, f);
        } else {
          const float4 hu = *reinterpret_cast<const float4*>(sh + ru * FT_RJ + c);
          yn = make_float4(ey_upd(y.x, h.x, hu.x), ey_upd(y.y, h.y, hu.y), ey_upd(y.z, h.z, hu.z),
                           ey_upd(y.w, h.w, hu.w));
        }
        float4 xn;
        xn.x = (j == 0) ? x.x : ex_upd(x.x, h.x, hl);
        xn.y = ex_upd(x.y, h.y, h.x);
        xn.z = ex_upd(x.z, h.z, h.y);
        xn.w = ex_upd(x.w, h.w, h.z);
        float4 hn = h;
        if (i < nx - 1) {
          const float4 yd = *reinterpret_cast<const float4*>(sy + rd * FT_RJ + c);
          const float4 hd = *reinterpret_cast<const float4*>(sh + rd * FT_RJ + c);
          const float4 ydn = make_float4(ey_upd(yd.x, hd.x, h.x), ey_upd(yd.y, hd.y, h.y), ey_upd(yd.z, hd.z, h.z),
                                         ey_upd(yd.w, hd.w, h.w));
          const float xrn = ex_upd(xr, hr, h.w);
          hn.x = hz_upd(h.x, xn.y, xn.x, ydn.x, yn.x);
          hn.y = hz_upd(h.y, xn.z, xn.y, ydn.y, yn.y);
          hn.z = hz_upd(h.z, xn.w, xn.z, ydn.z, yn.z);
          if (!last_col) hn.w = hz_upd(h.w, xrn, xn.w, ydn.w, yn.w);
        }
        nxv[u] = xn;
        nyv[u] = yn;
        nhv[u] = hn;
      }
      __syncthreads();  // every thread has read the old state
#pragma unroll
      for (int u = 0; u < FT_G; ++u) {
        const int g = tid + u * FT_THREADS;
        if (g >= FT_GROUPS) continue;
        const int r = g / (FT_RJ / 4), c = (g % (FT_RJ / 4)) * 4;
        *reinterpret_cast<float4*>(sx + r * FT_RJ + c) = nxv[u];
        *reinterpret_cast<float4*>(sy + r * FT_RJ + c) = nyv[u];
        *reinterpret_cast<float4*>(sh + r * FT_RJ + c) = nhv[u];
      }
      __syncthreads();
    }
    // 3. publish the core: into the exchange copy (parity e+1), or - after the last
    //    epoch, once every neighbour is done reading - into the caller's arrays
    const bool last = (e + 1 == nep);
    if (last) {
      if (tid == 0) {
        __threadfence();
        st_rel(&flags[blockIdx.x], (unsigned)(nep + 1));  // "done reading" marker
      }
      ft_wait_neighbours(flags, ti, tj, tiles_i, tiles_j, (unsigned)(nep + 1));
    }
    float* px = last ? ex : grid2 + (size_t)((e + 1) & 1) * 3 * N;
    float* py = last ? ey : px + N;
    float* ph = last ? hz : px + 2 * N;
    for (int g = tid; g < FT_I * FT_J / 4; g += FT_THREADS) {
      const int r = g / (FT_J / 4), c = (g % (FT_J / 4)) * 4;
      // exchange copies need only the core's outer FT_H-wide band (what neighbours' halos read)
      if (!last && r >= FT_H && r < FT_I - FT_H && c >= FT_H && c < FT_J - FT_H) continue;
      const int i = i0 + r, j = j0 + c;
      if (i < nx && j < ny) {
        const size_t o = (size_t)i * ny + j;
        const int so = (r + FT_H) * FT_RJ + c + FT_H;
        *reinterpret_cast<float4*>(px + o) = *reinterpret_cast<const float4*>(sx + so);
        *reinterpret_cast<float4*>(py + o) = *reinterpret_cast<const float4*>(sy + so);
        *reinterpret_cast<float4*>(ph + o) = *reinterpret_cast<const float4*>(sh + so);
      }
    }
    if (!last) {
      __syncthreads();
      if (tid == 0) {
        __threadfence();
        st_rel(&flags[blockIdx.x], (unsigned)(e + 1));
      }
    }
  }
}


// ---- ablation: the SYCL-Bench kernel shape (one work-item per output point, every
// tap a global load, no staging: what the paper's loop internalization would have to
// stage, PAPER.md:551 notes it did not apply to these). Weights from the parameter
// block; same FMA order per point as the march kernel's rows (dj outer... per tap).
__global__ void __launch_bounds__(256) conv2d_naive_kernel(const float* __restrict__ A, float* __restrict__ B, int ni,
                                                           int nj, const __grid_constant__ W27x2 w) {
  const long long g = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long i = g / nj, j = g % nj;
  if (i < 1 || i >= ni - 1 || j < 1 || j >= nj - 1) return;
  float acc = 0.f;
#pragma unroll
  for (int di = -1; di <= 1; ++di)
#pragma unroll
    for (int dj = -1; dj <= 1; ++dj) acc = fmaf(w.w[(di + 1) * 3 + (dj + 1)].x, A[(i + di) * nj + (j + dj)], acc);
  B[i * nj + j] = acc;
}

__global__ void __launch_bounds__(256) conv3d_naive_kernel(const float* __restrict__ A, float* __restrict__ B, int ni,
                                                           int nj, int nk, const __grid_constant__ W27x2 w) {
  const long long g = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long k = g % nk, j = (g / nk) % nj, i = g / ((long long)nk * nj);
  if (i < 1 || i >= ni - 1 || j < 1 || j >= nj - 1 || k < 1 || k >= nk - 1) return;
  const long long pl = (long long)nj * nk;
  float acc = 0.f;
#pragma unroll
  for (int di = -1; di <= 1; ++di)
#pragma unroll
    for (int dj = -1; dj <= 1; ++dj)
#pragma unroll
      for (int dk = -1; dk <= 1; ++dk) {
        const float wv = w.w[(di + 1) * 9 + (dj + 1) * 3 + (dk + 1)].x;
        if (wv != 0.f) acc = fmaf(wv, A[(i + di) * pl + (j + dj) * nk + (k + dk)], acc);
      }
  B[(i * nj + j) * nk + k] = acc;
}

}  // namespace

cudaError_t launch_conv2d(const float* A, float* B, int ni, int nj, const float* w9, cudaStream_t s, int* launches) {
  if (ni < 3 || nj < 3) return cudaSuccess;  // no interior
  W27x2 w = {};
  for (int e = 0; e < 9; ++e) w.w[e] = make_float2(w9[e], w9[e]);
  ++*launches;
  // 2-D: the march axis is i, the stencil's column axis j is the tile's column axis
  // (no tile rows), taps w[(di+1)*3 + (dj+1)]
  return launch_march<1, 1, 8, 1, MASK_DENSE9>(A, B, ni, 1, nj, w, s);
}

cudaError_t launch_conv3d(const float* A, float* B, int ni, int nj, int nk, const float* w27, cudaStream_t s,
                          int* launches) {
  if (ni < 3 || nj < 3 || nk < 3) return cudaSuccess;
  W27x2 w;
  for (int e = 0; e < 27; ++e) w.w[e] = make_float2(w27[e], w27[e]);
  ++*launches;
  const uint32_t m = weight_mask(w27, 27);
  // Large grids: 16-row tiles, two output rows per warp (halo re-reads 18/16 instead of
  // 10/8 rows), 256 columns per tile when the rows are long enough (k-halo 8/256):
  // 1024^3: 1.60 (8 x 128) -> 1.54 (16 x 128) -> 1.50 ms (16 x 256). Smaller grids keep
  // 8-row tiles (more CTAs; 512^3: 0.209 vs 0.215 ms). PB_C3_RPW=1|2 overrides.
  static const int rpw_env = getenv("PB_C3_RPW") ? atoi(getenv("PB_C3_RPW")) : 0;
  const bool rpw2 = rpw_env ? rpw_env == 2 : (long long)ni * nj * nk >= (1ll << 28);
  const bool wide = rpw2 && nk >= 256;
  if ((m & ~MASK_PBGPU3D) == 0) {
    if (wide) return launch_march<3, 16, 2, 2, MASK_PBGPU3D>(A, B, ni, nj, nk, w, s);
    return rpw2 ? launch_march<3, 16, 1, 2, MASK_PBGPU3D>(A, B, ni, nj, nk, w, s)
                : launch_march<3, 8, 1, 1, MASK_PBGPU3D>(A, B, ni, nj, nk, w, s);
  }
  if (wide) return launch_march<3, 16, 2, 2, MASK_DENSE>(A, B, ni, nj, nk, w, s);
  return rpw2 ? launch_march<3, 16, 1, 2, MASK_DENSE>(A, B, ni, nj, nk, w, s)
              : launch_march<3, 8, 1, 1, MASK_DENSE>(A, B, ni, nj, nk, w, s);
}

namespace {
constexpr size_t ft_smem_bytes(int h) { return (size_t)3 * (FT_I + 2 * h) * (FT_J + 2 * h) * sizeof(float); }
size_t fdtd_persist_ws(int nx, int ny) {
  const size_t tiles = (size_t)((nx + FT_I - 1) / FT_I) * ((ny + FT_J - 1) / FT_J);
  return 2 * align_up(3 * (size_t)nx * ny * sizeof(float), 256) + align_up(tiles * sizeof(unsigned), 256);
}
}  // namespace

cudaError_t launch_conv_naive(bool three_d, const float* A, float* B, int ni, int nj, int nk, const float* w,
                              cudaStream_t s, int* launches) {
  if (ni < 3 || nj < 3 || (three_d && nk < 3)) return cudaSuccess;
  W27x2 wp = {};
  for (int e = 0; e < (three_d ? 27 : 9); ++e) wp.w[e] = make_float2(w[e], w[e]);
  const long long pts = (long long)ni * nj * (three_d ? nk : 1);
  const unsigned grid = (unsigned)((pts + 255) / 256);
  ++*launches;
  if (three_d) conv3d_naive_kernel<<<grid, 256, 0, s>>>(A, B, ni, nj, nk, wp);
  else conv2d_naive_kernel<<<grid, 256, 0, s>>>(A, B, ni, nj, wp);
  return cudaGetLastError();
}

size_t fdtd_ws_bytes(int nx, int ny) {
  return std::max(3 * align_up((size_t)nx * ny * sizeof(float), 256), fdtd_persist_ws(nx, ny));
}

cudaError_t launch_fdtd2d(int tmax, int nx, int ny, float* ex, float* ey, float* hz, const float* fict, void* ws,
                          cudaStream_t s, int* launches) {
  // Persistent path when every tile fits on the GPU at once (one CTA per SM: 135 KB at H = 8).
  static const int force_steps = getenv("PB_FDTD_STEPS") && atoi(getenv("PB_FDTD_STEPS")) == 1;  // tuning aid
  const int tiles_i = (nx + FT_I - 1) / FT_I, tiles_j = (ny + FT_J - 1) / FT_J;
  if (!force_steps && tmax > 0 && tiles_i * tiles_j <= sm_count()) {
    static const int h = getenv("PB_FDTD_H") ? atoi(getenv("PB_FDTD_H")) : 8;  // tuning aid: 4, 8, 16
    const size_t smem = ft_smem_bytes(h);
    cudaError_t e = h == 4 ? ensure_smem<fdtd_persist_kernel<4>>(smem)
                   : h == 16 ? ensure_smem<fdtd_persist_kernel<16>>(smem) : ensure_smem<fdtd_persist_kernel<8>>(smem);
    if (e != cudaSuccess) return e;
    const int tiles = tiles_i * tiles_j;
    float* grid2 = static_cast<float*>(ws);
    unsigned* flags = reinterpret_cast<unsigned*>(static_cast<char*>(ws) +
                                                  2 * align_up(3 * (size_t)nx * ny * sizeof(float), 256));
    if ((e = cudaMemsetAsync(flags, 0, tiles * sizeof(unsigned), s)) != cudaSuccess) return e;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(tiles);
    cfg.blockDim = dim3(FT_THREADS);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeCooperative;  // all tiles co-resident: the flag waits are safe
    at[0].val.cooperative = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    ++*launches;
    if (h == 4) return cudaLaunchKernelEx(&cfg, fdtd_persist_kernel<4>, ex, ey, hz, fict, tmax, nx, ny, tiles_j, grid2, flags);
    if (h == 16)
      return cudaLaunchKernelEx(&cfg, fdtd_persist_kernel<16>, ex, ey, hz, fict, tmax, nx, ny, tiles_j, grid2, flags);
    return cudaLaunchKernelEx(&cfg, fdtd_persist_kernel<8>, ex, ey, hz, fict, tmax, nx, ny, tiles_j, grid2, flags);
  }
  const size_t plane = align_up((size_t)nx * ny * sizeof(float), 256);
  float* wex = static_cast<float*>(ws);
  float* wey = reinterpret_cast<float*>(static_cast<char*>(ws) + plane);
  float* whz = reinterpret_cast<float*>(static_cast<char*>(ws) + 2 * plane);
  const long long threads = (long long)nx * (ny / 4);
  const unsigned grid = (unsigned)((threads + 255) / 256);
  for (int t = 0; t < tmax; ++t) {
    const bool even = (t % 2) == 0;
    cudaError_t e = launch_pdl(fdtd_step_kernel, dim3(grid), dim3(256), 0, s, even ? ex : wex, even ? ey : wey,
                               even ? hz : whz, even ? wex : ex, even ? wey : ey, even ? whz : hz, fict, t, nx, ny);
    if (e != cudaSuccess) return e;
    ++*launches;
  }
  if (tmax % 2 == 1) {  // the last step wrote the workspace copy
    const size_t bytes = (size_t)nx * ny * sizeof(float);
    cudaError_t e;
    if ((e = cudaMemcpyAsync(ex, wex, bytes, cudaMemcpyDeviceToDevice, s)) != cudaSuccess) return e;
    if ((e = cudaMemcpyAsync(ey, wey, bytes, cudaMemcpyDeviceToDevice, s)) != cudaSuccess) return e;
    if ((e = cudaMemcpyAsync(hz, whz, bytes, cudaMemcpyDeviceToDevice, s)) != cudaSuccess) return e;
  }
  return cudaSuccess;
}

}  // namespace pb
