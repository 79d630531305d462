// k_matvec.cu — S14-S16 of the hot path: the HBM-bound
// matrix-vector kernels of atax / bicg / mvt / gesummv.
//
// Paper mapping: the SYCL kernels walk a row (or a column) of A per
// work-item with a loop over global memory (PAPER.md:379 — local memory helps
// accesses "not conducive to being coalesced"). Here every matrix byte is read
// exactly once with coalesced 128-bit streaming loads (ld.global.nc,
// L1::no_allocate); the vector with temporal reuse (x / p / y_1) is kept in
// registers per thread (the loop-internalised operand), the
// reductions are register accumulators (detect-reduction)
// closed by warp shuffles, and the transposed product accumulates per-tile
// column partials that a second tiny kernel sums in a fixed order
// (deterministic, no float atomics). bicg and mvt compute both products in ONE
// pass over A (the paper's future-work kernel fusion).
#include <stdlib.h>

#include "pb_device.cuh"
#include "pb_internal.h"

namespace pb {
namespace {

// ------------------------------------------------------------------ rowdot
// y[i] = alpha*(A_i . x) + beta*(B_i . x); tmp[i] = A_i . x.  R rows per CTA.
template <int R, bool TWO>
__global__ void __launch_bounds__(256) rowdot_kernel(const float* __restrict__ A, const float* __restrict__ B,
                                                     const float* __restrict__ x, int rows, int cols, float alpha,
                                                     float beta, float* __restrict__ y, float* __restrict__ tmp) {
  const int row0 = blockIdx.x * R;
  const int cols4 = cols >> 2;
  const float4* x4 = reinterpret_cast<const float4*>(x);
  const float4* Ar[R];
  const float4* Br[R];
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const int row = min(row0 + r, rows - 1);
    Ar[r] = reinterpret_cast<const float4*>(A + (long long)row * cols);
    if (TWO) Br[r] = reinterpret_cast<const float4*>(B + (long long)row * cols);
  }
  float acc[R], accb[R];
#pragma unroll
  for (int r = 0; r < R; ++r) { acc[r] = 0.f; accb[r] = 0.f; }

  int c = threadIdx.x;
  for (; c + 256 < cols4; c += 512) {  // two column chunks in flight
    float4 a0[R], a1[R], b0[R], b1[R];
#pragma unroll
    for (int r = 0; r < R; ++r) {
      a0[r] = ldg_stream(Ar[r] + c);
      a1[r] = ldg_stream(Ar[r] + c + 256);
      if (TWO) { b0[r] = ldg_stream(Br[r] + c); b1[r] = ldg_stream(Br[r] + c + 256); }
    }
    const float4 xv0 = x4[c], xv1 = x4[c + 256];
#pragma unroll
    for (int r = 0; r < R; ++r) {
      acc[r] += a0[r].x * xv0.x + a0[r].y * xv0.y + a0[r].z * xv0.z + a0[r].w * xv0.w;
      acc[r] += a1[r].x * xv1.x + a1[r].y * xv1.y + a1[r].z * xv1.z + a1[r].w * xv1.w;
      if (TWO) {
        accb[r] += b0[r].x * xv0.x + b0[r].y * xv0.y + b0[r].z * xv0.z + b0[r].w * xv0.w;
        accb[r] += b1[r].x * xv1.x + b1[r].y * xv1.y + b1[r].z * xv1.z + b1[r].w * xv1.w;
      }
    }
  }
  for (; c < cols4; c += 256) {
    const float4 xv = x4[c];
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const float4 a = ldg_stream(Ar[r] + c);
      acc[r] += a.x * xv.x + a.y * xv.y + a.z * xv.z + a.w * xv.w;
      if (TWO) {
        const float4 b = ldg_stream(Br[r] + c);
        accb[r] += b.x * xv.x + b.y * xv.y + b.z * xv.z + b.w * xv.w;
      }
    }
  }
  __shared__ float red[2][8][R];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
#pragma unroll
  for (int r = 0; r < R; ++r) {
    float s = warp_sum(acc[r]);
    float sb = TWO ? warp_sum(accb[r]) : 0.f;
    if (lane == 0) { red[0][warp][r] = s; red[1][warp][r] = sb; }
  }
  __syncthreads();
  if (threadIdx.x < R && row0 + threadIdx.x < rows) {
    const int r = threadIdx.x;
    float s = 0.f, sb = 0.f;
#pragma unroll
    for (int w = 0; w < 8; ++w) { s += red[0][w][r]; sb += red[1][w][r]; }
    if (tmp) tmp[row0 + r] = s;
    if (y) y[row0 + r] = TWO ? alpha * s + beta * sb : alpha * s;
  }
}

// ------------------------------------------------------------------ fused mv / mv^T tiles
constexpr int TC = 512;  // columns per tile: 32 lanes x 4 float4 groups (128 cols apart)
constexpr int TR = 256;  // rows per tile: 8 warps x 32 rows
constexpr int G = TC / 128;
constexpr int RU = 4;    // rows in flight per warp

template <bool DO_ROW, bool DO_COL>
__global__ void __launch_bounds__(256, 2) mvmt_kernel(const float* __restrict__ A, int rows, int cols,
                                                      const float* __restrict__ v, const float* __restrict__ w,
                                                      float* __restrict__ rowpart, float* __restrict__ colpart) {
  const int ct = blockIdx.x, rt = blockIdx.y;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int c0 = ct * TC;
  bool cok[G];
  float4 vv[G], cacc[G];
#pragma unroll
  for (int g = 0; g < G; ++g) {
    const int c = c0 + g * 128 + lane * 4;
    cok[g] = c < cols;
    vv[g] = make_float4(0.f, 0.f, 0.f, 0.f);
    if (DO_ROW && cok[g]) vv[g] = *reinterpret_cast<const float4*>(v + c);
    cacc[g] = make_float4(0.f, 0.f, 0.f, 0.f);
  }
  const int r_begin = rt * TR, r_end = min(r_begin + TR, rows);
  for (int rb = r_begin + warp * RU; rb < r_end; rb += 8 * RU) {
    float4 a[RU][G];
#pragma unroll
    for (int u = 0; u < RU; ++u) {
      const int r = rb + u;
#pragma unroll
      for (int g = 0; g < G; ++g) {
        const int c = c0 + g * 128 + lane * 4;
        a[u][g] = (r < r_end && cok[g]) ? ldg_stream(reinterpret_cast<const float4*>(A + (long long)r * cols + c))
                                        : make_float4(0.f, 0.f, 0.f, 0.f);
      }
    }
#pragma unroll
    for (int u = 0; u < RU; ++u) {
      const int r = rb + u;
      if (DO_COL) {
        const float wr = r < r_end ? w[r] : 0.f;
#pragma unroll
        for (int g = 0; g < G; ++g) {
          cacc[g].x += wr * a[u][g].x; cacc[g].y += wr * a[u][g].y;
          cacc[g].z += wr * a[u][g].z; cacc[g].w += wr * a[u][g].w;
        }
      }
      if (DO_ROW) {
        float s = 0.f;
#pragma unroll
        for (int g = 0; g < G; ++g)
          s += a[u][g].x * vv[g].x + a[u][g].y * vv[g].y + a[u][g].z * vv[g].z + a[u][g].w * vv[g].w;
        s = warp_sum(s);
        if (lane == 0 && r < r_end) rowpart[(long long)ct * rows + r] = s;
      }
    }
  }
  if (DO_COL) {
    __shared__ float4 red[8][TC / 4];
#pragma unroll
    for (int g = 0; g < G; ++g) red[warp][g * 32 + lane] = cacc[g];
    __syncthreads();
    // 256 threads, TC/4 = 128 float4 columns: threads 0..127 each own one float4
    if (threadIdx.x < TC / 4) {
      const int f = threadIdx.x;  // float4 index within tile: g*32 + lane
      const int c = c0 + (f >> 5) * 128 + (f & 31) * 4;
      float4 s = red[0][f];
#pragma unroll
      for (int k = 1; k < 8; ++k) { s.x += red[k][f].x; s.y += red[k][f].y; s.z += red[k][f].z; s.w += red[k][f].w; }
      if (c < cols) *reinterpret_cast<float4*>(colpart + (long long)rt * cols + c) = s;
    }
  }
}

// gesummv in the 2-D tile pattern of mvmt_kernel (row dots only), A and B streamed
// together: CTA (ct, rt) writes pa[ct][r] = A[r][tile] . x[tile] and pb likewise for
// B; gesummv_reduce_kernel then forms y = alpha*sum_ct pa + beta*sum_ct pb in fixed
// order. Each matrix is read once; 2 rows of each in flight per warp (<= 128 regs).
constexpr int RU2 = 2;
__global__ void __launch_bounds__(256, 2) gesummv_tile_kernel(const float* __restrict__ A, const float* __restrict__ B,
                                                              int rows, int cols, const float* __restrict__ x,
                                                              float* __restrict__ pa, float* __restrict__ pb) {
  const int ct = blockIdx.x, rt = blockIdx.y;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int c0 = ct * TC;
  bool cok[G];
  float4 xv[G];
#pragma unroll
  for (int g = 0; g < G; ++g) {
    const int c = c0 + g * 128 + lane * 4;
    cok[g] = c < cols;
    xv[g] = cok[g] ? *reinterpret_cast<const float4*>(x + c) : make_float4(0.f, 0.f, 0.f, 0.f);
  }
  const int r_begin = rt * TR, r_end = min(r_begin + TR, rows);
  for (int rb = r_begin + warp * RU2; rb < r_end; rb += 8 * RU2) {
    float4 a[RU2][G], b[RU2][G];
#pragma unroll
    for (int u = 0; u < RU2; ++u) {
      const int r = rb + u;
#pragma unroll
      for (int g = 0; g < G; ++g) {
        const int c = c0 + g * 128 + lane * 4;
        const bool ok = r < r_end && cok[g];
        a[u][g] = ok ? ldg_stream(reinterpret_cast<const float4*>(A + (long long)r * cols + c))
                     : make_float4(0.f, 0.f, 0.f, 0.f);
        b[u][g] = ok ? ldg_stream(reinterpret_cast<const float4*>(B + (long long)r * cols + c))
                     : make_float4(0.f, 0.f, 0.f, 0.f);
      }
    }
#pragma unroll
    for (int u = 0; u < RU2; ++u) {
      const int r = rb + u;
      float sa = 0.f, sb = 0.f;
#pragma unroll
      for (int g = 0; g < G; ++g) {
        sa += a[u][g].x * xv[g].x + a[u][g].y * xv[g].y + a[u][g].z * xv[g].z + a[u][g].w * xv[g].w;
        sb += b[u][g].x * xv[g].x + b[u][g].y * xv[g].y + b[u][g].z * xv[g].z + b[u][g].w * xv[g].w;
      }
      sa = warp_sum(sa);
      sb = warp_sum(sb);
      if (lane == 0 && r < r_end) {
        pa[(long long)ct * rows + r] = sa;
        pb[(long long)ct * rows + r] = sb;
      }
    }
  }
}

__global__ void __launch_bounds__(256) gesummv_reduce_kernel(const float* __restrict__ pa, const float* __restrict__ pb,
                                                             int nparts, int rows, float alpha, float beta,
                                                             float* __restrict__ y, float* __restrict__ tmp) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= rows) return;
  float sa = 0.f, sb = 0.f;
  for (int t = 0; t < nparts; ++t) {
    sa += pa[(long long)t * rows + i];
    sb += pb[(long long)t * rows + i];
  }
  y[i] = alpha * sa + beta * sb;
  if (tmp) tmp[i] = sa;
}

// out[i] = (base ? base[i] : 0) + sum_{t < nparts} part[t][i]
__global__ void __launch_bounds__(256) reduce_parts_kernel(const float* __restrict__ part, int nparts, int len,
                                                           const float* __restrict__ base, float* __restrict__ out) {
  const int i = blockIdx.x * 256 + threadIdx.x;
  if (i >= len) return;
  float s = 0.f;
  for (int t = 0; t < nparts; ++t) s += part[(long long)t * len + i];
  out[i] = base ? base[i] + s : s;
}

// ------------------------------------------------------------------ atax, single pass
// y = A^T (A x) reading A ONCE (S16). A 2-CTA cluster owns a contiguous block of
// rows; CTA `rank` holds the column slice [c0, c0 + w) of every row. Per row b:
//   dot  : the slice arrives in an smem stage by 1-D bulk copy (TMA engine);
//          512 threads dot it with their registers of x -> CTA partial -> written
//          into BOTH CTAs' smem (DSMEM) and announced by a cluster-scope mbarrier
//          arrive (release), so neither CTA blocks on the other;
//   axpy : once both partials of row b are in (acquire), tmp_b = p0 + p1 (fixed
//          order, identical in both CTAs) and y_acc += tmp_b * A[b][slice] from the
//          SAME smem stage — the row is never re-read from HBM or L2.
// dot(b+1) is issued before axpy(b), hiding the DSMEM round trip. y_acc (the
// loop-carried reduction) lives in registers; the per-cluster
// partial y vectors are summed by reduce_parts_kernel in a fixed order.
constexpr int AX_THREADS = 512;
constexpr int AX_V = 8;                               // float4 per thread per slice
constexpr int AX_SLICE = AX_THREADS * AX_V * 4;       // 16384 floats = 64 KiB
constexpr int AX_STAGES = 3;
constexpr int AX_RED = 4;  // partial slots: a peer's dot(b+4) can only start after our axpy(b)

struct __align__(16) AxCtl {
  uint64_t full[AX_STAGES];
  uint64_t red[AX_RED];
  float part[AX_RED][2];
  float wred[AX_THREADS / 32];
};

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(AX_THREADS, 1)
    atax_onepass_kernel(const float* __restrict__ A, const float* __restrict__ x, int m, int n, int w0,
                        float* __restrict__ tmp, float* __restrict__ ypart) {
  extern __shared__ __align__(128) uint8_t sm[];
  float* stage_buf = reinterpret_cast<float*>(sm);
  AxCtl* ctl = reinterpret_cast<AxCtl*>(sm + (size_t)AX_STAGES * AX_SLICE * 4);
  const uint32_t rank = cluster_rank(), peer = rank ^ 1u;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int cl = blockIdx.x >> 1, ncl = gridDim.x >> 1;
  const int c0 = rank ? w0 : 0;
  const int w = rank ? n - w0 : w0;
  const int w4 = w >> 2;
  const int r0 = (int)((long long)m * cl / ncl), r1 = (int)((long long)m * (cl + 1) / ncl);
  const int nb = r1 - r0;

  if (tid == 0) {
    for (int s = 0; s < AX_STAGES; ++s) mbar_init(&ctl->full[s], 1);
    for (int s = 0; s < AX_RED; ++s) mbar_init(&ctl->red[s], 2);
    fence_mbar_init();
  }
  cluster_sync_all();  // both CTAs' barriers exist before any remote arrive

  float4 xv[AX_V], yacc[AX_V];
  const float4* x4 = reinterpret_cast<const float4*>(x + c0);
#pragma unroll
  for (int v = 0; v < AX_V; ++v) {
    const int idx = tid + v * AX_THREADS;
    xv[v] = idx < w4 ? x4[idx] : make_float4(0.f, 0.f, 0.f, 0.f);
    yacc[v] = make_float4(0.f, 0.f, 0.f, 0.f);
  }
  auto issue = [&](int b) {  // thread 0: row b's slice -> stage b % STAGES
    const int s = b % AX_STAGES;
    mbar_arrive_expect_tx(&ctl->full[s], (uint32_t)w * 4u);
    if (w > 0) bulk_g2s(stage_buf + (size_t)s * AX_SLICE, A + (long long)(r0 + b) * n + c0, (uint32_t)w * 4u,
                        &ctl->full[s]);
  };
  if (tid == 0)
    for (int b = 0; b < AX_STAGES && b < nb; ++b) issue(b);

  const uint32_t red0 = smem_u32(&ctl->red[0]);
  const uint32_t part0 = smem_u32(&ctl->part[0][0]);
  auto dot = [&](int b) {
    const int s = b % AX_STAGES;
    mbar_wait(&ctl->full[s], (uint32_t)(b / AX_STAGES) & 1u);
    const float4* row = reinterpret_cast<const float4*>(stage_buf + (size_t)s * AX_SLICE);
    float p = 0.f;
#pragma unroll
    for (int v = 0; v < AX_V; ++v) {
      const int idx = tid + v * AX_THREADS;
      if (idx < w4) {
        const float4 a = row[idx];
        p += a.x * xv[v].x + a.y * xv[v].y + a.z * xv[v].z + a.w * xv[v].w;
      }
    }
    p = warp_sum(p);
    if (lane == 0) ctl->wred[warp] = p;
    __syncthreads();
    if (tid == 0) {
      float q = 0.f;
#pragma unroll
      for (int k = 0; k < AX_THREADS / 32; ++k) q += ctl->wred[k];
      const int slot = b % AX_RED;
      const uint32_t poff = (uint32_t)(slot * 2 + rank) * 4u;
      const uint32_t roff = (uint32_t)slot * 8u;
      st_cluster_f32(map_peer(part0 + poff, rank), q);
      st_cluster_f32(map_peer(part0 + poff, peer), q);
      mbar_arrive_cluster(map_peer(red0 + roff, rank));
      mbar_arrive_cluster(map_peer(red0 + roff, peer));
    }
  };
  auto axpy = [&](int b) {
    const int slot = b % AX_RED;
    mbar_wait_cluster(&ctl->red[slot], (uint32_t)(b / AX_RED) & 1u);
    const float t = ctl->part[slot][0] + ctl->part[slot][1];
    if (tmp && rank == 0 && tid == 0) tmp[r0 + b] = t;
    const float4* row = reinterpret_cast<const float4*>(stage_buf + (size_t)(b % AX_STAGES) * AX_SLICE);
#pragma unroll
    for (int v = 0; v < AX_V; ++v) {
      const int idx = tid + v * AX_THREADS;
      if (idx < w4) {
        const float4 a = row[idx];
        yacc[v].x += t * a.x; yacc[v].y += t * a.y; yacc[v].z += t * a.z; yacc[v].w += t * a.w;
      }
    }
    __syncthreads();  // every thread is done with this stage
    if (tid == 0 && b + AX_STAGES < nb) issue(b + AX_STAGES);
  };

  if (nb > 0) dot(0);
  for (int b = 0; b < nb; ++b) {
    if (b + 1 < nb) dot(b + 1);
    axpy(b);
  }
  float4* yp = reinterpret_cast<float4*>(ypart + (long long)cl * n + c0);
#pragma unroll
  for (int v = 0; v < AX_V; ++v) {
    const int idx = tid + v * AX_THREADS;
    if (idx < w4) yp[idx] = yacc[v];
  }
  cluster_sync_all();  // no CTA leaves while its peer may still touch its smem
}

// a*b + c on two lanes at once (fma.rn.f32x2: one packed FFMA2 issue for two RN FMAs)
__device__ __forceinline__ float2 ffma2(float2 a, float2 b, float2 c) {
  unsigned long long d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;"
      : "=l"(d)
      : "l"(*reinterpret_cast<unsigned long long*>(&a)), "l"(*reinterpret_cast<unsigned long long*>(&b)),
        "l"(*reinterpret_cast<unsigned long long*>(&c)));
  return *reinterpret_cast<float2*>(&d);
}

// ------------------------------------------------------------------ atax, single pass, register rows
// Variant of the kernel above: each thread copies ITS float4s of row b from the
// smem stage into registers and the stage is handed back to the TMA engine at
// once (one CTA barrier per row), so stage reuse no longer waits for the DSMEM
// partial-dot exchange; x lives in smem, row b-1 stays in registers until its
// tmp arrives, the CTA partial is formed by the last warp to post (no barrier).
constexpr int AR_STAGES = 2;

struct __align__(16) ArCtl {
  uint64_t full[AR_STAGES];
  uint64_t red[AX_RED];
  unsigned cnt[AX_RED];
  float part[AX_RED][2];
  float wred[AX_RED][AX_THREADS / 32];
};

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(AX_THREADS, 1)
    atax_reg_kernel(const float* __restrict__ A, const float* __restrict__ x, int m, int n, int w0,
                    float* __restrict__ tmp, float* __restrict__ ypart) {
  extern __shared__ __align__(128) uint8_t sm[];
  float* xs = reinterpret_cast<float*>(sm);                          // AX_SLICE floats
  float* stage_buf = xs + AX_SLICE;                                  // AR_STAGES x AX_SLICE
  ArCtl* ctl = reinterpret_cast<ArCtl*>(stage_buf + (size_t)AR_STAGES * AX_SLICE);
  const uint32_t rank = cluster_rank(), peer = rank ^ 1u;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  constexpr int NW = AX_THREADS / 32;
  const int cl = blockIdx.x >> 1, ncl = gridDim.x >> 1;
  const int c0 = rank ? w0 : 0;
  const int w = rank ? n - w0 : w0;
  const int w4 = w >> 2;
  const int r0 = (int)((long long)m * cl / ncl), r1 = (int)((long long)m * (cl + 1) / ncl);
  const int nb = r1 - r0;

  if (tid == 0) {
    for (int s = 0; s < AR_STAGES; ++s) mbar_init(&ctl->full[s], 1);
    for (int s = 0; s < AX_RED; ++s) {
      mbar_init(&ctl->red[s], 2);
      ctl->cnt[s] = 0;
    }
    fence_mbar_init();
  }
  {
    const float4* x4 = reinterpret_cast<const float4*>(x + c0);
    float4* xs4 = reinterpret_cast<float4*>(xs);
    for (int i = tid; i < w4; i += AX_THREADS) xs4[i] = x4[i];
  }
  cluster_sync_all();  // barriers exist in both CTAs; x slice staged
  auto issue = [&](int b) {
    const int s = b % AR_STAGES;
    mbar_arrive_expect_tx(&ctl->full[s], (uint32_t)w * 4u);
    if (w > 0) bulk_g2s(stage_buf + (size_t)s * AX_SLICE, A + (long long)(r0 + b) * n + c0, (uint32_t)w * 4u,
                        &ctl->full[s]);
  };
  if (tid == 0)
    for (int b = 0; b < AR_STAGES && b < nb; ++b) issue(b);
  float4 yacc[AX_V];
#pragma unroll
  for (int v = 0; v < AX_V; ++v) yacc[v] = make_float4(0.f, 0.f, 0.f, 0.f);
  const uint32_t red0 = smem_u32(&ctl->red[0]);
  const uint32_t part0 = smem_u32(&ctl->part[0][0]);
  const float4* xs4 = reinterpret_cast<const float4*>(xs);

  // row b: load into `cur`, free the stage, dot, post; then finish row b-1 from `prev`
  auto step = [&](int b, float4(&cur)[AX_V], float4(&prev)[AX_V]) {
    const int s = b % AR_STAGES, slot = b % AX_RED;
    mbar_wait(&ctl->full[s], (uint32_t)(b / AR_STAGES) & 1u);
    const float4* row = reinterpret_cast<const float4*>(stage_buf + (size_t)s * AX_SLICE);
#pragma unroll
    for (int v = 0; v < AX_V; ++v) {
      const int idx = tid + v * AX_THREADS;
      cur[v] = idx < w4 ? row[idx] : make_float4(0.f, 0.f, 0.f, 0.f);
    }
    __syncthreads();  // every thread holds its part of row b: the stage can be refilled
    if (tid == 0 && b + AR_STAGES < nb) issue(b + AR_STAGES);
    // packed FMAs (two lanes per issue): the kernel's per-row instruction path is what the
    // power-capped SM clock slows down in the suite (DESIGN.md §8 atax)
    float2 pa = make_float2(0.f, 0.f), pb = make_float2(0.f, 0.f);
#pragma unroll
    for (int v = 0; v < AX_V; ++v) {
      const int idx = tid + v * AX_THREADS;
      if (idx < w4) {
        const float4 xv = xs4[idx];
        pa = ffma2(make_float2(cur[v].x, cur[v].y), make_float2(xv.x, xv.y), pa);
        pb = ffma2(make_float2(cur[v].z, cur[v].w), make_float2(xv.z, xv.w), pb);
      }
    }
    float p = (pa.x + pa.y) + (pb.x + pb.y);
    p = warp_sum(p);
    if (lane == 0) {
      volatile float* wr = ctl->wred[slot];
      wr[warp] = p;
      __threadfence_block();
      if (atomicAdd(&ctl->cnt[slot], 1u) == NW - 1) {  // last warp forms the CTA partial
        __threadfence_block();
        atomicExch(&ctl->cnt[slot], 0u);
        float q = 0.f;
#pragma unroll
        for (int k = 0; k < NW; ++k) q += wr[k];
        const uint32_t poff = (uint32_t)(slot * 2 + rank) * 4u, roff = (uint32_t)slot * 8u;
        st_cluster_f32(map_peer(part0 + poff, rank), q);
        st_cluster_f32(map_peer(part0 + poff, peer), q);
        mbar_arrive_cluster(map_peer(red0 + roff, rank));
        mbar_arrive_cluster(map_peer(red0 + roff, peer));
      }
    }
    if (b >= 1) {  // axpy of row b-1 (its partials had the whole dot of row b to arrive)
      const int ps = (b - 1) % AX_RED;
      mbar_wait_cluster(&ctl->red[ps], (uint32_t)((b - 1) / AX_RED) & 1u);
      const float t = ctl->part[ps][0] + ctl->part[ps][1];
      if (tmp && rank == 0 && tid == 0) tmp[r0 + b - 1] = t;
      const float2 t2 = make_float2(t, t);
#pragma unroll
      for (int v = 0; v < AX_V; ++v) {
        const float2 lo = ffma2(t2, make_float2(prev[v].x, prev[v].y), make_float2(yacc[v].x, yacc[v].y));
        const float2 hi = ffma2(t2, make_float2(prev[v].z, prev[v].w), make_float2(yacc[v].z, yacc[v].w));
        yacc[v] = make_float4(lo.x, lo.y, hi.x, hi.y);
      }
    }
  };
  float4 ra[AX_V], rb[AX_V];
  int b = 0;
  for (; b + 1 < nb; b += 2) {
    step(b, ra, rb);
    step(b + 1, rb, ra);
  }
  if (b < nb) step(b, ra, rb);
  if (nb > 0) {  // last row's axpy
    const int last = nb - 1, ps = last % AX_RED;
    float4(&lr)[AX_V] = (last & 1) ? rb : ra;
    mbar_wait_cluster(&ctl->red[ps], (uint32_t)(last / AX_RED) & 1u);
    const float t = ctl->part[ps][0] + ctl->part[ps][1];
    if (tmp && rank == 0 && tid == 0) tmp[r0 + last] = t;
    const float2 t2 = make_float2(t, t);
#pragma unroll
    for (int v = 0; v < AX_V; ++v) {
      const float2 lo = ffma2(t2, make_float2(lr[v].x, lr[v].y), make_float2(yacc[v].x, yacc[v].y));
      const float2 hi = ffma2(t2, make_float2(lr[v].z, lr[v].w), make_float2(yacc[v].z, yacc[v].w));
      yacc[v] = make_float4(lo.x, lo.y, hi.x, hi.y);
    }
  }
  float4* yp = reinterpret_cast<float4*>(ypart + (long long)cl * n + c0);
#pragma unroll
  for (int v = 0; v < AX_V; ++v) {
    const int idx = tid + v * AX_THREADS;
    if (idx < w4) yp[idx] = yacc[v];
  }
  cluster_sync_all();
}


// ------------------------------------------------------------------ atax, single pass, x in TMEM
// atax_reg_kernel with x held in tensor memory instead of shared memory. TMEM (256 KB per SM,
// otherwise idle here) is read with tcgen05.ld straight into registers, so the per-row dot no
// longer reads a 64 KB x slice through the shared-memory port (which also serves the TMA
// writes and the stage copies: 192 -> 128 KB of smem traffic per row), and the freed 64 KB
// holds a third stage. Thread (warp w, lane l) keeps its 32 x values in TMEM lane
// 32 (w % 4) + l, columns 32 (w / 4) .. + 31 (a warp may only touch its lane quarter).
// The CTA's partial dot is formed by the last warp to post (fence + counter, as in
// atax_reg_kernel); the warp partials go through shared-memory atomics so the hand-off has
// no plain racing accesses. (Posting every warp's partial into both CTAs with 2 x 16
// cluster-barrier arrivals per row was measured slower: 844 vs 702 us.)
constexpr int AT_STAGES = 3;
constexpr uint32_t AT_TMEM_COLS = 128;

struct __align__(16) AtCtl {
  uint64_t full[AT_STAGES];
  uint64_t red[AX_RED];
  unsigned cnt[AX_RED];
  float part[AX_RED][2];
  unsigned wred[AX_RED][AX_THREADS / 32];  // warp partials (fp32 bits)
  uint32_t tmem_base;
};

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(AX_THREADS, 1)
    atax_tm_kernel(const float* __restrict__ A, const float* __restrict__ x, int m, int n, int w0,
                   float* __restrict__ tmp, float* __restrict__ ypart, int chunks) {
  extern __shared__ __align__(128) uint8_t sm[];
  float* stage_buf = reinterpret_cast<float*>(sm);  // AT_STAGES x AX_SLICE
  AtCtl* ctl = reinterpret_cast<AtCtl*>(stage_buf + (size_t)AT_STAGES * AX_SLICE);
  const uint32_t rank = cluster_rank(), peer = rank ^ 1u;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  constexpr int NW = AX_THREADS / 32;
  const int cl = blockIdx.x >> 1, ncl = gridDim.x >> 1;
  const int c0 = rank ? w0 : 0;
  const int w = rank ? n - w0 : w0;
  const int w4 = w >> 2;
  const int r0 = (int)((long long)m * cl / ncl), r1 = (int)((long long)m * (cl + 1) / ncl);
  const int nb = r1 - r0;

  if (tid == 0) {
    for (int s = 0; s < AT_STAGES; ++s) mbar_init(&ctl->full[s], 1);
    for (int s = 0; s < AX_RED; ++s) {
      mbar_init(&ctl->red[s], 2);
      ctl->cnt[s] = 0;
    }
    fence_mbar_init();
  }
  if (warp == 0) tmem_alloc(&ctl->tmem_base, AT_TMEM_COLS);
  // a row slice arrives as `chunks` bulk copies (16-B multiples) on one barrier (PB_ATAX_CHUNKS)
  const uint32_t cbytes = (((uint32_t)w * 4u + (uint32_t)chunks - 1u) / (uint32_t)chunks + 15u) & ~15u;
  auto issue = [&](int b) {
    const int s = b % AT_STAGES;
    mbar_arrive_expect_tx(&ctl->full[s], (uint32_t)w * 4u);
    const char* src = reinterpret_cast<const char*>(A + (long long)(r0 + b) * n + c0);
    char* dst = reinterpret_cast<char*>(stage_buf + (size_t)s * AX_SLICE);
    for (uint32_t off = 0; off < (uint32_t)w * 4u; off += cbytes) {
      const uint32_t len = min(cbytes, (uint32_t)w * 4u - off);
      bulk_g2s(dst + off, src + off, len, &ctl->full[s]);
    }
  };
  tc_fence_before();
  cluster_sync_all();  // barriers exist in both CTAs; TMEM allocated
  tc_fence_after();
  if (tid == 0)
    for (int b = 0; b < AT_STAGES && b < nb; ++b) issue(b);
  const uint32_t tx = ctl->tmem_base + ((uint32_t)(32 * (warp & 3)) << 16) + (uint32_t)(warp >> 2) * 32u;
  {  // this thread's x float4s (idx = tid + v AX_THREADS, zero past the slice) -> TMEM
    const float4* x4 = reinterpret_cast<const float4*>(x + c0);
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      uint32_t r[16];
#pragma unroll
      for (int v = 0; v < 4; ++v) {
        const int idx = tid + (h * 4 + v) * AX_THREADS;
        const float4 xv = idx < w4 ? x4[idx] : make_float4(0.f, 0.f, 0.f, 0.f);
        r[4 * v] = __float_as_uint(xv.x); r[4 * v + 1] = __float_as_uint(xv.y);
        r[4 * v + 2] = __float_as_uint(xv.z); r[4 * v + 3] = __float_as_uint(xv.w);
      }
      tmem_st16(tx + 16u * h, r);
    }
    tmem_wait_st();
  }
  float4 yacc[AX_V];
#pragma unroll
  for (int v = 0; v < AX_V; ++v) yacc[v] = make_float4(0.f, 0.f, 0.f, 0.f);
  const uint32_t red0 = smem_u32(&ctl->red[0]);
  const uint32_t part0 = smem_u32(&ctl->part[0][0]);

  auto step = [&](int b, float4(&cur)[AX_V], float4(&prev)[AX_V]) {
    const int s = b % AT_STAGES, slot = b % AX_RED;
    mbar_wait(&ctl->full[s], (uint32_t)(b / AT_STAGES) & 1u);
    const float4* row = reinterpret_cast<const float4*>(stage_buf + (size_t)s * AX_SLICE);
#pragma unroll
    for (int v = 0; v < AX_V; ++v) {
      const int idx = tid + v * AX_THREADS;
      cur[v] = idx < w4 ? row[idx] : make_float4(0.f, 0.f, 0.f, 0.f);
    }
    __syncthreads();  // every thread holds its part of row b: the stage can be refilled
    if (tid == 0 && b + AT_STAGES < nb) issue(b + AT_STAGES);
    float2 pa = make_float2(0.f, 0.f), pb = make_float2(0.f, 0.f);
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      uint32_t xr[16];
      tmem_ld16(tx + 16u * h, xr);
      tmem_wait_ld();
#pragma unroll
      for (int v = 0; v < 4; ++v) {
        const float4 c = cur[h * 4 + v];
        pa = ffma2(make_float2(c.x, c.y), make_float2(__uint_as_float(xr[4 * v]), __uint_as_float(xr[4 * v + 1])), pa);
        pb = ffma2(make_float2(c.z, c.w), make_float2(__uint_as_float(xr[4 * v + 2]), __uint_as_float(xr[4 * v + 3])),
                   pb);
      }
    }
    float p = (pa.x + pa.y) + (pb.x + pb.y);
    p = warp_sum(p);
    if (lane == 0) {
      unsigned* wr = ctl->wred[slot];
      atomicExch(&wr[warp], __float_as_uint(p));  // (atomics: the hand-off below is fence + counter)
      __threadfence_block();
      if (atomicAdd(&ctl->cnt[slot], 1u) == NW - 1) {  // last warp forms the CTA partial
        __threadfence_block();
        atomicExch(&ctl->cnt[slot], 0u);
        float q = 0.f;
#pragma unroll
        for (int k = 0; k < NW; ++k) q += __uint_as_float(atomicAdd(&wr[k], 0u));
        const uint32_t poff = (uint32_t)(slot * 2 + rank) * 4u, roff = (uint32_t)slot * 8u;
        st_cluster_f32(map_peer(part0 + poff, rank), q);
        st_cluster_f32(map_peer(part0 + poff, peer), q);
        mbar_arrive_cluster(map_peer(red0 + roff, rank));
        mbar_arrive_cluster(map_peer(red0 + roff, peer));
      }
    }
    if (b >= 1) {  // axpy of row b-1 (its partials had the whole dot of row b to arrive)
      const int ps = (b - 1) % AX_RED;
      mbar_wait_cluster(&ctl->red[ps], (uint32_t)((b - 1) / AX_RED) & 1u);
      const float t = ctl->part[ps][0] + ctl->part[ps][1];
      if (tmp && rank == 0 && tid == 0) tmp[r0 + b - 1] = t;
      const float2 t2 = make_float2(t, t);
#pragma unroll
      for (int v = 0; v < AX_V; ++v) {
        const float2 lo = ffma2(t2, make_float2(prev[v].x, prev[v].y), make_float2(yacc[v].x, yacc[v].y));
        const float2 hi = ffma2(t2, make_float2(prev[v].z, prev[v].w), make_float2(yacc[v].z, yacc[v].w));
        yacc[v] = make_float4(lo.x, lo.y, hi.x, hi.y);
      }
    }
  };
  float4 ra[AX_V], rb[AX_V];
  int b = 0;
  for (; b + 1 < nb; b += 2) {
    step(b, ra, rb);
    step(b + 1, rb, ra);
  }
  if (b < nb) step(b, ra, rb);
  if (nb > 0) {  // last row's axpy
    const int last = nb - 1, ps = last % AX_RED;
    float4(&lr)[AX_V] = (last & 1) ? rb : ra;
    mbar_wait_cluster(&ctl->red[ps], (uint32_t)(last / AX_RED) & 1u);
    const float t = ctl->part[ps][0] + ctl->part[ps][1];
    if (tmp && rank == 0 && tid == 0) tmp[r0 + last] = t;
    const float2 t2 = make_float2(t, t);
#pragma unroll
    for (int v = 0; v < AX_V; ++v) {
      const float2 lo = ffma2(t2, make_float2(lr[v].x, lr[v].y), make_float2(yacc[v].x, yacc[v].y));
      const float2 hi = ffma2(t2, make_float2(lr[v].z, lr[v].w), make_float2(yacc[v].z, yacc[v].w));
      yacc[v] = make_float4(lo.x, lo.y, hi.x, hi.y);
    }
  }
  float4* yp = reinterpret_cast<float4*>(ypart + (long long)cl * n + c0);
#pragma unroll
  for (int v = 0; v < AX_V; ++v) {
    const int idx = tid + v * AX_THREADS;
    if (idx < w4) yp[idx] = yacc[v];
  }
  tc_fence_before();
  cluster_sync_all();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc(ctl->tmem_base, AT_TMEM_COLS);
  }
}

}  // namespace

size_t atax_ws_bytes(int m, int n) {
  const size_t onepass = align_up((size_t)74 * n * 4, 256);
  const size_t twopass = mvmt_ws_bytes(m, n);
  return (onepass > twopass ? onepass : twopass) + align_up((size_t)m * 4, 256);
}

cudaError_t launch_atax(const float* A, const float* x, int m, int n, float* y, float* tmp, void* ws,
                        cudaStream_t s, int* launches) {
  float* t = reinterpret_cast<float*>(static_cast<char*>(ws) + (atax_ws_bytes(m, n) - align_up((size_t)m * 4, 256)));
  if (!tmp) tmp = t;
  // Single pass only for long rows of a matrix larger than L2. With two stages of
  // half-rows in flight per CTA, short rows leave too few bytes outstanding (the
  // cluster kernel is then latency-bound), and a matrix that fits in L2 is read
  // from HBM once by the two-pass form anyway. Measured crossover (B200, cold L2):
  // n = 8192: 160 vs 96 us two-pass; n = 16384: 317 vs 346; n = 24576: 497 vs 713.
  static const long long onepass_min = (getenv("PB_ATAX_ONEPASS_MIN_MB") ? atoll(getenv("PB_ATAX_ONEPASS_MIN_MB"))
                                                                          : 96ll) << 20;
  if (n >= 16384 && n <= 2 * AX_SLICE && m >= 2 * 74 && (long long)m * n * 4 >= onepass_min) {
    static std::atomic<int> ncl_dev[64];  // clusters that fit, per device
    int dev = 0;
    cudaGetDevice(&dev);
    int ncl = ncl_dev[dev & 63].load(std::memory_order_relaxed);
    const size_t smem = (size_t)AX_STAGES * AX_SLICE * 4 + sizeof(AxCtl);
    {
      const cudaError_t e = ensure_smem<atax_onepass_kernel>(smem);
      if (e != cudaSuccess) return e;
    }
    if (!ncl) {
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(148);
      cfg.blockDim = dim3(AX_THREADS);
      cfg.dynamicSmemBytes = smem;
      cudaLaunchAttribute at;
      at.id = cudaLaunchAttributeClusterDimension;
      at.val.clusterDim.x = 2; at.val.clusterDim.y = 1; at.val.clusterDim.z = 1;
      cfg.attrs = &at;
      cfg.numAttrs = 1;
      int nc = 0;
      if (cudaOccupancyMaxActiveClusters(&nc, atax_onepass_kernel, &cfg) != cudaSuccess || nc <= 0) {
        cudaGetLastError();
        nc = 74;
      }
      ncl = nc < 74 ? nc : 74;
      ncl_dev[dev & 63].store(ncl, std::memory_order_relaxed);
    }
    const int w0 = ((n / 4 + 1) / 2) * 4;
    float* ypart = static_cast<float*>(ws);
    static const int variant = getenv("PB_ATAX_VARIANT") ? atoi(getenv("PB_ATAX_VARIANT")) : 3;
    if (variant == 3) {
      const size_t smem3 = (size_t)AT_STAGES * AX_SLICE * 4 + sizeof(AtCtl);
      {
        const cudaError_t e = ensure_smem<atax_tm_kernel>(smem3);
        if (e != cudaSuccess) return e;
      }
      static const int chunks = getenv("PB_ATAX_CHUNKS") ? std::max(1, std::min(64, atoi(getenv("PB_ATAX_CHUNKS")))) : 1;
      atax_tm_kernel<<<2 * ncl, AX_THREADS, smem3, s>>>(A, x, m, n, w0, tmp, ypart, chunks);
    } else if (variant == 2) {
      const size_t smem2 = (size_t)(1 + AR_STAGES) * AX_SLICE * 4 + sizeof(ArCtl);
      {
        const cudaError_t e = ensure_smem<atax_reg_kernel>(smem2);
        if (e != cudaSuccess) return e;
      }
      atax_reg_kernel<<<2 * ncl, AX_THREADS, smem2, s>>>(A, x, m, n, w0, tmp, ypart);
    } else {
      atax_onepass_kernel<<<2 * ncl, AX_THREADS, smem, s>>>(A, x, m, n, w0, tmp, ypart);
    }
    reduce_parts_kernel<<<(n + 255) / 256, 256, 0, s>>>(ypart, ncl, n, nullptr, y);
    *launches += 2;
    return cudaGetLastError();
  }
  // two passes: tmp = A x, then y = A^T tmp
  cudaError_t e = launch_rowdot(A, nullptr, x, m, n, 1.f, 0.f, nullptr, tmp, s);
  if (e != cudaSuccess) return e;
  ++*launches;
  return launch_mvmt(A, m, n, nullptr, tmp, nullptr, nullptr, nullptr, y, ws, s, launches);
}

cudaError_t launch_rowdot(const float* A, const float* B, const float* x, int rows, int cols, float alpha, float beta,
                          float* y, float* tmp, cudaStream_t s) {
  if (B) {
    constexpr int R = 4;
    rowdot_kernel<R, true><<<(rows + R - 1) / R, 256, 0, s>>>(A, B, x, rows, cols, alpha, beta, y, tmp);
  } else {
    constexpr int R = 8;
    rowdot_kernel<R, false><<<(rows + R - 1) / R, 256, 0, s>>>(A, nullptr, x, rows, cols, alpha, beta, y, tmp);
  }
  return cudaGetLastError();
}

size_t gesummv_ws_bytes(int rows, int cols) {
  const size_t nct = (cols + TC - 1) / TC;
  return 2 * align_up(nct * rows * 4, 256);
}

cudaError_t launch_gesummv(const float* A, const float* B, const float* x, int rows, int cols, float alpha, float beta,
                           float* y, float* tmp, void* ws, cudaStream_t s, int* launches) {
  const int nct = (cols + TC - 1) / TC, nrt = (rows + TR - 1) / TR;
  float* pa = static_cast<float*>(ws);
  float* pb = reinterpret_cast<float*>(static_cast<char*>(ws) + align_up((size_t)nct * rows * 4, 256));
  gesummv_tile_kernel<<<dim3(nct, nrt), 256, 0, s>>>(A, B, rows, cols, x, pa, pb);
  gesummv_reduce_kernel<<<(rows + 255) / 256, 256, 0, s>>>(pa, pb, nct, rows, alpha, beta, y, tmp);
  *launches += 2;
  return cudaGetLastError();
}

size_t mvmt_ws_bytes(int rows, int cols) {
  const size_t nct = (cols + TC - 1) / TC, nrt = (rows + TR - 1) / TR;
  return align_up(nct * rows * 4, 256) + align_up(nrt * cols * 4, 256);
}

cudaError_t launch_mvmt(const float* A, int rows, int cols, const float* v, const float* w, const float* base_row,
                        float* out_row, const float* base_col, float* out_col, void* ws, cudaStream_t s,
                        int* launches) {
  const int nct = (cols + TC - 1) / TC, nrt = (rows + TR - 1) / TR;
  float* rowpart = static_cast<float*>(ws);
  float* colpart = reinterpret_cast<float*>(static_cast<char*>(ws) + align_up((size_t)nct * rows * 4, 256));
  dim3 grid(nct, nrt);
  if (v && w)
    mvmt_kernel<true, true><<<grid, 256, 0, s>>>(A, rows, cols, v, w, rowpart, colpart);
  else if (v)
    mvmt_kernel<true, false><<<grid, 256, 0, s>>>(A, rows, cols, v, w, rowpart, colpart);
  else
    mvmt_kernel<false, true><<<grid, 256, 0, s>>>(A, rows, cols, v, w, rowpart, colpart);
  ++*launches;
  if (v) {
    reduce_parts_kernel<<<(rows + 255) / 256, 256, 0, s>>>(rowpart, nct, rows, base_row, out_row);
    ++*launches;
  }
  if (w) {
    reduce_parts_kernel<<<(cols + 255) / 256, 256, 0, s>>>(colpart, nrt, cols, base_col, out_col);
    ++*launches;
  }
  return cudaGetLastError();
}

}  // namespace pb
