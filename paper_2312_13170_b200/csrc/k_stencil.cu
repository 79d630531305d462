// k_stencil.cu — the SYCL-Bench polybench stencils (§VIII lists
// "2D Convolution", "3D Convolution" and "FDTD2D"; SURVEY.md §8(f) NEXT-3;
// definitions = readings R19-R21 in DESIGN.md).
//
// All three are HBM- (or, for FDTD at the paper's 1024^2, L2-) streaming
// kernels: no contraction, so no tensor cores. Loop internalization's role
// (stage what neighbouring work-items re-read through local
// memory) is played by
//   conv2d: registers. A warp owns 128 contiguous columns and marches down a row
//           strip; each lane keeps a 3-row window (float4 + its two neighbour
//           columns, taken from the adjacent lanes by shuffles), so every element
//           of A is loaded from global memory once per strip.
//   conv3d: a shared-memory ring of plane tiles (10 rows x 136 floats: the CTA's
//           8 output rows, their j-halo and a k-halo) filled by 1-D bulk copies
//           (the TMA engine) STAGES planes ahead; the CTA marches along i and
//           each plane contributes to three output planes held in registers
//           (register pipelining), so every plane tile is read from smem once.
//   fdtd2d: one fused launch per time step. The three PolyBench sweeps are
//           evaluated per point from the previous step's state; the two
//           neighbour values the hz update needs (ex'[i][j+1], ey'[i+1][j]) are
//           recomputed with the identical fp32 operations, so the result equals
//           the sequential sweeps bitwise. State ping-pongs between the caller's
//           arrays and the workspace (the sweeps' Jacobi structure needs the old
//           neighbours).
#include <cuda_runtime.h>
#include <stdint.h>

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

// ============================================================== conv2d
struct W9 {
  float w[9];
};

// One lane's view of one row: 4 owned columns and the two neighbours.
struct Row6 {
  float l, a, b, c, d, r;
};

__device__ __forceinline__ Row6 load_row2d(const float* __restrict__ row, int c0, int j, bool active, int lane,
                                           int nj) {
  float4 v = active ? ldg_stream(reinterpret_cast<const float4*>(row + j)) : make_float4(0.f, 0.f, 0.f, 0.f);
  Row6 o;
  o.a = v.x; o.b = v.y; o.c = v.z; o.d = v.w;
  float left = __shfl_up_sync(0xffffffffu, v.w, 1);
  float right = __shfl_down_sync(0xffffffffu, v.x, 1);
  if (lane == 0) left = (c0 > 0) ? __ldg(row + c0 - 1) : 0.f;
  if (lane == 31) right = (c0 + 128 < nj) ? __ldg(row + c0 + 128) : 0.f;
  o.l = left;
  o.r = right;
  return o;
}

__device__ __forceinline__ void acc_row(float (&o)[4], const Row6& x, float w0, float w1, float w2) {
  o[0] = fmaf(w0, x.l, o[0]); o[0] = fmaf(w1, x.a, o[0]); o[0] = fmaf(w2, x.b, o[0]);
  o[1] = fmaf(w0, x.a, o[1]); o[1] = fmaf(w1, x.b, o[1]); o[1] = fmaf(w2, x.c, o[1]);
  o[2] = fmaf(w0, x.b, o[2]); o[2] = fmaf(w1, x.c, o[2]); o[2] = fmaf(w2, x.d, o[2]);
  o[3] = fmaf(w0, x.c, o[3]); o[3] = fmaf(w1, x.d, o[3]); o[3] = fmaf(w2, x.r, o[3]);
}

// Store the interior part of 4 outputs at (i, j..j+3): float4 when all four are
// interior columns, else element-wise (border columns 0 and nj-1 untouched).
__device__ __forceinline__ void store4_interior(float* dst, int j, int jlo, int jhi, const float (&o)[4]) {
  if (j >= jlo && j + 3 <= jhi) {
    __stcs(reinterpret_cast<float4*>(dst + j), make_float4(o[0], o[1], o[2], o[3]));
  } else {
#pragma unroll
    for (int e = 0; e < 4; ++e)
      if (j + e >= jlo && j + e <= jhi) dst[j + e] = o[e];
  }
}

constexpr int C2_WARPS = 8;
constexpr int C2_U = 4;  // rows loaded per batch (memory parallelism)

// Work unit = (128-column chunk, strip of R output rows). Warp-granular.
__global__ void __launch_bounds__(32 * C2_WARPS) conv2d_kernel(const float* __restrict__ A, float* __restrict__ B,
                                                               int ni, int nj, int R, int nchunks, long long units,
                                                               const __grid_constant__ W9 w) {
  pdl_wait();
  const int lane = threadIdx.x & 31;
  const long long unit = (long long)blockIdx.x * C2_WARPS + (threadIdx.x >> 5);
  if (unit >= units) return;
  const int chunk = (int)(unit % nchunks);
  const int strip = (int)(unit / nchunks);
  const int c0 = chunk * 128;
  const int j = c0 + 4 * lane;
  const bool active = j < nj;
  const int o0 = 1 + strip * R;
  const int o1 = min(o0 + R, ni - 1);  // output rows [o0, o1)
  if (o0 >= o1) return;
  Row6 x0 = load_row2d(A + (size_t)(o0 - 1) * nj, c0, j, active, lane, nj);
  Row6 x1 = load_row2d(A + (size_t)o0 * nj, c0, j, active, lane, nj);
  for (int i = o0; i < o1; i += C2_U) {
    Row6 nx[C2_U];
#pragma unroll
    for (int u = 0; u < C2_U; ++u) {
      const int r = i + 1 + u;  // rows i+1 .. i+U (r <= ni-1 is in range while the output row i+u < o1)
      nx[u] = (i + u < o1) ? load_row2d(A + (size_t)r * nj, c0, j, active, lane, nj) : x1;
    }
#pragma unroll
    for (int u = 0; u < C2_U; ++u) {
      if (i + u < o1) {
        float o[4] = {0.f, 0.f, 0.f, 0.f};
        acc_row(o, x0, w.w[0], w.w[1], w.w[2]);
        acc_row(o, x1, w.w[3], w.w[4], w.w[5]);
        acc_row(o, nx[u], w.w[6], w.w[7], w.w[8]);
        if (active) store4_interior(B + (size_t)(i + u) * nj, j, 1, nj - 2, o);
      }
      x0 = x1;
      x1 = nx[u];
    }
  }
}

// ============================================================== conv3d
struct W27 {
  float w[27];
};

constexpr int C3_ROWS = 8;          // output j-rows per CTA (one warp each)
constexpr int C3_TROWS = C3_ROWS + 2;
constexpr int C3_PITCH = 136;       // floats per tile row: [0..3] pad/left halo at 3, values at 4..131, right halo 132
constexpr int C3_STAGES = 4;
constexpr int C3_TILE = C3_TROWS * C3_PITCH;

struct C3Row {
  float l, a, b, c, d, r;
};

__device__ __forceinline__ C3Row read_tile_row(const float* t, int lane) {
  const float4 v = *reinterpret_cast<const float4*>(t + 4 + 4 * lane);
  C3Row o;
  o.a = v.x; o.b = v.y; o.c = v.z; o.d = v.w;
  o.l = t[3 + 4 * lane];
  o.r = t[8 + 4 * lane];
  return o;
}

__device__ __forceinline__ void acc3(float (&o)[4], const C3Row& x, const float* w3) {
  o[0] = fmaf(w3[0], x.l, o[0]); o[0] = fmaf(w3[1], x.a, o[0]); o[0] = fmaf(w3[2], x.b, o[0]);
  o[1] = fmaf(w3[0], x.a, o[1]); o[1] = fmaf(w3[1], x.b, o[1]); o[1] = fmaf(w3[2], x.c, o[1]);
  o[2] = fmaf(w3[0], x.b, o[2]); o[2] = fmaf(w3[1], x.c, o[2]); o[2] = fmaf(w3[2], x.d, o[2]);
  o[3] = fmaf(w3[0], x.c, o[3]); o[3] = fmaf(w3[1], x.d, o[3]); o[3] = fmaf(w3[2], x.r, o[3]);
}

// Issue the bulk copies of plane q's tile into buffer `buf` (one thread). Returns bytes.
__device__ __forceinline__ void c3_issue(const float* A, float* buf, uint64_t* bar, int q, int j0, int k0, int nj,
                                         int nk) {
  // k range [ka, kb): k0-4 .. k0+132 clipped to [0, nk); lands at offset 4 + (ka - k0)
  const int ka = max(k0 - 4, 0);
  const int kb = min(k0 + 132, nk);
  const uint32_t row_bytes = (uint32_t)(kb - ka) * 4u;
  int nrows = 0;
#pragma unroll 1
  for (int r = 0; r < C3_TROWS; ++r) {
    const int jj = j0 - 1 + r;
    if (jj >= 0 && jj < nj) ++nrows;
  }
  mbar_arrive_expect_tx(bar, row_bytes * (uint32_t)nrows);
#pragma unroll 1
  for (int r = 0; r < C3_TROWS; ++r) {
    const int jj = j0 - 1 + r;
    if (jj < 0 || jj >= nj) continue;
    const float* src = A + ((size_t)q * nj + jj) * nk + ka;
    bulk_g2s(buf + r * C3_PITCH + 4 + (ka - k0), src, row_bytes, bar);
  }
}

// Work unit = (k chunk of 128, group of 8 j-rows, segment of output planes).
__global__ void __launch_bounds__(32 * C3_ROWS) conv3d_kernel(const float* __restrict__ A, float* __restrict__ B,
                                                              int ni, int nj, int nk, int seg, int nkc, int njg,
                                                              const __grid_constant__ W27 w) {
  extern __shared__ __align__(128) float c3_smem[];
  float* tiles = c3_smem;
  uint64_t* full = reinterpret_cast<uint64_t*>(c3_smem + C3_STAGES * C3_TILE);
  const int lane = threadIdx.x & 31, wp = threadIdx.x >> 5;
  const int kc = blockIdx.x % nkc;
  const int jg = (blockIdx.x / nkc) % njg;
  const int sg = blockIdx.x / (nkc * njg);
  const int k0 = kc * 128, j0 = jg * C3_ROWS;
  const int o0 = 1 + sg * seg;
  const int o1 = min(o0 + seg, ni - 1);  // output planes [o0, o1)
  if (o0 >= o1) return;
  const int q0 = o0 - 1, q1 = o1 + 1;   // planes loaded [q0, q1)
  const int nplanes = q1 - q0;
  if (threadIdx.x == 0) {
    for (int s = 0; s < C3_STAGES; ++s) mbar_init(&full[s], 1);
    fence_mbar_init();
  }
  __syncthreads();
  pdl_wait();
  if (threadIdx.x == 0) {
    for (int s = 0; s < C3_STAGES && s < nplanes; ++s)
      c3_issue(A, tiles + s * C3_TILE, &full[s], q0 + s, j0, k0, nj, nk);
  }
  const int j = j0 + wp;
  const int k = k0 + 4 * lane;
  const bool store_ok = (j >= 1 && j <= nj - 2 && k < nk);
  float am[4] = {0.f, 0.f, 0.f, 0.f}, a0[4] = {0.f, 0.f, 0.f, 0.f}, ap[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll 1
  for (int p = 0; p < nplanes; ++p) {
    const int s = p % C3_STAGES;
    mbar_wait(&full[s], (uint32_t)((p / C3_STAGES) & 1));
    const float* t = tiles + s * C3_TILE + wp * C3_PITCH;
    const C3Row r0 = read_tile_row(t, lane);
    const C3Row r1 = read_tile_row(t + C3_PITCH, lane);
    const C3Row r2 = read_tile_row(t + 2 * C3_PITCH, lane);
    // plane q = q0 + p: di = +1 for output q-1 (am), 0 for q (a0), -1 for q+1 (ap)
    acc3(am, r0, &w.w[18 + 0]); acc3(am, r1, &w.w[18 + 3]); acc3(am, r2, &w.w[18 + 6]);
    acc3(a0, r0, &w.w[9 + 0]);  acc3(a0, r1, &w.w[9 + 3]);  acc3(a0, r2, &w.w[9 + 6]);
    acc3(ap, r0, &w.w[0]);      acc3(ap, r1, &w.w[3]);      acc3(ap, r2, &w.w[6]);
    __syncthreads();  // every warp is done with buffer s
    if (threadIdx.x == 0 && p + C3_STAGES < nplanes)
      c3_issue(A, tiles + s * C3_TILE, &full[s], q0 + p + C3_STAGES, j0, k0, nj, nk);
    const int oq = q0 + p - 1;  // output plane completed by this plane
    if (p >= 2 && store_ok) store4_interior(B + ((size_t)oq * nj + j) * nk, k, 1, nk - 2, am);
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      am[e] = a0[e];
      a0[e] = ap[e];
      ap[e] = 0.f;
    }
  }
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

}  // namespace

cudaError_t launch_conv2d(const float* A, float* B, int ni, int nj, const float* w9, cudaStream_t s, int* launches) {
  if (ni < 3 || nj < 3) return cudaSuccess;  // no interior
  W9 w;
  for (int e = 0; e < 9; ++e) w.w[e] = w9[e];
  const int nchunks = (nj + 127) / 128;
  const int interior = ni - 2;
  // strips so that the warp units fill the resident warps about once
  static int per_sm = 0;  // resident CTAs per SM (same on every B200)
  if (!per_sm && (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, conv2d_kernel, 32 * C2_WARPS, 0) !=
                      cudaSuccess || per_sm <= 0))
    per_sm = 4;
  const long long resident = (long long)sm_count() * per_sm * C2_WARPS;
  long long strips = (resident + nchunks - 1) / nchunks;
  if (strips > interior) strips = interior;
  int R = (int)((interior + strips - 1) / strips);
  R = (R + C2_U - 1) / C2_U * C2_U;
  strips = (interior + R - 1) / R;
  const long long units = strips * nchunks;
  const unsigned grid = (unsigned)((units + C2_WARPS - 1) / C2_WARPS);
  ++*launches;
  return launch_pdl(conv2d_kernel, dim3(grid), dim3(32 * C2_WARPS), 0, s, A, B, ni, nj, R, nchunks, units, w);
}

cudaError_t launch_conv3d(const float* A, float* B, int ni, int nj, int nk, const float* w27, cudaStream_t s,
                          int* launches) {
  if (ni < 3 || nj < 3 || nk < 3) return cudaSuccess;
  W27 w;
  for (int e = 0; e < 27; ++e) w.w[e] = w27[e];
  const size_t smem = (size_t)C3_STAGES * C3_TILE * sizeof(float) + C3_STAGES * sizeof(uint64_t);
  cudaError_t e = ensure_smem<conv3d_kernel>(smem);
  if (e != cudaSuccess) return e;
  const int nkc = (nk + 127) / 128;
  const int njg = (nj + C3_ROWS - 1) / C3_ROWS;
  const long long tiles = (long long)nkc * njg;
  const int interior = ni - 2;
  // segments of the i march: enough CTAs for ~4 waves
  static int per_sm = 0;
  if (!per_sm && (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, conv3d_kernel, 32 * C3_ROWS, smem) !=
                      cudaSuccess || per_sm <= 0))
    per_sm = 4;
  const long long want = (long long)sm_count() * per_sm * 4;
  long long nseg = (want + tiles - 1) / tiles;
  if (nseg > interior) nseg = interior;
  if (nseg < 1) nseg = 1;
  const int seg = (int)((interior + nseg - 1) / nseg);
  nseg = (interior + seg - 1) / seg;
  const long long grid = tiles * nseg;
  ++*launches;
  return launch_pdl(conv3d_kernel, dim3((unsigned)grid), dim3(32 * C3_ROWS), smem, s, A, B, ni, nj, nk, seg, nkc,
                    njg, w);
}

size_t fdtd_ws_bytes(int nx, int ny) { return 3 * align_up((size_t)nx * ny * sizeof(float), 256); }

cudaError_t launch_fdtd2d(int tmax, int nx, int ny, float* ex, float* ey, float* hz, const float* fict, void* ws,
                          cudaStream_t s, int* launches) {
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
