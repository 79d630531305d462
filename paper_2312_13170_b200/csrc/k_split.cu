// k_split.cu — S1/S12 of the hot path: fp32 -> (hi, lo) TF32 split
// of a contraction operand, written K-major for the tcgen05 GEMM, optionally
// transposed and optionally centred/normalised (covariance / correlation).
//
// Memory-bound: one read of X (4 B/elem) and two writes (8 B/elem). The plain
// split streams float4; the transposed split stages a 32x32 tile through
// shared memory (padded, conflict-free) so both the read and the write are
// coalesced 128-byte rows.
#include "pb_device.cuh"
#include "pb_internal.h"

namespace pb {
namespace {

// Threads along the columns (float4 c4 = blockIdx.x * 256 + tid), CTAs step over rows
// SPLIT_U at a time: SPLIT_U independent float4 loads in flight per thread, no index
// division, coalesced 4 KiB row segments per CTA.
constexpr int SPLIT_U = 4;
// done != nullptr: every CTA adds 1 (release) when its stores are complete: a chained GEMM
// running concurrently on another stream acquires the count instead of a stream dependency.
// (<= 42 registers: a CTA fits beside a resident chain CTA on the same SM, see launch_umma_chain.)
__device__ __forceinline__ void signal_done(unsigned* done) {
  if (!done) return;
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(done) : "memory");
  }
}

__global__ void __launch_bounds__(256, 6) split_kernel(const float* __restrict__ X, int rows, int cols4, int ldx,
                                                       float* __restrict__ hi, float* __restrict__ lo, int ldo,
                                                       unsigned* done) {
  pdl_trigger();  // dependents may start their setup once every CTA here runs
  pdl_wait();
  const int c4 = blockIdx.x * 256 + threadIdx.x;
  const int c = 4 * c4;
  for (int r0 = blockIdx.y * SPLIT_U; c4 < cols4 && r0 < rows; r0 += gridDim.y * SPLIT_U) {
    float4 v[SPLIT_U];
#pragma unroll
    for (int u = 0; u < SPLIT_U; ++u)
      v[u] = r0 + u < rows ? *reinterpret_cast<const float4*>(X + (long long)(r0 + u) * ldx + c)
                           : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
    for (int u = 0; u < SPLIT_U; ++u) {
      if (r0 + u >= rows) break;
      float4 h, l;
      split3x(v[u].x, h.x, l.x);
      split3x(v[u].y, h.y, l.y);
      split3x(v[u].z, h.z, l.z);
      split3x(v[u].w, h.w, l.w);
      const long long o = (long long)(r0 + u) * ldo + c;
      *reinterpret_cast<float4*>(hi + o) = h;
      *reinterpret_cast<float4*>(lo + o) = l;
    }
  }
  signal_done(done);
}

// lo only (raw-hi split): lo[r][c] = lo_of_raw(X[r][c]); the GEMM reads X itself as hi.
__global__ void __launch_bounds__(256, 6) split_lo_kernel(const float* __restrict__ X, int rows, int cols4, int ldx,
                                                          float* __restrict__ lo, int ldo) {
  pdl_trigger();  // dependents may start their setup once every CTA here runs
  pdl_wait();
  const int c4 = blockIdx.x * 256 + threadIdx.x;
  const int c = 4 * c4;
  for (int r0 = blockIdx.y * SPLIT_U; c4 < cols4 && r0 < rows; r0 += gridDim.y * SPLIT_U) {
    float4 v[SPLIT_U];
#pragma unroll
    for (int u = 0; u < SPLIT_U; ++u)
      v[u] = r0 + u < rows ? *reinterpret_cast<const float4*>(X + (long long)(r0 + u) * ldx + c)
                           : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
    for (int u = 0; u < SPLIT_U; ++u) {
      if (r0 + u >= rows) break;
      const float4 l = make_float4(lo_of_raw(v[u].x), lo_of_raw(v[u].y), lo_of_raw(v[u].z), lo_of_raw(v[u].w));
      *reinterpret_cast<float4*>(lo + (long long)(r0 + u) * ldo + c) = l;
    }
  }
}

// out[c][r] = split(f(X[r][c])) with f(x) = ((double)x - mean[c]) * inv[c] when mean != null.
// 64 x 64 tile per CTA: float4 loads of X rows, padded smem transpose, float4
// stores of the hi / lo rows (output pitch ldo is a multiple of 4).
__global__ void __launch_bounds__(256, 6) split_t_kernel(const float* __restrict__ X, int rows, int cols, int ldx,
                                                         float* __restrict__ hiT, float* __restrict__ loT, int ldo,
                                                         const double* __restrict__ mean,
                                                         const double* __restrict__ inv, unsigned* done) {
  __shared__ float tile[64][65];
  pdl_trigger();  // dependents may start their setup once every CTA here runs
  pdl_wait();
  const int r0 = blockIdx.y * 64, c0 = blockIdx.x * 64;
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  const int c = c0 + 4 * tx;
  double mu[4] = {0, 0, 0, 0}, sc[4] = {1, 1, 1, 1};
  if (mean && c < cols) {
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      mu[u] = mean[c + u];
      if (inv) sc[u] = inv[c + u];
    }
  }
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const int rl = ty + 16 * k, r = r0 + rl;
    float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
    if (r < rows && c < cols) {
      v = *reinterpret_cast<const float4*>(X + (long long)r * ldx + c);
      if (mean) {
        v.x = (float)(((double)v.x - mu[0]) * sc[0]);
        v.y = (float)(((double)v.y - mu[1]) * sc[1]);
        v.z = (float)(((double)v.z - mu[2]) * sc[2]);
        v.w = (float)(((double)v.w - mu[3]) * sc[3]);
      }
    }
    tile[rl][4 * tx + 0] = v.x;
    tile[rl][4 * tx + 1] = v.y;
    tile[rl][4 * tx + 2] = v.z;
    tile[rl][4 * tx + 3] = v.w;
  }
  __syncthreads();
  const int r = r0 + 4 * tx;  // first of 4 output columns (input rows) of this thread
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const int cl = ty + 16 * k;  // output row within the tile (input column)
    if (c0 + cl < cols && r < rows) {
      float4 h, l;
      split3x(tile[4 * tx + 0][cl], h.x, l.x);
      split3x(tile[4 * tx + 1][cl], h.y, l.y);
      split3x(tile[4 * tx + 2][cl], h.z, l.z);
      split3x(tile[4 * tx + 3][cl], h.w, l.w);
      *reinterpret_cast<float4*>(hiT + (long long)(c0 + cl) * ldo + r) = h;
      *reinterpret_cast<float4*>(loT + (long long)(c0 + cl) * ldo + r) = l;
    }
  }
  signal_done(done);
}

}  // namespace

cudaError_t launch_split(const float* X, int rows, int cols, int ldx, float* hi, float* lo, int ldo,
                         cudaStream_t s, unsigned* done, unsigned* ctas) {
  const int cols4 = cols / 4;  // cols % 4 == 0 validated by the ABI
  const int gx = (cols4 + 255) / 256;
  const int row_steps = (rows + SPLIT_U - 1) / SPLIT_U;
  int gy = (148 * 8 + gx - 1) / gx;  // ~8 CTAs per SM in total
  if (gy > row_steps) gy = row_steps;
  if (gy > 65535) gy = 65535;
  if (gy < 1) gy = 1;
  if (ctas) *ctas += (unsigned)(gx * gy);
  return launch_pdl(split_kernel, dim3((unsigned)gx, (unsigned)gy), dim3(256), 0, s, X, rows, cols4, ldx, hi, lo, ldo,
                    done);
}

cudaError_t launch_split_lo(const float* X, int rows, int cols, int ldx, float* lo, int ldo, cudaStream_t s) {
  const int cols4 = cols / 4;
  const int gx = (cols4 + 255) / 256;
  const int row_steps = (rows + SPLIT_U - 1) / SPLIT_U;
  int gy = (148 * 8 + gx - 1) / gx;
  if (gy > row_steps) gy = row_steps;
  if (gy > 65535) gy = 65535;
  if (gy < 1) gy = 1;
  return launch_pdl(split_lo_kernel, dim3((unsigned)gx, (unsigned)gy), dim3(256), 0, s, X, rows, cols4, ldx, lo, ldo);
}

cudaError_t launch_split_T(const float* X, int rows, int cols, int ldx, float* hiT, float* loT, int ldo,
                           const double* mean, const double* inv, cudaStream_t s, unsigned* done, unsigned* ctas) {
  dim3 grid((cols + 63) / 64, (rows + 63) / 64);
  if (ctas) *ctas += grid.x * grid.y;
  return launch_pdl(split_t_kernel, grid, dim3(256), 0, s, X, rows, cols, ldx, hiT, loT, ldo, mean, inv, done);
}

}  // namespace pb
