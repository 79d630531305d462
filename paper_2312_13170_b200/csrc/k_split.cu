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

__global__ void __launch_bounds__(256) split_kernel(const float* __restrict__ X, int rows, int cols4, int ldx,
                                                    float* __restrict__ hi, float* __restrict__ lo, int ldo) {
  const long long total = (long long)rows * cols4;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    const long long r = e / cols4;
    const int c = (int)(e - r * cols4) * 4;
    float4 v = *reinterpret_cast<const float4*>(X + r * ldx + c);
    float4 h, l;
    split3x(v.x, h.x, l.x);
    split3x(v.y, h.y, l.y);
    split3x(v.z, h.z, l.z);
    split3x(v.w, h.w, l.w);
    *reinterpret_cast<float4*>(hi + r * ldo + c) = h;
    *reinterpret_cast<float4*>(lo + r * ldo + c) = l;
  }
}

// out[c][r] = split(f(X[r][c])) with f(x) = ((double)x - mean[c]) * inv[c] when mean != null.
__global__ void __launch_bounds__(256) split_t_kernel(const float* __restrict__ X, int rows, int cols, int ldx,
                                                      float* __restrict__ hiT, float* __restrict__ loT, int ldo,
                                                      const double* __restrict__ mean,
                                                      const double* __restrict__ inv) {
  __shared__ float tile[32][33];
  const int r0 = blockIdx.y * 32, c0 = blockIdx.x * 32;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // 8 rows of 32
  for (int k = ty; k < 32; k += 8) {
    const int r = r0 + k, c = c0 + tx;
    float v = 0.f;
    if (r < rows && c < cols) {
      v = X[(long long)r * ldx + c];
      if (mean) {
        double d = (double)v - mean[c];
        if (inv) d *= inv[c];
        v = (float)d;
      }
    }
    tile[k][tx] = v;
  }
  __syncthreads();
  for (int k = ty; k < 32; k += 8) {
    const int c = c0 + k, r = r0 + tx;  // output row c, output col r
    if (c < cols && r < rows) {
      float h, l;
      split3x(tile[tx][k], h, l);
      hiT[(long long)c * ldo + r] = h;
      loT[(long long)c * ldo + r] = l;
    }
  }
}

}  // namespace

cudaError_t launch_split(const float* X, int rows, int cols, int ldx, float* hi, float* lo, int ldo,
                         cudaStream_t s) {
  const int cols4 = cols / 4;  // cols % 4 == 0 validated by the ABI
  long long total = (long long)rows * cols4;
  long long blocks = (total + 255) / 256;
  if (blocks > 148 * 16) blocks = 148 * 16;
  if (blocks < 1) blocks = 1;
  split_kernel<<<(unsigned)blocks, 256, 0, s>>>(X, rows, cols4, ldx, hi, lo, ldo);
  return cudaGetLastError();
}

cudaError_t launch_split_T(const float* X, int rows, int cols, int ldx, float* hiT, float* loT, int ldo,
                           const double* mean, const double* inv, cudaStream_t s) {
  dim3 grid((cols + 31) / 32, (rows + 31) / 32);
  split_t_kernel<<<grid, 256, 0, s>>>(X, rows, cols, ldx, hiT, loT, ldo, mean, inv);
  return cudaGetLastError();
}

}  // namespace pb
