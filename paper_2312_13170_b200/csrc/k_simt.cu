// k_simt.cu — the paper's own GEMM kernel shapes, recompiled for sm_100a as
// plain fp32 SIMT code (ablation baseline):
//   variant 0 = PAPER.md Listing 8: one work-item per C[i][j],
//               k-loop reading A and B from global memory, C updated in place
//               every iteration (PolyBench: C *= beta first).
//   variant 1 = PAPER.md Listing 9: the same loop after loop
//               internalization — M x M local tiles of A and B (M = 16), two group
//               barriers per tile step; C still updated in global memory.
//   variant 2 = Listing 9 + detect-reduction (Listing 5): the
//               C[i][j] running sum kept in a register, stored once.
// These are what the paper's transformations produce; the production path is
// the tcgen05 3xTF32 kernel (k_umma.cu). Variants 0 and 1 preserve the k order
// of the definition, so they are bitwise equal to each other.
#include "pb_device.cuh"
#include "pb_internal.h"

namespace pb {
namespace {

constexpr int M = 16;

__global__ void listing8_kernel(int ni, int nj, int nk, float alpha, float beta, float* C,
                                const float* __restrict__ A, const float* __restrict__ B) {
  const int i = blockIdx.y * M + threadIdx.y, j = blockIdx.x * M + threadIdx.x;
  if (i >= ni || j >= nj) return;
  volatile float* c = C + (long long)i * nj + j;  // global RMW every iteration, as written
  *c = *c * beta;
  for (int k = 0; k < nk; ++k) *c = *c + alpha * A[(long long)i * nk + k] * B[(long long)k * nj + j];
}

template <bool REG_ACC>
__global__ void listing9_kernel(int ni, int nj, int nk, float alpha, float beta, float* C,
                                const float* __restrict__ A, const float* __restrict__ B) {
  __shared__ float A_tile[M][M];
  __shared__ float B_tile[M][M];
  const int x = threadIdx.y, y = threadIdx.x;  // local ids (row, col)
  const int i = blockIdx.y * M + x, j = blockIdx.x * M + y;
  const bool ok = i < ni && j < nj;
  volatile float* c = C + (long long)i * nj + j;
  float acc = 0.f;
  if (ok) {
    if (REG_ACC) acc = c[0] * beta; else *c = *c * beta;
  }
  for (int t = 0; t < nk; t += M) {  // uniform loop: barriers never diverge
    A_tile[x][y] = (i < ni && t + y < nk) ? A[(long long)i * nk + t + y] : 0.f;
    B_tile[x][y] = (t + x < nk && j < nj) ? B[(long long)(t + x) * nj + j] : 0.f;
    __syncthreads();
    const int kmax = min(M, nk - t);
    if (ok) {
      if (REG_ACC) {
        for (int k = 0; k < kmax; ++k) acc = acc + alpha * A_tile[x][k] * B_tile[k][y];
      } else {
        for (int k = 0; k < kmax; ++k) *c = *c + alpha * A_tile[x][k] * B_tile[k][y];
      }
    }
    __syncthreads();
  }
  if (REG_ACC && ok) *c = acc;
}

}  // namespace

cudaError_t launch_gemm_listing8(int ni, int nj, int nk, float alpha, float beta, float* C, const float* A,
                                 const float* B, cudaStream_t s) {
  dim3 grid((nj + M - 1) / M, (ni + M - 1) / M), block(M, M);
  listing8_kernel<<<grid, block, 0, s>>>(ni, nj, nk, alpha, beta, C, A, B);
  return cudaGetLastError();
}

cudaError_t launch_gemm_listing9(int ni, int nj, int nk, float alpha, float beta, float* C, const float* A,
                                 const float* B, cudaStream_t s) {
  dim3 grid((nj + M - 1) / M, (ni + M - 1) / M), block(M, M);
  listing9_kernel<false><<<grid, block, 0, s>>>(ni, nj, nk, alpha, beta, C, A, B);
  return cudaGetLastError();
}

cudaError_t launch_gemm_listing9_reg(int ni, int nj, int nk, float alpha, float beta, float* C, const float* A,
                                     const float* B, cudaStream_t s) {
  dim3 grid((nj + M - 1) / M, (ni + M - 1) / M), block(M, M);
  listing9_kernel<true><<<grid, block, 0, s>>>(ni, nj, nk, alpha, beta, C, A, B);
  return cudaGetLastError();
}

}  // namespace pb
