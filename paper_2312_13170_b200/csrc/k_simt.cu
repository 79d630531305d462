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

// Small-problem GEMM (pb_gemm below SMALL_GEMM_MACS, e.g. the N = 128 config, where
// a launch costs more than the math). Loop internalization with the whole K strip
// (up to KC = 128) as the local tile: one global round trip per strip instead of one
// per 16-wide tile step, all float4 loads in flight together; detect-reduction into
// four register accumulators (exact fp32 FMAs, fixed order: deterministic). C is
// read before the strip loads only when beta != 0 (BLAS convention, include/pb.h).
constexpr int ST = 16, KC = 128;

__global__ void __launch_bounds__(256) small_gemm_kernel(int ni, int nj, int nk, float alpha, float beta, float* C,
                                                         const float* __restrict__ A, const float* __restrict__ B) {
  __shared__ __align__(16) float As[ST][KC + 4];
  __shared__ __align__(16) float Bs[KC][ST];
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  const int i0 = blockIdx.y * ST, j0 = blockIdx.x * ST;
  const int i = i0 + ty, j = j0 + tx;
  const bool ok = i < ni && j < nj;
  const float cin = (ok && beta != 0.f) ? C[(long long)i * nj + j] : 0.f;
  const float4 zero = make_float4(0.f, 0.f, 0.f, 0.f);
  float acc[4] = {0.f, 0.f, 0.f, 0.f};
  for (int k0 = 0; k0 < nk; k0 += KC) {  // nk % 4 == 0 and nj % 4 == 0 (validated): whole float4s
#pragma unroll
    for (int e = threadIdx.x; e < ST * KC / 4; e += 256) {
      const int r = e / (KC / 4), c4 = e % (KC / 4);
      const int gi = i0 + r, gk = k0 + 4 * c4;
      *reinterpret_cast<float4*>(&As[r][4 * c4]) =
          (gi < ni && gk < nk) ? *reinterpret_cast<const float4*>(A + (long long)gi * nk + gk) : zero;
    }
#pragma unroll
    for (int e = threadIdx.x; e < KC * ST / 4; e += 256) {
      const int k = e / (ST / 4), c4 = e % (ST / 4);
      const int gk = k0 + k, gj = j0 + 4 * c4;
      *reinterpret_cast<float4*>(&Bs[k][4 * c4]) =
          (gk < nk && gj < nj) ? *reinterpret_cast<const float4*>(B + (long long)gk * nj + gj) : zero;
    }
    __syncthreads();
    const int kc = min(KC, nk - k0);
    for (int k = 0; k < kc; k += 4) {
#pragma unroll
      for (int u = 0; u < 4; ++u) acc[u] = fmaf(As[ty][k + u], Bs[k + u][tx], acc[u]);
    }
    __syncthreads();
  }
  if (ok) {
    const float sum = (acc[0] + acc[1]) + (acc[2] + acc[3]);
    C[(long long)i * nj + j] = beta != 0.f ? alpha * sum + beta * cin : alpha * sum;
  }
}

}  // namespace

cudaError_t launch_gemm_small(int ni, int nj, int nk, float alpha, float beta, float* C, const float* A,
                              const float* B, cudaStream_t s) {
  dim3 grid((nj + ST - 1) / ST, (ni + ST - 1) / ST);
  small_gemm_kernel<<<grid, 256, 0, s>>>(ni, nj, nk, alpha, beta, C, A, B);
  return cudaGetLastError();
}

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
