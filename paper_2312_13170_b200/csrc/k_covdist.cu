// k_covdist.cu — the device steps of covariance / correlation with the OBSERVATIONS
// split over ranks (pb_covariance_dist / pb_correlation_dist in pb_dist.cu; SURVEY.md
// §8(e) and S17, BASELINE north_star: "an allreduce of column sums for
// covariance/correlation"). Definitions: the PolyBench/C 4.2 kernel_covariance /
// kernel_correlation statements (readings R4-R6, R17 in DESIGN.md),
// whose column sums are the "array reduction" opportunities of PAPER.md:542 §VIII.
//
// Rank g holds observations [o0, o1) of data (n_g x m). The column statistics need
// every observation, the Gram only a sum over observations, so:
//   1. obs_sums_kernel: this rank's fp64 column sums S1 = sum x and S2 = sum x^2;
//   2. (pb_dist.cu) all-gather of every rank's (S1, S2) rows: an allreduce of the column
//      sums done as a gather + a fixed rank-order sum, so every rank holds bitwise the
//      same totals;
//   3. obs_center_t_kernel: totals -> mean = S1 / float_n, variance (S2 - 2 mean S1 +
//      n mean^2) / float_n in fp64 (the single-GPU exact path's formula, R17), the eps
//      rule, then Yt[j][k] = ((double)x[k][j] - mean_j) * inv_j rounded to fp32, written
//      transposed (m x ldy, K-major for the Gram; zero for k >= n_g), inv_j = 1 /
//      (sqrt(float_n) sd_j) for correlation, else 1;
//   4. (pb_dist.cu) P_g = Yt Yt^T through pb_syrk_full (3xTF32 tcgen05 GEMM, full square);
//   5. (pb_dist.cu) reduce-scatter of P = sum_g P_g into the output row bands;
//   6. obs_finish_kernel: cov = P / (float_n - 1); corr: diag := 1.
#include "pb_device.cuh"
#include "pb_internal.h"

namespace pb {
namespace {

constexpr int OC = 16;   // columns per CTA (obs_sums_kernel)
constexpr int OT = 256;  // threads per CTA

// S1[j], S2[j] (out[0..m), out[m..2m)) over the rows of X (nl x m, pitch m). Thread (column
// quad cq, row lane rl) sums rows rl, rl + 64, ... in fp64; the 64 lanes are then added in
// lane order: a fixed order, bitwise reproducible.
__global__ void __launch_bounds__(OT) obs_sums_kernel(const float* __restrict__ X, int nl, int m,
                                                     double* __restrict__ out) {
  __shared__ double rs[OT / 4][OC], rq[OT / 4][OC];
  const int t = threadIdx.x, cq = t & 3, rl = t >> 2;
  const int c = blockIdx.x * OC + 4 * cq;
  double s[4] = {0, 0, 0, 0}, q[4] = {0, 0, 0, 0};
  if (c < m) {
    constexpr int U = 4;  // rows in flight per thread
    for (int r0 = rl; r0 < nl; r0 += U * (OT / 4)) {
      float4 v[U];
#pragma unroll
      for (int k = 0; k < U; ++k) {
        const int r = r0 + k * (OT / 4);
        v[k] = r < nl ? __ldg(reinterpret_cast<const float4*>(X + (long long)r * m + c)) : make_float4(0.f, 0.f, 0.f, 0.f);
      }
#pragma unroll
      for (int k = 0; k < U; ++k) {
        const double a[4] = {v[k].x, v[k].y, v[k].z, v[k].w};
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          s[e] += a[e];
          q[e] = fma(a[e], a[e], q[e]);
        }
      }
    }
  }
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    rs[rl][4 * cq + e] = s[e];
    rq[rl][4 * cq + e] = q[e];
  }
  __syncthreads();
  if (t < OC && blockIdx.x * OC + t < m) {
    double S = 0.0, Q = 0.0;
    for (int i = 0; i < OT / 4; ++i) {
      S += rs[i][t];
      Q += rq[i][t];
    }
    out[blockIdx.x * OC + t] = S;
    out[m + blockIdx.x * OC + t] = Q;
  }
}

// Column statistics from every rank's sums (sums[g][0..m) = S1, sums[g][m..2m) = S2, g in
// rank order), then the centred (and, for correlation, normalised) transposed block.
// CTA = 32 columns x 32 local rows; blockIdx.y == 0 CTAs also write mean / sd.
template <bool CORR>
__global__ void __launch_bounds__(256) obs_center_t_kernel(const float* __restrict__ X, int nl, int m,
                                                          const double* __restrict__ sums, int nranks, int n,
                                                          double float_n, double eps, float* __restrict__ Yt,
                                                          int ldy, float* __restrict__ mean_out,
                                                          float* __restrict__ sd_out) {
  __shared__ double mu[32], inv[32];
  __shared__ float tile[32][33];
  const int c0 = blockIdx.x * 32, k0 = blockIdx.y * 32;
  const int t = threadIdx.x;
  if (t < 32) {
    const int j = c0 + t;
    double S1 = 0.0, S2 = 0.0;
    if (j < m)
      for (int g = 0; g < nranks; ++g) {
        S1 += sums[(long long)g * 2 * m + j];
        S2 += sums[(long long)g * 2 * m + m + j];
      }
    const double mean = S1 / float_n;
    double iv = 1.0, sd = 0.0;
    if (CORR) {  // sum (x - mean)^2 = S2 - 2 mean S1 + n mean^2 (float_n need not be n)
      const double var = (S2 - 2.0 * mean * S1 + (double)n * mean * mean) / float_n;
      sd = sqrt(var > 0.0 ? var : 0.0);
      if (sd <= eps) sd = 1.0;
      iv = 1.0 / (sqrt(float_n) * sd);
    }
    mu[t] = mean;
    inv[t] = iv;
    if (blockIdx.y == 0 && j < m) {
      if (mean_out) mean_out[j] = (float)mean;
      if (CORR && sd_out) sd_out[j] = (float)sd;
    }
  }
  __syncthreads();
  // load 32 rows x 32 columns (coalesced along columns), store transposed (coalesced along k)
  const int tx = t & 31, ty = t >> 5;  // 8 row groups
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int k = k0 + ty + 8 * i, j = c0 + tx;
    float v = 0.f;
    if (k < nl && j < m) v = (float)(((double)X[(long long)k * m + j] - mu[tx]) * inv[tx]);
    tile[ty + 8 * i][tx] = v;
  }
  __syncthreads();
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int j = c0 + ty + 8 * i, k = k0 + tx;
    if (j < m && k < ldy) Yt[(long long)j * ldy + k] = tile[tx][ty + 8 * i];
  }
}

// Output row band (rows [r0, r0 + rows) of the m x m result, in place): covariance
// scales by 1 / (float_n - 1); correlation sets the band's diagonal entries to exactly 1 (R6).
__global__ void __launch_bounds__(256) obs_scale_kernel(float* __restrict__ out, long long total, float alpha) {
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (long long)gridDim.x * blockDim.x)
    out[e] *= alpha;
}
__global__ void __launch_bounds__(256) obs_diag_kernel(float* __restrict__ out, int rows, int m, int r0) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < rows && r0 + i < m) out[(long long)i * m + r0 + i] = 1.0f;
}

}  // namespace

cudaError_t launch_obs_sums(const float* X, int nl, int m, double* out, cudaStream_t s) {
  obs_sums_kernel<<<(m + OC - 1) / OC, OT, 0, s>>>(X, nl, m, out);
  return cudaGetLastError();
}

cudaError_t launch_obs_center_t(bool corr, const float* X, int nl, int m, const double* sums, int nranks, int n,
                                double float_n, double eps, float* Yt, int ldy, float* mean, float* sd, cudaStream_t s) {
  const dim3 grid((m + 31) / 32, ldy > 0 ? (ldy + 31) / 32 : 1);
  if (corr)
    obs_center_t_kernel<true><<<grid, 256, 0, s>>>(X, nl, m, sums, nranks, n, float_n, eps, Yt, ldy, mean, sd);
  else
    obs_center_t_kernel<false><<<grid, 256, 0, s>>>(X, nl, m, sums, nranks, n, float_n, eps, Yt, ldy, mean, sd);
  return cudaGetLastError();
}

cudaError_t launch_obs_finish(bool corr, float* out, int rows, int m, int r0, float alpha, cudaStream_t s) {
  if (rows <= 0) return cudaSuccess;
  if (corr) {
    obs_diag_kernel<<<(rows + 255) / 256, 256, 0, s>>>(out, rows, m, r0);
  } else {
    const long long total = (long long)rows * m;
    const int grid = (int)((total + 255) / 256 < 148LL * 8 ? (total + 255) / 256 : 148LL * 8);
    obs_scale_kernel<<<grid, 256, 0, s>>>(out, total, alpha);
  }
  return cudaGetLastError();
}

}  // namespace pb
