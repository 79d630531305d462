// k_stats.cu — S10/S11 of the hot path: column means and standard
// deviations for covariance / correlation ("array reduction" opportunities,
// PAPER.md:542; detect-reduction PAPER.md:344-374: each column sum is a
// register accumulator, written once per row chunk).
//
// Pass 1: part[rc][j] = sum_{i in chunk rc} data[i][j]       (fp64 accumulate)
// Fin 1 : mean[j] = (sum_rc part[rc][j]) / float_n             (fixed order)
// Pass 2: part[rc][j] = sum_{i in chunk} (data[i][j]-mean[j])^2
// Fin 2 : sd[j] = sqrt(sum_rc part / float_n); sd <= eps -> 1 (reading R5);
//         inv[j] = 1 / (sqrt(float_n) * sd[j])
// One thread per column, consecutive threads on consecutive columns, so every
// row access is a coalesced 1 KiB segment. Deterministic (no atomics).
#include <math.h>

#include "pb_device.cuh"
#include "pb_internal.h"

namespace pb {
namespace {

constexpr int RC = 64;   // rows per chunk
constexpr int TPB = 256; // columns per CTA

__global__ void __launch_bounds__(TPB) colsum_kernel(const float* __restrict__ data, int n, int m,
                                                     const double* __restrict__ mean, double* __restrict__ part) {
  const int j = blockIdx.x * TPB + threadIdx.x;
  const int r0 = blockIdx.y * RC;
  if (j >= m) return;
  const int r1 = min(r0 + RC, n);
  double acc = 0.0;
  if (mean == nullptr) {
#pragma unroll 8
    for (int i = r0; i < r1; ++i) acc += (double)data[(long long)i * m + j];
  } else {
    const double mu = mean[j];
#pragma unroll 8
    for (int i = r0; i < r1; ++i) {
      double d = (double)data[(long long)i * m + j] - mu;
      acc += d * d;
    }
  }
  part[(long long)blockIdx.y * m + j] = acc;
}

__global__ void __launch_bounds__(TPB) finalize_kernel(const double* __restrict__ part, int nchunks, int m,
                                                       double float_n, double eps, int stage,
                                                       double* __restrict__ mean, double* __restrict__ inv,
                                                       float* __restrict__ mean_out, float* __restrict__ sd_out) {
  const int j = blockIdx.x * TPB + threadIdx.x;
  if (j >= m) return;
  double acc = 0.0;
  for (int c = 0; c < nchunks; ++c) acc += part[(long long)c * m + j];
  if (stage == 0) {
    const double mu = acc / float_n;
    mean[j] = mu;
    if (mean_out) mean_out[j] = (float)mu;
  } else {
    double sd = sqrt(acc / float_n);
    if (sd <= eps) sd = 1.0;
    inv[j] = 1.0 / (sqrt(float_n) * sd);
    if (sd_out) sd_out[j] = (float)sd;
  }
}

}  // namespace

size_t stats_part_doubles(int m, int n) { return (size_t)((n + RC - 1) / RC) * (size_t)m; }

cudaError_t launch_colstats(const float* data, int n, int m, double float_n, double eps, bool want_sd,
                            double* part, double* mean, double* inv, float* mean_out, float* sd_out,
                            cudaStream_t s, int* launches) {
  const int nchunks = (n + RC - 1) / RC;
  dim3 grid((m + TPB - 1) / TPB, nchunks);
  dim3 fgrid((m + TPB - 1) / TPB);
  colsum_kernel<<<grid, TPB, 0, s>>>(data, n, m, nullptr, part);
  finalize_kernel<<<fgrid, TPB, 0, s>>>(part, nchunks, m, float_n, eps, 0, mean, inv, mean_out, sd_out);
  *launches += 2;
  if (want_sd) {
    colsum_kernel<<<grid, TPB, 0, s>>>(data, n, m, mean, part);
    finalize_kernel<<<fgrid, TPB, 0, s>>>(part, nchunks, m, float_n, eps, 1, mean, inv, mean_out, sd_out);
    *launches += 2;
  }
  return cudaGetLastError();
}

}  // namespace pb
