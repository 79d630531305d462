// k_stats.cu — S10/S11 of the hot path: column means and standard
// deviations for covariance / correlation ("array reduction" opportunities,
// PAPER.md:542; detect-reduction PAPER.md:344-374: each column sum is a
// register accumulator, written once per row chunk).
//
// Pass  : part[rc][j] = (sum_{i in chunk rc} x[i][j], sum x^2)   fp64, one read of data
//         (thread = 4 adjacent columns, float4 loads, whole chunk unrolled)
// Final : one warp per column: lane c sums chunks c, c+32, ... then a fixed
//         butterfly -> mean[j] = S/float_n;
//         var[j] = (Q - S*S/float_n)/float_n  (fp64; reading R17 in DESIGN.md)
//         sd[j] = sqrt(var); sd <= eps -> 1 (reading R5); inv[j] = 1/(sqrt(float_n)*sd)
// Deterministic (no atomics): every sum has a fixed order.
#include <math.h>

#include "pb_device.cuh"
#include "pb_internal.h"

namespace pb {
namespace {

constexpr int RC = 16;    // rows per chunk (all loads of a chunk in flight together)
constexpr int TPB = 256;  // threads per CTA; 4 columns each -> 1024 columns per CTA

template <bool SQ>
__global__ void __launch_bounds__(TPB) colsum_kernel(const float* __restrict__ data, int n, int m,
                                                     double* __restrict__ psum, double* __restrict__ psq) {
  const int j = (blockIdx.x * TPB + threadIdx.x) * 4;
  const int r0 = blockIdx.y * RC;
  if (j >= m) return;
  const int r1 = min(r0 + RC, n);
  float4 v[RC];
#pragma unroll
  for (int k = 0; k < RC; ++k)
    v[k] = (r0 + k < r1) ? *reinterpret_cast<const float4*>(data + (long long)(r0 + k) * m + j)
                         : make_float4(0.f, 0.f, 0.f, 0.f);
  double s[4] = {0, 0, 0, 0}, q[4] = {0, 0, 0, 0};
#pragma unroll
  for (int k = 0; k < RC; ++k) {
    const double a = v[k].x, b = v[k].y, c = v[k].z, d = v[k].w;
    s[0] += a; s[1] += b; s[2] += c; s[3] += d;
    if (SQ) { q[0] += a * a; q[1] += b * b; q[2] += c * c; q[3] += d * d; }
  }
  double* ps = psum + (long long)blockIdx.y * m + j;
#pragma unroll
  for (int u = 0; u < 4; ++u) ps[u] = s[u];
  if (SQ) {
    double* pq = psq + (long long)blockIdx.y * m + j;
#pragma unroll
    for (int u = 0; u < 4; ++u) pq[u] = q[u];
  }
}

template <bool SQ>
__global__ void __launch_bounds__(256) finalize_kernel(const double* __restrict__ psum, const double* __restrict__ psq,
                                                       int nchunks, int m, double float_n, double eps,
                                                       double* __restrict__ mean, double* __restrict__ inv,
                                                       float* __restrict__ mean_out, float* __restrict__ sd_out) {
  const int j = blockIdx.x * 8 + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (j >= m) return;
  double s = 0.0, q = 0.0;
  for (int c = lane; c < nchunks; c += 32) {
    s += psum[(long long)c * m + j];
    if (SQ) q += psq[(long long)c * m + j];
  }
  s = warp_sum_d(s);
  if (SQ) q = warp_sum_d(q);
  if (lane == 0) {
    const double mu = s / float_n;
    mean[j] = mu;
    if (mean_out) mean_out[j] = (float)mu;
    if (SQ) {
      double var = (q - s * mu) / float_n;
      if (var < 0.0) var = 0.0;
      double sd = sqrt(var);
      if (sd <= eps) sd = 1.0;
      inv[j] = 1.0 / (sqrt(float_n) * sd);
      if (sd_out) sd_out[j] = (float)sd;
    }
  }
}

}  // namespace

size_t stats_part_doubles(int m, int n) { return 2 * (size_t)((n + RC - 1) / RC) * (size_t)m; }

cudaError_t launch_colstats(const float* data, int n, int m, double float_n, double eps, bool want_sd,
                            double* part, double* mean, double* inv, float* mean_out, float* sd_out,
                            cudaStream_t s, int* launches) {
  const int nchunks = (n + RC - 1) / RC;
  double* psum = part;
  double* psq = part + (size_t)nchunks * m;
  dim3 grid((m / 4 + TPB - 1) / TPB, nchunks);
  dim3 fgrid((m + 7) / 8);
  if (want_sd) {
    colsum_kernel<true><<<grid, TPB, 0, s>>>(data, n, m, psum, psq);
    finalize_kernel<true><<<fgrid, 256, 0, s>>>(psum, psq, nchunks, m, float_n, eps, mean, inv, mean_out, sd_out);
  } else {
    colsum_kernel<false><<<grid, TPB, 0, s>>>(data, n, m, psum, psq);
    finalize_kernel<false><<<fgrid, 256, 0, s>>>(psum, psq, nchunks, m, float_n, eps, mean, inv, mean_out, sd_out);
  }
  *launches += 2;
  return cudaGetLastError();
}

}  // namespace pb
