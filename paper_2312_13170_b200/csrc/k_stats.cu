// k_stats.cu — S10-S12 of the hot path: column means and standard
// deviations for covariance / correlation ("array reduction" opportunities,
// PAPER.md:542; detect-reduction PAPER.md:344-374: each column sum is a
// register accumulator) fused with the centring / normalisation and the TF32
// split of the Gram operand. Variance: (sum x^2 - (sum x) mu) / float_n in fp64
// (reading R17 in DESIGN.md). Deterministic: every sum has a fixed order.
#include <math.h>

#include "pb_device.cuh"
#include "pb_internal.h"

namespace pb {
namespace {

// ------------------------------------------------------------------ fused prep
// One CTA owns PC = 16 columns of data (n x m) and all n rows:
//  pass 1: fp64 sums (and sums of squares) of its columns -> mean, stddev (eps
//          rule), inv = 1/(sqrt(float_n)*sd) (correlation) or 1 (covariance);
//  pass 2: Xt[c][r] = split(((double)x - mean[c]) * inv[c]) written transposed
//          (m x ldo, K-major for the Gram core) from 4x4 register transposes, so
//          every store is a 16-byte piece of a contiguous Xt row.
// The CTA's 16 x n slab (128 KiB at n = 2048) is re-read in pass 2 from L1/L2.
constexpr int PC = 16;
constexpr int PT = 512;

template <bool CORR>
__global__ void __launch_bounds__(PT, 1) stats_split_kernel(const float* __restrict__ data, int n, int m, double float_n,
                                                         double eps, float* __restrict__ hiT, float* __restrict__ loT,
                                                         int ldo, float* __restrict__ mean_out,
                                                         float* __restrict__ sd_out) {
  __shared__ double red_s[PT / 4][PC], red_q[CORR ? PT / 4 : 1][PC];
  __shared__ double mu_s[PC], inv_s[PC];
  const int c0 = blockIdx.x * PC;
  const int t = threadIdx.x;
  // ---- pass 1: thread = (column quad cq, row lane rl); rows rl, rl + 64, ...
  {
    const int cq = t & 3, rl = t >> 2;
    const int c = c0 + 4 * cq;
    double s[4] = {0, 0, 0, 0}, q[4] = {0, 0, 0, 0};
    if (c < m) {
#pragma unroll 8
      for (int r = rl; r < n; r += PT / 4) {
        const float4 v = *reinterpret_cast<const float4*>(data + (long long)r * m + c);
        const double a = v.x, b = v.y, cc = v.z, d = v.w;
        s[0] += a; s[1] += b; s[2] += cc; s[3] += d;
        if (CORR) { q[0] += a * a; q[1] += b * b; q[2] += cc * cc; q[3] += d * d; }
      }
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      red_s[rl][4 * cq + u] = s[u];
      if (CORR) red_q[rl][4 * cq + u] = q[u];
    }
  }
  __syncthreads();
  if (t < PC) {  // fixed-order column reduction and the per-column statistics
    double S = 0.0, Q = 0.0;
    for (int k = 0; k < PT / 4; ++k) {
      S += red_s[k][t];
      if (CORR) Q += red_q[k][t];
    }
    const double mu = S / float_n;
    double inv = 1.0;
    if (c0 + t < m) {
      if (mean_out) mean_out[c0 + t] = (float)mu;
      if (CORR) {
        double var = (Q - S * mu) / float_n;
        if (var < 0.0) var = 0.0;
        double sd = sqrt(var);
        if (sd <= eps) sd = 1.0;
        inv = 1.0 / (sqrt(float_n) * sd);
        if (sd_out) sd_out[c0 + t] = (float)sd;
      }
    }
    mu_s[t] = mu;
    inv_s[t] = inv;
  }
  __syncthreads();
  // ---- pass 2: 4x4 blocks (4 rows x 4 columns); lanes walk consecutive row quads
  const int nrq = (n + 3) / 4;
  const int nblk = nrq * (PC / 4);
  for (int b = t; b < nblk; b += PT) {
    const int cq = b / nrq, rq = b - cq * nrq;
    const int c = c0 + 4 * cq, r = 4 * rq;
    if (c >= m) continue;
    float x[4][4];  // x[row u][col v]
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
      if (r + u < n) v = *reinterpret_cast<const float4*>(data + (long long)(r + u) * m + c);
      x[u][0] = v.x; x[u][1] = v.y; x[u][2] = v.z; x[u][3] = v.w;
    }
#pragma unroll
    for (int v = 0; v < 4; ++v) {
      const double mu = mu_s[4 * cq + v], inv = inv_s[4 * cq + v];
      float h[4], l[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const float val = (r + u < n) ? (float)(((double)x[u][v] - mu) * inv) : 0.f;
        split3x(val, h[u], l[u]);
      }
      const long long o = (long long)(c + v) * ldo + r;
      *reinterpret_cast<float4*>(hiT + o) = make_float4(h[0], h[1], h[2], h[3]);
      *reinterpret_cast<float4*>(loT + o) = make_float4(l[0], l[1], l[2], l[3]);
    }
  }
}

}  // namespace

cudaError_t launch_stats_split(const float* data, int n, int m, double float_n, double eps, bool corr, float* hiT,
                               float* loT, int ldo, float* mean_out, float* sd_out, cudaStream_t s) {
  const int grid = (m + PC - 1) / PC;
  if (corr)
    stats_split_kernel<true><<<grid, PT, 0, s>>>(data, n, m, float_n, eps, hiT, loT, ldo, mean_out, sd_out);
  else
    stats_split_kernel<false><<<grid, PT, 0, s>>>(data, n, m, float_n, eps, hiT, loT, ldo, mean_out, sd_out);
  return cudaGetLastError();
}

}  // namespace pb
