// k_stats.cu — S10-S12 of the hot path: column means and standard
// deviations for covariance / correlation ("array reduction" opportunities,
// PAPER.md:542; detect-reduction PAPER.md:344-374: each column sum is a
// register accumulator) fused with the centring / normalisation and the TF32
// split of the Gram operand. Variance: (sum x^2 - 2 mu sum x + n mu^2) / float_n in fp64
// (reading R17 in DESIGN.md). Deterministic: every sum has a fixed order.
#include <math.h>
#include <stdio.h>

#include <algorithm>
#include <vector>

#include "pb_band_prep.cuh"
#include "pb_device.cuh"
#include "pb_internal.h"

namespace pb {
namespace {

__device__ int g_tl_on;                  // PB_TIMELINE (tuning only)
__device__ unsigned long long g_tl[2];   // band_prep: [entry, exit]
__device__ unsigned long long g_phase[1024][4];  // band_prep per CTA: entry, loads, stats, stores

// ------------------------------------------------------------------ fused prep
// Used for long columns (n > 2048; shorter ones take the banded prep below).
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
  pdl_trigger();  // dependents may start their setup once every CTA here runs
  pdl_wait();
  const int c0 = blockIdx.x * PC;
  const int t = threadIdx.x;
  // ---- pass 1: thread = (column quad cq, row lane rl); rows rl, rl + 64, ...
  {
    const int cq = t & 3, rl = t >> 2;
    const int c = c0 + 4 * cq;
    double s[4] = {0, 0, 0, 0}, q[4] = {0, 0, 0, 0};
    if (c < m) {
      constexpr int U = 8;  // rows in flight per thread
      for (int r0 = rl; r0 < n; r0 += U * (PT / 4)) {
        float4 v[U];
#pragma unroll
        for (int k = 0; k < U; ++k) {
          const int r = r0 + k * (PT / 4);
          v[k] = r < n ? *reinterpret_cast<const float4*>(data + (long long)r * m + c) : make_float4(0.f, 0.f, 0.f, 0.f);
        }
#pragma unroll
        for (int k = 0; k < U; ++k) {
          const double a = v[k].x, b = v[k].y, cc = v[k].z, d = v[k].w;
          s[0] += a; s[1] += b; s[2] += cc; s[3] += d;
          if (CORR) { q[0] += a * a; q[1] += b * b; q[2] += cc * cc; q[3] += d * d; }
        }
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
        // sum_i (x_i - mu)^2 = Q - 2 mu S + n mu^2 (mu = S / float_n; float_n need not be n)
        double var = (Q - 2.0 * mu * S + (double)n * mu * mu) / float_n;
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
  constexpr int B = 2;  // 4x4 blocks whose loads are in flight together
  for (int b0 = t; b0 < nblk; b0 += B * PT) {
    float x[B][4][4];  // x[block][row u][col v]
#pragma unroll
    for (int k = 0; k < B; ++k) {
      const int b = b0 + k * PT;
      const int cq = b / nrq, rq = b - cq * nrq;
      const int c = c0 + 4 * cq, r = 4 * rq;
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
        if (b < nblk && c < m && r + u < n) v = *reinterpret_cast<const float4*>(data + (long long)(r + u) * m + c);
        x[k][u][0] = v.x; x[k][u][1] = v.y; x[k][u][2] = v.z; x[k][u][3] = v.w;
      }
    }
#pragma unroll
    for (int k = 0; k < B; ++k) {
    const int b = b0 + k * PT;
    const int cq = b / nrq, rq = b - cq * nrq;
    const int c = c0 + 4 * cq, r = 4 * rq;
    if (b >= nblk || c >= m) continue;
#pragma unroll
    for (int v = 0; v < 4; ++v) {
      const double mu = mu_s[4 * cq + v], inv = inv_s[4 * cq + v];
      float h[4], l[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const float val = (r + u < n) ? (float)(((double)x[k][u][v] - mu) * inv) : 0.f;
        split3x(val, h[u], l[u]);
      }
      const long long o = (long long)(c + v) * ldo + r;
      *reinterpret_cast<float4*>(hiT + o) = make_float4(h[0], h[1], h[2], h[3]);
      *reinterpret_cast<float4*>(loT + o) = make_float4(l[0], l[1], l[2], l[3]);
    }
    }
  }
}

// ------------------------------------------------------------------ banded single-pass prep (n <= 2048)
// Standalone kernel around band_prep_block (pb_band_prep.cuh): one CTA per
// (64-column block, 256-row band). The Gram of band-centred data plus the
// between-band scatter sum_b n_b (mu_b - mu)(mu_b - mu)^T (Chan et al.) is
// exactly X_c^T X_c; gram_combine adds that term (reading R18).
template <bool CORR>
__global__ void __launch_bounds__(BT, 2)
    band_prep_kernel(const float* __restrict__ data, int n, int m, float* __restrict__ hiT, float* __restrict__ loT,
                     int ldo, double* __restrict__ band_mean, double* __restrict__ band_m2) {
  __shared__ BandScratch sc;
  extern __shared__ __align__(16) float band_tile[];  // BAND_TILE_BYTES (dynamic)
  pdl_trigger();  // dependents may start their setup once every CTA here runs
  pdl_wait();
  const int tl = g_tl_on;
  tl_enter(tl, g_tl, 0);
  const int cta = blockIdx.y * gridDim.x + blockIdx.x;
  unsigned long long* ph = (tl && cta < 1024) ? g_phase[cta] : nullptr;
  if (ph && threadIdx.x == 0) ph[0] = gtimer_ns();
  band_prep_block<CORR, CtaSync>(data, n, m, hiT, loT, ldo, band_mean, band_m2, blockIdx.x, blockIdx.y, threadIdx.x,
                                 sc, band_tile, ph);
  tl_exit(tl, g_tl, 0);
}

}  // namespace

int band_count(int n) { return (n + BAND - 1) / BAND; }

void timeline_stats(bool reset, unsigned long long* out2) {
  if (reset) {
    const int on = 1;
    const unsigned long long init[2] = {~0ull, 0ull};
    static const unsigned long long zeros[1024][4] = {};
    cudaMemcpyToSymbol(g_tl_on, &on, sizeof on);
    cudaMemcpyToSymbol(g_tl, init, sizeof init);
    cudaMemcpyToSymbol(g_phase, zeros, sizeof zeros);  // CTAs of this call only
  } else {
    cudaMemcpyFromSymbol(out2, g_tl, 2 * sizeof(unsigned long long));
    // per-CTA phase medians (tuning only)
    static unsigned long long ph[1024][4];
    cudaMemcpyFromSymbol(ph, g_phase, sizeof ph);
    std::vector<double> ld, st, sto, start;
    for (int i = 0; i < 1024; ++i) {
      if (!ph[i][0] || !ph[i][3]) continue;
      start.push_back((ph[i][0] - out2[0]) / 1e3);
      ld.push_back((ph[i][1] - ph[i][0]) / 1e3);
      st.push_back((ph[i][2] - ph[i][1]) / 1e3);
      sto.push_back((ph[i][3] - ph[i][2]) / 1e3);
    }
    auto med = [](std::vector<double> v) { if (v.empty()) return 0.0; std::sort(v.begin(), v.end()); return v[v.size() / 2]; };
    auto mx = [](std::vector<double> v) { return v.empty() ? 0.0 : *std::max_element(v.begin(), v.end()); };
    fprintf(stderr, "[pb prep phases] n=%zu start med %.1f max %.1f | loads %.1f (max %.1f) | stats %.1f | stores %.1f (max %.1f) us\n",
            ld.size(), med(start), mx(start), med(ld), mx(ld), med(st), med(sto), mx(sto));
  }
}

cudaError_t launch_band_prep(const float* data, int n, int m, bool corr, float* hiT, float* loT, int ldo,
                             double* band_mean, double* band_m2, cudaStream_t s) {
  dim3 grid((m + BCOLS - 1) / BCOLS, band_count(n));
  cudaError_t e;
  if (corr) {
    if ((e = ensure_smem<band_prep_kernel<true>>(BAND_TILE_BYTES)) != cudaSuccess) return e;
    return launch_pdl(band_prep_kernel<true>, grid, dim3(BT), BAND_TILE_BYTES, s, data, n, m, hiT, loT, ldo,
                      band_mean, band_m2);
  }
  if ((e = ensure_smem<band_prep_kernel<false>>(BAND_TILE_BYTES)) != cudaSuccess) return e;
  return launch_pdl(band_prep_kernel<false>, grid, dim3(BT), BAND_TILE_BYTES, s, data, n, m, hiT, loT, ldo, band_mean,
                    band_m2);
}

cudaError_t launch_stats_split(const float* data, int n, int m, double float_n, double eps, bool corr, float* hiT,
                               float* loT, int ldo, float* mean_out, float* sd_out, cudaStream_t s) {
  const int grid = (m + PC - 1) / PC;
  if (corr)
    return launch_pdl(stats_split_kernel<true>, dim3(grid), dim3(PT), 0, s, data, n, m, float_n, eps, hiT, loT, ldo,
                      mean_out, sd_out);
  return launch_pdl(stats_split_kernel<false>, dim3(grid), dim3(PT), 0, s, data, n, m, float_n, eps, hiT, loT, ldo,
                    mean_out, sd_out);
}

}  // namespace pb
