// pb_band_prep.cuh — the banded single-pass covariance/correlation prep as a
// device function (used by the standalone kernel in k_stats.cu and by the fused
// Gram kernel in k_umma.cu). Product code; reading R18.
//
// Block (column block cb of 64 columns, row band b of <= 256 rows), 256 threads:
// the band is held in registers, its column means (and M2 for correlation) are
// computed exactly in fp64, written per band, and the band-centred values are
// written split (hi/lo) and transposed (m x ldo, K-major for the Gram core).
#pragma once
#include "pb_device.cuh"

namespace pb {

constexpr int BAND = 256, BCOLS = 64, BT = 256, BB = 4;

struct BandScratch {
  double red[BT / 16][BCOLS];
  double mu[BCOLS];
};

// Sync: struct with `static void run()` synchronising the 256 participating threads.
struct CtaSync {
  __device__ static void run() { __syncthreads(); }
};
struct NamedSync256 {  // barrier 2 over threads 0..255 (the rest of the CTA does not take part)
  __device__ static void run() { asm volatile("bar.sync 2, 256;" ::: "memory"); }
};

// Padded row stride (floats) of the band tile staged in shared memory: the
// column-wise reads below then hit distinct banks (2-way at worst).
constexpr int TS = BCOLS + 1;
constexpr size_t BAND_TILE_BYTES = (size_t)BAND * TS * sizeof(float);

template <bool CORR, class Sync>
__device__ __forceinline__ void band_prep_block(const float* __restrict__ data, int n, int m, float* __restrict__ hiT,
                                                float* __restrict__ loT, int ldo, double* __restrict__ band_mean,
                                                double* __restrict__ band_m2, int cb, int b, int t, BandScratch& sc,
                                                float* __restrict__ tile, unsigned long long* phase = nullptr) {
  const int c0 = cb * BCOLS;
  const int r_begin = b * BAND, r_end = min(r_begin + BAND, n);
  const double nb = (double)(r_end - r_begin);
  {  // coalesced loads: a warp reads 2 rows x 256 B per instruction, staged into the padded tile
    const int cql = t & 15, rs = t >> 4;
    const int cc = c0 + 4 * cql;
    float4 v[BAND / 16];
#pragma unroll
    for (int i = 0; i < BAND / 16; ++i) {
      const int r = r_begin + rs + 16 * i;
      v[i] = (cc < m && r < r_end) ? *reinterpret_cast<const float4*>(data + (long long)r * m + cc)
                                   : make_float4(0.f, 0.f, 0.f, 0.f);
    }
#pragma unroll
    for (int i = 0; i < BAND / 16; ++i) {
      float* tp = tile + (rs + 16 * i) * TS + 4 * cql;
      tp[0] = v[i].x; tp[1] = v[i].y; tp[2] = v[i].z; tp[3] = v[i].w;
    }
  }
  Sync::run();
  const int rq0 = t & 15, cq = t >> 4;  // lanes on row quads: coalesced transposed stores
  const int c = c0 + 4 * cq;
  // this thread's 4x4 blocks are read from the tile in each pass (no register copy:
  // keeps the kernel free of spills, correlation's second pass included)
  auto x = [&](int k, int u, int v) -> float { return tile[(4 * (rq0 + 16 * k) + u) * TS + 4 * cq + v]; };
  {
    double sv[4] = {0, 0, 0, 0};
#pragma unroll
    for (int k = 0; k < BB; ++k)
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int v = 0; v < 4; ++v) sv[v] += (double)x(k, u, v);
#pragma unroll
    for (int v = 0; v < 4; ++v) sc.red[rq0][4 * cq + v] = sv[v];
  }
  if (phase && t == 0) phase[1] = gtimer_ns();  // thread 0's loads arrived
  Sync::run();
  if (t < BCOLS) {
    double S = 0.0;
    for (int k = 0; k < BT / 16; ++k) S += sc.red[k][t];
    const double mu = S / nb;
    sc.mu[t] = mu;
    if (c0 + t < m) band_mean[(long long)b * m + c0 + t] = mu;
  }
  Sync::run();
  double mu[4];
#pragma unroll
  for (int v = 0; v < 4; ++v) mu[v] = sc.mu[4 * cq + v];
  if (CORR) {  // M2_b = sum (x - mu_b)^2, second pass over the tile
    double qv[4] = {0, 0, 0, 0};
#pragma unroll
    for (int k = 0; k < BB; ++k) {
      const int r = r_begin + 4 * (rq0 + 16 * k);
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int v = 0; v < 4; ++v)
          if (r + u < r_end) {
            const double d = (double)x(k, u, v) - mu[v];
            qv[v] += d * d;
          }
    }
    Sync::run();
#pragma unroll
    for (int v = 0; v < 4; ++v) sc.red[rq0][4 * cq + v] = qv[v];
    Sync::run();
    if (t < BCOLS && c0 + t < m) {
      double Q = 0.0;
      for (int k = 0; k < BT / 16; ++k) Q += sc.red[k][t];
      band_m2[(long long)b * m + c0 + t] = Q;
    }
  }
  if (phase && t == 0) phase[2] = gtimer_ns();  // band statistics done
  if (c < m) {
#pragma unroll
    for (int k = 0; k < BB; ++k) {
      const int r = r_begin + 4 * (rq0 + 16 * k);
      if (r >= r_end) continue;
#pragma unroll
      for (int v = 0; v < 4; ++v) {
        float h[4], l[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const float val = (r + u < r_end) ? (float)((double)x(k, u, v) - mu[v]) : 0.f;
          split3x(val, h[u], l[u]);
        }
        const long long o = (long long)(c + v) * ldo + r;
        *reinterpret_cast<float4*>(hiT + o) = make_float4(h[0], h[1], h[2], h[3]);
        *reinterpret_cast<float4*>(loT + o) = make_float4(l[0], l[1], l[2], l[3]);
      }
    }
  }
  Sync::run();  // scratch reusable by the next block
  if (phase && t == 0) phase[3] = gtimer_ns();  // stores issued by every thread
}

}  // namespace pb
