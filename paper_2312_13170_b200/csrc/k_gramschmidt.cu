// k_gramschmidt.cu — SYCL-Bench "Gramschmidt" (§VIII; the benchmark
// whose candidate loop sits in a divergent region), i.e. PolyBench/C
// 4.2 kernel_gramschmidt = modified Gram-Schmidt (reading R22 in DESIGN.md).
//
// The k loop is a chain of n dependent steps: column k must have received every
// projection q_0..q_{k-1} before q_k exists. On B200 the chain runs inside ONE
// persistent kernel, one CTA per SM (cooperative launch, so spinning is safe):
//   * column j belongs to CTA j mod G and lives in that CTA's shared memory, in
//     fp64, for the whole factorisation (the loop-internalised working set);
//   * step k: every CTA waits for q_k (an acquire on a monotone counter), reads it
//     from L2, and applies it to its columns j > k. The owner of column k+1 does
//     that column FIRST, then its norm, R[k+1][k+1] and q_{k+1}, publishes q_{k+1}
//     (release), and only then updates its other columns — so the critical path
//     per step is one column's dot + axpy + norm, not a grid barrier.
//   * q_k is kept (Qc, fp64, column-major in the workspace), so no buffer is reused
//     while a slow CTA might still read it.
// Precision: fp64 state (the fp32 data are conditioned badly enough that fp32 MGS
// would not hold 1e-4; R22); outputs rounded to fp32 once.
// Launch sequence: transpose A (row-major fp32) -> W (column-major fp64); the
// persistent kernel; transpose W -> A, Qc -> Q (row-major fp32).
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>

#include "pb_device.cuh"
#include "pb_internal.h"

namespace pb {
namespace {

constexpr int GS_THREADS = 512;
constexpr int GS_WARPS = GS_THREADS / 32;
constexpr int GS_MAXC = 16;  // owned columns handled per batch
constexpr int GS_QREG = 4;   // q elements kept in registers per thread (m <= 2048 fully)

__device__ __forceinline__ unsigned ld_acquire_u32(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_u32(unsigned* p, unsigned v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ double ld_cg_f64(const double* p) {
  double v;
  asm volatile("ld.global.cg.f64 %0, [%1];" : "=d"(v) : "l"(p));
  return v;
}

// Sum of one value per thread over the CTA; every thread gets the result.
__device__ __forceinline__ double block_sum1(double v, double* red) {
  const int lane = threadIdx.x & 31, wp = threadIdx.x >> 5;
  v = warp_sum_d(v);
  if (lane == 0) red[wp] = v;
  __syncthreads();
  double t = (lane < GS_WARPS) ? red[lane] : 0.0;
  t = warp_sum_d(t);  // every warp reduces the same GS_WARPS values in the same order
  __syncthreads();    // red may be reused
  return t;
}

// As block_sum1 with one barrier: the caller alternates buffers (red, red + GS_WARPS)
// so a buffer is rewritten only after a later barrier.
__device__ __forceinline__ double block_sum_buf(double v, double* red) {
  const int lane = threadIdx.x & 31, wp = threadIdx.x >> 5;
  v = warp_sum_d(v);
  if (lane == 0) red[wp] = v;
  __syncthreads();
  double t = (lane < GS_WARPS) ? red[lane] : 0.0;
  return warp_sum_d(t);
}

struct GsArgs {
  int m, n, cpc;  // rows, columns, columns per CTA (ceil(n / G))
  double* W;      // column-major fp64 working copy, n x m (column j at W + j*m)
  double* Qc;     // column-major fp64 q vectors, n x m
  float* R;       // row-major fp32 n x n (output)
  unsigned* ready;  // q_0..q_{ready-1} are published
  int in_smem;      // owned columns held in dynamic shared memory
};

// Wait until q_k is published (thread 0 spins, bounded: a trap instead of a hang).
__device__ __forceinline__ void wait_ready(const unsigned* ready, unsigned need) {
  if (threadIdx.x == 0) {
    unsigned long long spins = 0;
    while (ld_acquire_u32(ready) < need) {
      if (++spins > (1ull << 31)) asm volatile("trap;");
    }
  }
  __syncthreads();
}

// Column c (pointer col, length m): norm, R[k][k], q = col / rkk -> Qc[k]; publish.
__device__ void make_q(const GsArgs& a, const double* col, int k, double* red) {
  double s = 0.0;
  for (int i = threadIdx.x; i < a.m; i += GS_THREADS) s += col[i] * col[i];
  const double rkk = sqrt(block_sum1(s, red));
  double* q = a.Qc + (size_t)k * a.m;
  for (int i = threadIdx.x; i < a.m; i += GS_THREADS) q[i] = col[i] / rkk;
  if (threadIdx.x == 0) a.R[(size_t)k * a.n + k] = (float)rkk;
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    st_release_u32(a.ready, (unsigned)(k + 1));
  }
}

// q_k (this thread's rows in qr, the rest from L2) applied to NB owned columns at
// base + c*cs (c < NB), global column index j0 + c*G: dot -> CTA reduce -> R -> axpy.
template <int NB>
__device__ __forceinline__ void gs_batch(const GsArgs& a, const double (&qr)[GS_QREG], const double* q, double* base,
                                         size_t cs, int j0, int G, int k, double* red, double* rsum) {
  const int lane = threadIdx.x & 31, wp = threadIdx.x >> 5;
  const int m = a.m;
  double part[NB];
#pragma unroll
  for (int c = 0; c < NB; ++c) part[c] = 0.0;
#pragma unroll
  for (int u = 0; u < GS_QREG; ++u) {
    const int i = threadIdx.x + u * GS_THREADS;
    if (i < m) {
#pragma unroll
      for (int c = 0; c < NB; ++c) part[c] += qr[u] * base[c * cs + i];
    }
  }
  for (int i = threadIdx.x + GS_QREG * GS_THREADS; i < m; i += GS_THREADS) {
    const double qi = ld_cg_f64(q + i);
#pragma unroll
    for (int c = 0; c < NB; ++c) part[c] += qi * base[c * cs + i];
  }
#pragma unroll
  for (int c = 0; c < NB; ++c) {
    const double v = warp_sum_d(part[c]);
    if (lane == 0) red[wp * GS_MAXC + c] = v;
  }
  __syncthreads();
  if (threadIdx.x < NB) {
    double s = 0.0;
    for (int w = 0; w < GS_WARPS; ++w) s += red[w * GS_MAXC + threadIdx.x];
    rsum[threadIdx.x] = s;
    a.R[(size_t)k * a.n + (j0 + threadIdx.x * G)] = (float)s;
  }
  __syncthreads();
  double r[NB];
#pragma unroll
  for (int c = 0; c < NB; ++c) r[c] = rsum[c];
#pragma unroll
  for (int u = 0; u < GS_QREG; ++u) {
    const int i = threadIdx.x + u * GS_THREADS;
    if (i < m) {
#pragma unroll
      for (int c = 0; c < NB; ++c) base[c * cs + i] -= qr[u] * r[c];
    }
  }
  for (int i = threadIdx.x + GS_QREG * GS_THREADS; i < m; i += GS_THREADS) {
    const double qi = ld_cg_f64(q + i);
#pragma unroll
    for (int c = 0; c < NB; ++c) base[c * cs + i] -= qi * r[c];
  }
  __syncthreads();
}

__global__ void __launch_bounds__(GS_THREADS, 1) gs_kernel(GsArgs a) {
  extern __shared__ __align__(16) double gs_smem[];
  __shared__ double red[GS_WARPS * GS_MAXC];
  __shared__ double rsum[GS_MAXC];
  const int G = gridDim.x, cta = blockIdx.x;
  const int m = a.m, n = a.n;
  const int lane = threadIdx.x & 31, wp = threadIdx.x >> 5;
  // owned columns: j = cta + t*G, t < nown
  const int nown = (n - cta + G - 1) / G;
  double* cols = a.in_smem ? gs_smem : nullptr;
  auto colp = [&](int t) -> double* {
    return a.in_smem ? cols + (size_t)t * m : a.W + (size_t)(cta + t * G) * m;
  };
  pdl_wait();
  if (a.in_smem) {
    for (int t = 0; t < nown; ++t) {
      const double* src = a.W + (size_t)(cta + t * G) * m;
      double* dst = cols + (size_t)t * m;
      for (int i = threadIdx.x; i < m; i += GS_THREADS) dst[i] = src[i];
    }
    __syncthreads();
  }
  if (cta == 0) make_q(a, colp(0), 0, red);

  for (int k = 0; k < n - 1; ++k) {
    // first owned column index with j > k
    const int t0 = (k + 1 - cta + G - 1) >= 0 ? (k + 1 - cta + G - 1) / G : 0;
    if (t0 >= nown) break;  // nothing left to update here (all later steps too)
    wait_ready(a.ready, (unsigned)(k + 1));
    // q_k into registers once (one L2 round trip per step): element i = tid + u*GS_THREADS
    const double* q = a.Qc + (size_t)k * m;
    double qr[GS_QREG];
#pragma unroll
    for (int u = 0; u < GS_QREG; ++u) {
      const int i = threadIdx.x + u * GS_THREADS;
      qr[u] = i < m ? ld_cg_f64(q + i) : 0.0;
    }
    // f(i, q_i) over this thread's rows: register part unrolled, the rest (m > 2048) from L2
    auto rows = [&](auto&& f) {
#pragma unroll
      for (int u = 0; u < GS_QREG; ++u) {
        const int i = threadIdx.x + u * GS_THREADS;
        if (i < m) f(i, qr[u]);
      }
      for (int i = threadIdx.x + GS_QREG * GS_THREADS; i < m; i += GS_THREADS) f(i, ld_cg_f64(q + i));
    };
    // critical column k+1 first (if owned)
    int tb = t0;
    if (cta + t0 * G == k + 1) {
      // dot, then axpy fused with the new column's norm, then q_{k+1}: three CTA
      // barriers (the reductions use separate buffers, so none needs a second one)
      double* c = colp(t0);
      double s = 0.0;
      rows([&](int i, double qi) { s += qi * c[i]; });
      const double r = block_sum_buf(s, red);
      double s2 = 0.0;
      rows([&](int i, double qi) {
        const double v = c[i] - qi * r;
        c[i] = v;
        s2 += v * v;
      });
      const double rkk = sqrt(block_sum_buf(s2, red + GS_WARPS));
      double* qn = a.Qc + (size_t)(k + 1) * m;
      for (int i = threadIdx.x; i < m; i += GS_THREADS) qn[i] = c[i] / rkk;  // this thread's own c[i]
      if (threadIdx.x == 0) {
        a.R[(size_t)k * n + (k + 1)] = (float)r;
        a.R[(size_t)(k + 1) * n + (k + 1)] = (float)rkk;
      }
      __syncthreads();
      if (threadIdx.x == 0) {
        __threadfence();
        st_release_u32(a.ready, (unsigned)(k + 2));
      }
      tb = t0 + 1;
    }
    // the other owned columns j > k+1, in batches of up to GS_MAXC with a compile-time
    // width (no predicated work for absent columns): dot -> CTA reduce -> axpy
    for (int b0 = tb; b0 < nown; b0 += GS_MAXC) {
      const int nb = min(GS_MAXC, nown - b0);
      double* base = colp(b0);
      const size_t cs = a.in_smem ? (size_t)m : (size_t)G * m;  // column stride
      const int j0 = cta + b0 * G;
      switch (nb) {
#define PB_GS_CASE(N) \
  case N: gs_batch<N>(a, qr, q, base, cs, j0, G, k, red, rsum); break;
        PB_GS_CASE(1) PB_GS_CASE(2) PB_GS_CASE(3) PB_GS_CASE(4) PB_GS_CASE(5) PB_GS_CASE(6) PB_GS_CASE(7)
        PB_GS_CASE(8) PB_GS_CASE(9) PB_GS_CASE(10) PB_GS_CASE(11) PB_GS_CASE(12) PB_GS_CASE(13) PB_GS_CASE(14)
        PB_GS_CASE(15) PB_GS_CASE(16)
#undef PB_GS_CASE
      }
    }
  }
  if (a.in_smem) {
    __syncthreads();
    for (int t = 0; t < nown; ++t) {
      double* dst = a.W + (size_t)(cta + t * G) * m;
      const double* src = cols + (size_t)t * m;
      for (int i = threadIdx.x; i < m; i += GS_THREADS) dst[i] = src[i];
    }
  }
}

// out[c][r] = (Tout) in[r][c]; in rows x cols (row-major), 32x32 tiles through smem.
template <typename Tin, typename Tout>
__global__ void __launch_bounds__(256) gs_transpose_kernel(const Tin* __restrict__ in, int rows, int cols,
                                                           Tout* __restrict__ out) {
  __shared__ Tin tile[32][33];
  pdl_wait();
  const int c0 = blockIdx.x * 32, r0 = blockIdx.y * 32;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  for (int y = ty; y < 32; y += 8) {
    const int r = r0 + y, c = c0 + tx;
    if (r < rows && c < cols) tile[y][tx] = in[(size_t)r * cols + c];
  }
  __syncthreads();
  for (int y = ty; y < 32; y += 8) {
    const int c = c0 + y, r = r0 + tx;
    if (r < rows && c < cols) out[(size_t)c * rows + r] = (Tout)tile[tx][y];
  }
}

int gs_sms() {
  static int cache[64] = {0};
  int dev = 0;
  cudaGetDevice(&dev);
  int& n = cache[dev & 63];
  if (!n) {
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}


// ---- ablation: the PolyBench-GPU / SYCL-Bench kernel shape --------------------------
// Three launches per column k over fp64 row-major working arrays: a single work-item
// computes the norm, m work-items normalise column k, and one work-item per column
// j > k forms R[k][j] and updates column j (each looping over the m rows).
__global__ void gsn_norm_kernel(const double* __restrict__ W, double* __restrict__ Rd, int m, int n, int k) {
  double nrm = 0.0;
  for (int i = 0; i < m; ++i) nrm += W[(size_t)i * n + k] * W[(size_t)i * n + k];
  Rd[(size_t)k * n + k] = sqrt(nrm);
}
__global__ void gsn_q_kernel(const double* __restrict__ W, const double* __restrict__ Rd, double* __restrict__ Qd,
                             int m, int n, int k) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < m) Qd[(size_t)i * n + k] = W[(size_t)i * n + k] / Rd[(size_t)k * n + k];
}
__global__ void gsn_update_kernel(double* __restrict__ W, double* __restrict__ Rd, const double* __restrict__ Qd,
                                  int m, int n, int k) {
  const int j = k + 1 + blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n) return;
  double r = 0.0;
  for (int i = 0; i < m; ++i) r += Qd[(size_t)i * n + k] * W[(size_t)i * n + j];
  Rd[(size_t)k * n + j] = r;
  for (int i = 0; i < m; ++i) W[(size_t)i * n + j] -= Qd[(size_t)i * n + k] * r;
}
template <typename Tin, typename Tout>
__global__ void gsn_copy_kernel(const Tin* __restrict__ in, Tout* __restrict__ out, long long count) {
  const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (e < count) out[e] = (Tout)in[e];
}
// R (fp32) upper triangle from Rd: R[k][j] for j >= k
__global__ void gsn_r_kernel(const double* __restrict__ Rd, float* __restrict__ R, int n) {
  const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (e < (long long)n * n && e % n >= e / n) R[e] = (float)Rd[e];
}

}  // namespace

size_t gramschmidt_ws_bytes(int m, int n) {
  const size_t mat = align_up((size_t)m * n * sizeof(double), 256);
  const size_t rn = align_up((size_t)n * n * sizeof(double), 256);
  return 2 * mat + 256 + rn;  // + fp64 R for the ablation variant
}

cudaError_t launch_gramschmidt_naive(int m, int n, float* A, float* R, float* Q, void* ws, cudaStream_t s,
                                     int* launches) {
  const size_t mat = align_up((size_t)m * n * sizeof(double), 256);
  double* W = static_cast<double*>(ws);
  double* Qd = reinterpret_cast<double*>(static_cast<char*>(ws) + mat);
  double* Rd = reinterpret_cast<double*>(static_cast<char*>(ws) + 2 * mat + 256);
  const long long mn = (long long)m * n;
  const unsigned gmn = (unsigned)((mn + 255) / 256);
  gsn_copy_kernel<float, double><<<gmn, 256, 0, s>>>(A, W, mn);
  int L = 1;
  for (int k = 0; k < n; ++k) {
    gsn_norm_kernel<<<1, 1, 0, s>>>(W, Rd, m, n, k);
    gsn_q_kernel<<<(m + 255) / 256, 256, 0, s>>>(W, Rd, Qd, m, n, k);
    L += 2;
    if (k + 1 < n) {
      gsn_update_kernel<<<(n - k - 1 + 255) / 256, 256, 0, s>>>(W, Rd, Qd, m, n, k);
      ++L;
    }
  }
  gsn_copy_kernel<double, float><<<gmn, 256, 0, s>>>(W, A, mn);
  gsn_copy_kernel<double, float><<<gmn, 256, 0, s>>>(Qd, Q, mn);
  gsn_r_kernel<<<(unsigned)(((long long)n * n + 255) / 256), 256, 0, s>>>(Rd, R, n);
  *launches += L + 3;
  return cudaGetLastError();
}

cudaError_t launch_gramschmidt(int m, int n, float* A, float* R, float* Q, void* ws, cudaStream_t s, int* launches) {
  const size_t mat = align_up((size_t)m * n * sizeof(double), 256);
  double* W = static_cast<double*>(ws);
  double* Qc = reinterpret_cast<double*>(static_cast<char*>(ws) + mat);
  unsigned* ready = reinterpret_cast<unsigned*>(static_cast<char*>(ws) + 2 * mat);
  cudaError_t e = cudaMemsetAsync(ready, 0, sizeof(unsigned), s);
  if (e != cudaSuccess) return e;
  const dim3 tb(256);
  // A (m x n, row-major fp32) -> W (n x m: column-major fp64)
  e = launch_pdl(gs_transpose_kernel<float, double>, dim3((n + 31) / 32, (m + 31) / 32), tb, 0, s, (const float*)A, m,
                 n, W);
  if (e != cudaSuccess) return e;
  const int G = std::min(gs_sms(), n);
  const int cpc = (n + G - 1) / G;
  const size_t smem_cols = (size_t)cpc * m * sizeof(double);
  const bool in_smem = smem_cols <= 200 * 1024;
  const size_t smem = in_smem ? smem_cols : 0;
  e = ensure_smem<gs_kernel>(200 * 1024);
  if (e != cudaSuccess) return e;
  GsArgs a{m, n, cpc, W, Qc, R, ready, in_smem ? 1 : 0};
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(G);
  cfg.blockDim = dim3(GS_THREADS);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeCooperative;  // all CTAs co-resident: the spin waits are safe
  at[0].val.cooperative = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  e = cudaLaunchKernelEx(&cfg, gs_kernel, a);
  if (e != cudaSuccess) return e;
  // W (n x m) -> A (m x n, fp32); Qc (n x m) -> Q (m x n, fp32)
  e = launch_pdl(gs_transpose_kernel<double, float>, dim3((m + 31) / 32, (n + 31) / 32), tb, 0, s, (const double*)W,
                 n, m, A);
  if (e != cudaSuccess) return e;
  e = launch_pdl(gs_transpose_kernel<double, float>, dim3((m + 31) / 32, (n + 31) / 32), tb, 0, s, (const double*)Qc,
                 n, m, Q);
  if (e != cudaSuccess) return e;
  *launches += 4;
  return cudaSuccess;
}

}  // namespace pb
