// pb_oracle.cpp — the CPU ORACLE for the PolyBench hot path. TEST INFRASTRUCTURE ONLY.
//
// Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline leg and
// --impl reference) may load this library. The product path (libpb) never
// links, loads or calls it, and it shares no code with libpb.
//
// What it computes. The paper (PAPER.md, arXiv 2312.13170) names the
// SYCL-Bench polybench kernels it optimises (§VIII "Evaluation")
// and shows only the GEMM body (Listing 8, §VI-C
// "Loop Internalization"). Loop internalization and
// detect-reduction (Listings 4-5) are semantics-preserving
// rewrites of those loops, so the oracle is the plain definition of each
// kernel, written out in the PolyBench/C 4.2 problem statements' order
// (readings R1-R16 in DESIGN.md).
//
// Precision. Inputs are the fp32 arrays; every product and sum is done in
// IEEE double (reading R2), results are returned as double. Build flags
// -O2 -fopenmp -ffp-contract=off (no FMA contraction, no fast-math): each
// output's summation order is the definition's k = 0..K-1 order and one thread
// owns each output, so results are bitwise identical for any thread count.
//
// absmode != 0 evaluates the same definition on absolute values of every term
// (|alpha|, |beta|, |x|), giving the per-element magnitude scale s_e used by
// the componentwise parity gate (reading R8): err = max_e |g_e - r_e| / s_e.
// For covariance/correlation the centring (mean) and the normalisation are
// computed as usual and the absolute value is applied to the centred /
// normalised values X, so s = |X|^T |X| (/(n-1)).
//
// Parity pins for every function live in tests/test_oracle_pins.py
// (closed forms, exact rational brute force, numpy library cross-checks,
// invariants); see DESIGN.md "Oracle and its pins".
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <vector>
#ifdef _OPENMP
#include <omp.h>
#endif

namespace {
inline double V(float x, int absmode) { return absmode ? std::fabs((double)x) : (double)x; }
inline double S(double x, int absmode) { return absmode ? std::fabs(x) : x; }
}  // namespace

extern "C" {

// gemm (PolyBench/C 4.2 kernel_gemm; Listing 8 is alpha=beta=1):
//   C'[i][j] = beta*C[i][j] + alpha * sum_{k<nk} A[i][k]*B[k][j]
// A ni x nk, B nk x nj, C ni x nj (row-major).
void pbo_gemm(int ni, int nj, int nk, double alpha, double beta, const float* C, const float* A,
              const float* B, double* Cout, int absmode) {
  alpha = S(alpha, absmode);
  beta = S(beta, absmode);
#pragma omp parallel for schedule(dynamic, 1)
  for (int i = 0; i < ni; ++i) {
    std::vector<double> acc(nj, 0.0);
    for (int k = 0; k < nk; ++k) {  // sum over k in order 0..nk-1 for every j
      double a = V(A[(size_t)i * nk + k], absmode);
      const float* Bk = B + (size_t)k * nj;
      for (int j = 0; j < nj; ++j) acc[j] += a * V(Bk[j], absmode);
    }
    for (int j = 0; j < nj; ++j)
      Cout[(size_t)i * nj + j] = beta * V(C[(size_t)i * nj + j], absmode) + alpha * acc[j];
  }
}

// Double-input matrix product used by the chained kernels (2mm, 3mm): the
// intermediates tmp/E/F are kept in double (reading R14).
static void mm_dd(int ni, int nj, int nk, const double* A, const double* B, double* out) {
#pragma omp parallel for schedule(dynamic, 1)
  for (int i = 0; i < ni; ++i) {
    std::vector<double> acc(nj, 0.0);
    for (int k = 0; k < nk; ++k) {
      double a = A[(size_t)i * nk + k];
      const double* Bk = B + (size_t)k * nj;
      for (int j = 0; j < nj; ++j) acc[j] += a * Bk[j];
    }
    for (int j = 0; j < nj; ++j) out[(size_t)i * nj + j] = acc[j];
  }
}

static std::vector<double> widen(const float* x, size_t n, int absmode) {
  std::vector<double> v(n);
  for (size_t i = 0; i < n; ++i) v[i] = V(x[i], absmode);
  return v;
}

// 2mm (PolyBench/C 4.2 kernel_2mm):
//   tmp[i][j] = alpha * sum_{k<nk} A[i][k]*B[k][j]
//   D'[i][l]  = beta*D[i][l] + sum_{j<nj} tmp[i][j]*C[j][l]
// A ni x nk, B nk x nj, tmp ni x nj, C nj x nl, D ni x nl.
void pbo_2mm(int ni, int nj, int nk, int nl, double alpha, double beta, const float* A,
             const float* B, const float* C, const float* D, double* tmp_out, double* D_out,
             int absmode) {
  alpha = S(alpha, absmode);
  beta = S(beta, absmode);
  std::vector<double> a = widen(A, (size_t)ni * nk, absmode), b = widen(B, (size_t)nk * nj, absmode),
                      c = widen(C, (size_t)nj * nl, absmode);
  std::vector<double> ab((size_t)ni * nj);
  mm_dd(ni, nj, nk, a.data(), b.data(), ab.data());
  for (size_t e = 0; e < ab.size(); ++e) tmp_out[e] = alpha * ab[e];
  std::vector<double> tc((size_t)ni * nl);
  mm_dd(ni, nl, nj, tmp_out, c.data(), tc.data());
  for (size_t e = 0; e < tc.size(); ++e) D_out[e] = beta * V(D[e], absmode) + tc[e];
}

// 3mm (PolyBench/C 4.2 kernel_3mm):
//   E = A*B (ni x nj, contraction nk);  F = C*D (nj x nl, contraction nm);
//   G = E*F (ni x nl, contraction nj).
void pbo_3mm(int ni, int nj, int nk, int nl, int nm, const float* A, const float* B,
             const float* C, const float* D, double* E_out, double* F_out, double* G_out,
             int absmode) {
  std::vector<double> a = widen(A, (size_t)ni * nk, absmode), b = widen(B, (size_t)nk * nj, absmode),
                      c = widen(C, (size_t)nj * nm, absmode), d = widen(D, (size_t)nm * nl, absmode);
  mm_dd(ni, nj, nk, a.data(), b.data(), E_out);
  mm_dd(nj, nl, nm, c.data(), d.data(), F_out);
  mm_dd(ni, nl, nj, E_out, F_out, G_out);
}

// syrk (PolyBench/C 4.2 kernel_syrk, lower triangle, reading R3):
//   for j <= i: C'[i][j] = beta*C[i][j] + alpha * sum_{k<m} A[i][k]*A[j][k]
//   for j >  i: C'[i][j] = C[i][j]   (untouched)
// A n x m, C n x n.
void pbo_syrk(int n, int m, double alpha, double beta, const float* C, const float* A,
              double* Cout, int absmode) {
  alpha = S(alpha, absmode);
  beta = S(beta, absmode);
#pragma omp parallel for schedule(dynamic, 1)
  for (int i = 0; i < n; ++i) {
    for (int j = 0; j < n; ++j) {
      size_t e = (size_t)i * n + j;
      if (j > i) { Cout[e] = V(C[e], absmode); continue; }
      double acc = 0.0;
      for (int k = 0; k < m; ++k)
        acc += V(A[(size_t)i * m + k], absmode) * V(A[(size_t)j * m + k], absmode);
      Cout[e] = beta * V(C[e], absmode) + alpha * acc;
    }
  }
}

// syr2k (PolyBench/C 4.2 kernel_syr2k, lower triangle, reading R3):
//   for j <= i: C'[i][j] = beta*C[i][j]
//                + alpha * sum_{k<m} (A[j][k]*B[i][k] + B[j][k]*A[i][k])
//   for j > i : untouched.   A, B n x m; C n x n.
void pbo_syr2k(int n, int m, double alpha, double beta, const float* C, const float* A,
               const float* B, double* Cout, int absmode) {
  alpha = S(alpha, absmode);
  beta = S(beta, absmode);
#pragma omp parallel for schedule(dynamic, 1)
  for (int i = 0; i < n; ++i) {
    for (int j = 0; j < n; ++j) {
      size_t e = (size_t)i * n + j;
      if (j > i) { Cout[e] = V(C[e], absmode); continue; }
      double acc = 0.0;
      for (int k = 0; k < m; ++k)
        acc += V(A[(size_t)j * m + k], absmode) * V(B[(size_t)i * m + k], absmode) +
               V(B[(size_t)j * m + k], absmode) * V(A[(size_t)i * m + k], absmode);
      Cout[e] = beta * V(C[e], absmode) + alpha * acc;
    }
  }
}

// Column means (PolyBench/C 4.2 kernel_covariance/correlation, first loop):
//   mean[j] = (sum_{i<n} data[i][j]) / float_n
static void col_mean(int m, int n, double float_n, const float* data, double* mean) {
#pragma omp parallel for schedule(static)
  for (int j = 0; j < m; ++j) {
    double acc = 0.0;
    for (int i = 0; i < n; ++i) acc += (double)data[(size_t)i * m + j];
    mean[j] = acc / float_n;
  }
}

// covariance (PolyBench/C 4.2 kernel_covariance; float_n and (float_n-1) per reading R4):
//   mean[j]  = sum_i data[i][j] / float_n
//   X[i][j]  = data[i][j] - mean[j]
//   for j >= i: cov[i][j] = sum_{k<n} X[k][i]*X[k][j] / (float_n - 1); cov[j][i] = cov[i][j]
// data n x m (n observations, m variables); cov m x m; mean m.
void pbo_covariance(int m, int n, double float_n, const float* data, double* cov, double* mean,
                    int absmode) {
  col_mean(m, n, float_n, data, mean);
  std::vector<double> X((size_t)n * m);
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < m; ++j) X[(size_t)i * m + j] = S((double)data[(size_t)i * m + j] - mean[j], absmode);
  if (absmode) {  // scale of the mean itself: sum |data| / float_n
    for (int j = 0; j < m; ++j) {
      double acc = 0.0;
      for (int i = 0; i < n; ++i) acc += std::fabs((double)data[(size_t)i * m + j]);
      mean[j] = acc / std::fabs(float_n);
    }
  }
  double den = S(float_n - 1.0, absmode);
#pragma omp parallel for schedule(dynamic, 1)
  for (int i = 0; i < m; ++i) {
    for (int j = i; j < m; ++j) {
      double acc = 0.0;
      for (int k = 0; k < n; ++k) acc += X[(size_t)k * m + i] * X[(size_t)k * m + j];
      cov[(size_t)i * m + j] = acc / den;
      cov[(size_t)j * m + i] = cov[(size_t)i * m + j];
    }
  }
}

// correlation (PolyBench/C 4.2 kernel_correlation; eps rule R5, diagonal R6):
//   mean[j]   = sum_i data[i][j] / float_n
//   stddev[j] = sqrt( sum_i (data[i][j]-mean[j])^2 / float_n );  stddev[j] <= eps => 1.0
//   X[i][j]   = (data[i][j] - mean[j]) / (sqrt(float_n) * stddev[j])
//   corr[i][i] = 1 (all i, including m-1)
//   for j > i: corr[i][j] = sum_{k<n} X[k][i]*X[k][j]; corr[j][i] = corr[i][j]
void pbo_correlation(int m, int n, double float_n, double eps, const float* data, double* corr,
                     double* mean, double* stddev, int absmode) {
  col_mean(m, n, float_n, data, mean);
#pragma omp parallel for schedule(static)
  for (int j = 0; j < m; ++j) {
    double acc = 0.0;
    for (int i = 0; i < n; ++i) {
      double d = (double)data[(size_t)i * m + j] - mean[j];
      acc += d * d;
    }
    stddev[j] = std::sqrt(acc / float_n);
    if (stddev[j] <= eps) stddev[j] = 1.0;
  }
  std::vector<double> X((size_t)n * m);
  double sq = std::sqrt(float_n);
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < m; ++j)
      X[(size_t)i * m + j] = S(((double)data[(size_t)i * m + j] - mean[j]) / (sq * stddev[j]), absmode);
  if (absmode) {
    for (int j = 0; j < m; ++j) {
      double acc = 0.0;
      for (int i = 0; i < n; ++i) acc += std::fabs((double)data[(size_t)i * m + j]);
      mean[j] = acc / std::fabs(float_n);
    }
  }
#pragma omp parallel for schedule(dynamic, 1)
  for (int i = 0; i < m; ++i) {
    corr[(size_t)i * m + i] = 1.0;
    for (int j = i + 1; j < m; ++j) {
      double acc = 0.0;
      for (int k = 0; k < n; ++k) acc += X[(size_t)k * m + i] * X[(size_t)k * m + j];
      corr[(size_t)i * m + j] = acc;
      corr[(size_t)j * m + i] = acc;
    }
  }
}

// Row dot products r_i = sum_{j<cols} M[i][j]*v[j] for i in [0,rows).
static void row_dots(int rows, int cols, const float* M, const double* v, double* out, int absmode) {
#pragma omp parallel for schedule(static)
  for (int i = 0; i < rows; ++i) {
    double acc = 0.0;
    for (int j = 0; j < cols; ++j) acc += V(M[(size_t)i * cols + j], absmode) * v[j];
    out[i] = acc;
  }
}

// Transposed products c_j = sum_{i<rows} w[i]*M[i][j]; each thread owns a
// contiguous range of j and walks i in order 0..rows-1, so every c_j is
// summed in the definition's order (loop interchange only, no reordering).
static void col_dots(int rows, int cols, const float* M, const double* w, double* out, int absmode) {
#pragma omp parallel
  {
#ifdef _OPENMP
    int t = omp_get_thread_num(), nt = omp_get_num_threads();
#else
    int t = 0, nt = 1;
#endif
    int j0 = (int)((long long)cols * t / nt), j1 = (int)((long long)cols * (t + 1) / nt);
    std::vector<double> acc(j1 - j0, 0.0);
    for (int i = 0; i < rows; ++i) {
      const float* Mi = M + (size_t)i * cols;
      double wi = w[i];
      for (int j = j0; j < j1; ++j) acc[j - j0] += wi * V(Mi[j], absmode);
    }
    for (int j = j0; j < j1; ++j) out[j] = acc[j - j0];
  }
}

// atax (PolyBench/C 4.2 kernel_atax):  tmp[i] = sum_j A[i][j]*x[j];  y[j] = sum_i A[i][j]*tmp[i]
// A m x n, x n, y n, tmp m.
void pbo_atax(int m, int n, const float* A, const float* x, double* y, double* tmp, int absmode) {
  std::vector<double> xv = widen(x, n, absmode);
  row_dots(m, n, A, xv.data(), tmp, absmode);
  col_dots(m, n, A, tmp, y, absmode);
}

// bicg (PolyBench/C 4.2 kernel_bicg):  s[j] = sum_i r[i]*A[i][j];  q[i] = sum_j A[i][j]*p[j]
// A n x m, s m, q n, p m, r n.
void pbo_bicg(int m, int n, const float* A, const float* p, const float* r, double* s, double* q,
              int absmode) {
  std::vector<double> pv = widen(p, m, absmode), rv = widen(r, n, absmode);
  row_dots(n, m, A, pv.data(), q, absmode);
  col_dots(n, m, A, rv.data(), s, absmode);
}

// mvt (PolyBench/C 4.2 kernel_mvt):
//   x1'[i] = x1[i] + sum_j A[i][j]*y_1[j];   x2'[i] = x2[i] + sum_j A[j][i]*y_2[j]
// A n x n.
void pbo_mvt(int n, const float* x1, const float* x2, const float* y_1, const float* y_2,
             const float* A, double* x1_out, double* x2_out, int absmode) {
  std::vector<double> y1v = widen(y_1, n, absmode), y2v = widen(y_2, n, absmode), d(n);
  row_dots(n, n, A, y1v.data(), d.data(), absmode);
  for (int i = 0; i < n; ++i) x1_out[i] = V(x1[i], absmode) + d[i];
  col_dots(n, n, A, y2v.data(), d.data(), absmode);
  for (int i = 0; i < n; ++i) x2_out[i] = V(x2[i], absmode) + d[i];
}

// gesummv (PolyBench/C 4.2 kernel_gesummv):
//   tmp[i] = sum_j A[i][j]*x[j];  y[i] = alpha*tmp[i] + beta * sum_j B[i][j]*x[j]
// A, B n x n; x, y, tmp n.
void pbo_gesummv(int n, double alpha, double beta, const float* A, const float* B, const float* x,
                 double* tmp, double* y, int absmode) {
  alpha = S(alpha, absmode);
  beta = S(beta, absmode);
  std::vector<double> xv = widen(x, n, absmode), bx(n);
  row_dots(n, n, A, xv.data(), tmp, absmode);
  row_dots(n, n, B, xv.data(), bx.data(), absmode);
  for (int i = 0; i < n; ++i) y[i] = alpha * tmp[i] + beta * bx[i];
}

// ---- sampled evaluation for the full-size configs (parity at BASELINE sizes) ----
// gemm entries at (rows[t], cols[t]); same arithmetic as pbo_gemm per entry.
void pbo_gemm_at(int ni, int nj, int nk, double alpha, double beta, const float* C, const float* A,
                 const float* B, int npts, const int* rows, const int* cols, double* out,
                 int absmode) {
  alpha = S(alpha, absmode);
  beta = S(beta, absmode);
  (void)ni;
#pragma omp parallel for schedule(dynamic, 4)
  for (int t = 0; t < npts; ++t) {
    int i = rows[t], j = cols[t];
    double acc = 0.0;
    for (int k = 0; k < nk; ++k)
      acc += V(A[(size_t)i * nk + k], absmode) * V(B[(size_t)k * nj + j], absmode);
    out[t] = beta * V(C[(size_t)i * nj + j], absmode) + alpha * acc;
  }
}

// syr2k / syrk entries at (rows[t], cols[t]) (B == A gives syrk when alpha is halved:
// not used that way — syrk passes B=NULL).
void pbo_syrk_at(int n, int m, double alpha, double beta, const float* C, const float* A,
                 const float* B, int npts, const int* rows, const int* cols, double* out,
                 int absmode) {
  alpha = S(alpha, absmode);
  beta = S(beta, absmode);
#pragma omp parallel for schedule(dynamic, 4)
  for (int t = 0; t < npts; ++t) {
    int i = rows[t], j = cols[t];
    size_t e = (size_t)i * n + j;
    if (j > i) { out[t] = V(C[e], absmode); continue; }
    double acc = 0.0;
    for (int k = 0; k < m; ++k) {
      if (B == nullptr)
        acc += V(A[(size_t)i * m + k], absmode) * V(A[(size_t)j * m + k], absmode);
      else
        acc += V(A[(size_t)j * m + k], absmode) * V(B[(size_t)i * m + k], absmode) +
               V(B[(size_t)j * m + k], absmode) * V(A[(size_t)i * m + k], absmode);
    }
    out[t] = beta * V(C[e], absmode) + alpha * acc;
  }
}

// Rows [r0, r1) of the product of two fp32 matrices in double: out = X[r0:r1] * Y
// (X rows x inner, Y inner x cols). Used to evaluate sampled ROWS of the 2mm/3mm
// chains: tmp rows = alpha*A[r]*B, then D rows = tmp rows * C + beta*D.
void pbo_rows_mm(int r0, int r1, int inner, int cols, const float* X, const float* Y, double* out,
                 int absmode) {
#pragma omp parallel for schedule(dynamic, 1)
  for (int i = r0; i < r1; ++i) {
    std::vector<double> acc(cols, 0.0);
    for (int k = 0; k < inner; ++k) {
      double a = V(X[(size_t)i * inner + k], absmode);
      const float* Yk = Y + (size_t)k * cols;
      for (int j = 0; j < cols; ++j) acc[j] += a * V(Yk[j], absmode);
    }
    for (int j = 0; j < cols; ++j) out[(size_t)(i - r0) * cols + j] = acc[j];
  }
}

// out (rows x cols) = X (rows x inner, double) * Y (inner x cols, fp32)
void pbo_dmm(int rows, int inner, int cols, const double* X, const float* Y, double* out,
             int absmode) {
#pragma omp parallel for schedule(dynamic, 1)
  for (int i = 0; i < rows; ++i) {
    std::vector<double> acc(cols, 0.0);
    for (int k = 0; k < inner; ++k) {
      double a = S(X[(size_t)i * inner + k], absmode);
      const float* Yk = Y + (size_t)k * cols;
      for (int j = 0; j < cols; ++j) acc[j] += a * V(Yk[j], absmode);
    }
    for (int j = 0; j < cols; ++j) out[(size_t)i * cols + j] = acc[j];
  }
}

// ---- SYCL-Bench polybench stencils (§VIII lists "2D Convolution",
// "3D Convolution", "FDTD2D"). The paper gives no body for
// them; readings R19-R21 in DESIGN.md fix the definitions used here.

// conv2d (reading R19): the SYCL-Bench / PolyBench-GPU 2DConvolution is a 3x3
// weighted stencil (a cross-correlation) over the interior:
//   B[i][j] = sum_{di=-1..1} sum_{dj=-1..1} w[(di+1)*3 + (dj+1)] * A[i+di][j+dj]
//   for 1 <= i <= ni-2, 1 <= j <= nj-2;  border entries of B keep B_in.
// A, B ni x nj. Rows [i0, i1) of the result are written to out ((i1-i0) x nj).
void pbo_conv2d(int ni, int nj, const double* w, const float* A, const float* B_in, int i0, int i1,
                double* out, int absmode) {
#pragma omp parallel for schedule(static)
  for (int i = i0; i < i1; ++i) {
    for (int j = 0; j < nj; ++j) {
      size_t e = (size_t)i * nj + j;
      double r;
      if (i == 0 || i == ni - 1 || j == 0 || j == nj - 1) {
        r = V(B_in[e], absmode);
      } else {
        r = 0.0;
        for (int di = -1; di <= 1; ++di)
          for (int dj = -1; dj <= 1; ++dj)
            r += S(w[(di + 1) * 3 + (dj + 1)], absmode) * V(A[(size_t)(i + di) * nj + (j + dj)], absmode);
      }
      out[(size_t)(i - i0) * nj + j] = r;
    }
  }
}

// conv3d (reading R20): 3x3x3 weighted stencil over the interior of an
// ni x nj x nk array (row-major, k fastest):
//   B[i][j][k] = sum_{di,dj,dk in -1..1} w[(di+1)*9 + (dj+1)*3 + (dk+1)] * A[i+di][j+dj][k+dk]
//   for 1 <= i <= ni-2, 1 <= j <= nj-2, 1 <= k <= nk-2; border entries keep B_in.
// Planes [i0, i1) of the result are written to out ((i1-i0) x nj x nk).
void pbo_conv3d(int ni, int nj, int nk, const double* w, const float* A, const float* B_in, int i0, int i1,
                double* out, int absmode) {
  const size_t plane = (size_t)nj * nk;
#pragma omp parallel for collapse(2) schedule(static)
  for (int i = i0; i < i1; ++i) {
    for (int j = 0; j < nj; ++j) {
      for (int k = 0; k < nk; ++k) {
        size_t e = (size_t)i * plane + (size_t)j * nk + k;
        double r;
        if (i == 0 || i == ni - 1 || j == 0 || j == nj - 1 || k == 0 || k == nk - 1) {
          r = V(B_in[e], absmode);
        } else {
          r = 0.0;
          for (int di = -1; di <= 1; ++di)
            for (int dj = -1; dj <= 1; ++dj)
              for (int dk = -1; dk <= 1; ++dk)
                r += S(w[(di + 1) * 9 + (dj + 1) * 3 + (dk + 1)], absmode) *
                     V(A[(size_t)(i + di) * plane + (size_t)(j + dj) * nk + (k + dk)], absmode);
        }
        out[(size_t)(i - i0) * plane + (size_t)j * nk + k] = r;
      }
    }
  }
}

// fdtd-2d (reading R21; PolyBench/C 4.2 kernel_fdtd_2d, the SYCL-Bench FDTD2D):
//   for t in 0..tmax-1:
//     ey[0][j] = fict[t]                                             (all j)
//     ey[i][j] = ey[i][j] - 0.5*(hz[i][j] - hz[i-1][j])              (1 <= i < nx, all j)
//     ex[i][j] = ex[i][j] - 0.5*(hz[i][j] - hz[i][j-1])              (all i, 1 <= j < ny)
//     hz[i][j] = hz[i][j] - 0.7*(ex[i][j+1] - ex[i][j] + ey[i+1][j] - ey[i][j])
//                                                                    (i < nx-1, j < ny-1)
// ex, ey, hz nx x ny; fict tmax. The three sweeps run in this order, each over
// the state the previous sweep left (Jacobi within a sweep: no statement reads a
// value its own sweep writes). State kept in double; inputs are the fp32 arrays.
void pbo_fdtd2d(int tmax, int nx, int ny, const float* ex, const float* ey, const float* hz,
                const float* fict, double* ex_o, double* ey_o, double* hz_o) {
  const size_t N = (size_t)nx * ny;
  for (size_t e = 0; e < N; ++e) { ex_o[e] = ex[e]; ey_o[e] = ey[e]; hz_o[e] = hz[e]; }
  for (int t = 0; t < tmax; ++t) {
    for (int j = 0; j < ny; ++j) ey_o[j] = (double)fict[t];
#pragma omp parallel for schedule(static)
    for (int i = 1; i < nx; ++i)
      for (int j = 0; j < ny; ++j)
        ey_o[(size_t)i * ny + j] = ey_o[(size_t)i * ny + j] - 0.5 * (hz_o[(size_t)i * ny + j] - hz_o[(size_t)(i - 1) * ny + j]);
#pragma omp parallel for schedule(static)
    for (int i = 0; i < nx; ++i)
      for (int j = 1; j < ny; ++j)
        ex_o[(size_t)i * ny + j] = ex_o[(size_t)i * ny + j] - 0.5 * (hz_o[(size_t)i * ny + j] - hz_o[(size_t)i * ny + j - 1]);
#pragma omp parallel for schedule(static)
    for (int i = 0; i < nx - 1; ++i)
      for (int j = 0; j < ny - 1; ++j) {
        size_t e = (size_t)i * ny + j;
        hz_o[e] = hz_o[e] - 0.7 * (ex_o[e + 1] - ex_o[e] + ey_o[e + ny] - ey_o[e]);
      }
  }
}

// The same statements evaluated in fp32 (PolyBench's DATA_TYPE float, constants
// 0.5f / 0.7f, C left-to-right evaluation, no contraction: built with
// -ffp-contract=off, SSE arithmetic, so every operation is one IEEE fp32 RN op).
// A GPU that issues the same fp32 operations in the same order reproduces it bitwise.
void pbo_fdtd2d_f32(int tmax, int nx, int ny, const float* ex, const float* ey, const float* hz,
                    const float* fict, float* ex_o, float* ey_o, float* hz_o) {
  const size_t N = (size_t)nx * ny;
  std::memcpy(ex_o, ex, N * sizeof(float));
  std::memcpy(ey_o, ey, N * sizeof(float));
  std::memcpy(hz_o, hz, N * sizeof(float));
  for (int t = 0; t < tmax; ++t) {
    for (int j = 0; j < ny; ++j) ey_o[j] = fict[t];
#pragma omp parallel for schedule(static)
    for (int i = 1; i < nx; ++i)
      for (int j = 0; j < ny; ++j)
        ey_o[(size_t)i * ny + j] = ey_o[(size_t)i * ny + j] - 0.5f * (hz_o[(size_t)i * ny + j] - hz_o[(size_t)(i - 1) * ny + j]);
#pragma omp parallel for schedule(static)
    for (int i = 0; i < nx; ++i)
      for (int j = 1; j < ny; ++j)
        ex_o[(size_t)i * ny + j] = ex_o[(size_t)i * ny + j] - 0.5f * (hz_o[(size_t)i * ny + j] - hz_o[(size_t)i * ny + j - 1]);
#pragma omp parallel for schedule(static)
    for (int i = 0; i < nx - 1; ++i)
      for (int j = 0; j < ny - 1; ++j) {
        size_t e = (size_t)i * ny + j;
        hz_o[e] = hz_o[e] - 0.7f * (ex_o[e + 1] - ex_o[e] + ey_o[e + ny] - ey_o[e]);
      }
  }
}

// gramschmidt (reading R22; PolyBench/C 4.2 kernel_gramschmidt, the SYCL-Bench
// "Gramschmidt" of PAPER.md:524 — the benchmark whose candidate loop sits in a
// divergent region). Modified Gram-Schmidt, in this order:
//   for k < n:  nrm = sum_{i<m} A[i][k]^2;  R[k][k] = sqrt(nrm);
//               Q[i][k] = A[i][k] / R[k][k]                       (i < m)
//               for j in k+1..n-1:  R[k][j] = sum_{i<m} Q[i][k]*A[i][j];
//                                   A[i][j] = A[i][j] - Q[i][k]*R[k][j]   (i < m)
// A m x n (in/out), R n x n (entries j < k not written: R_out keeps 0 there),
// Q m x n. State and outputs in double; inputs are the fp32 A.
void pbo_gramschmidt(int m, int n, const float* A, double* A_out, double* R, double* Q) {
  for (size_t e = 0; e < (size_t)m * n; ++e) A_out[e] = (double)A[e];
  for (size_t e = 0; e < (size_t)n * n; ++e) R[e] = 0.0;
  for (int k = 0; k < n; ++k) {
    double nrm = 0.0;
    for (int i = 0; i < m; ++i) nrm += A_out[(size_t)i * n + k] * A_out[(size_t)i * n + k];
    R[(size_t)k * n + k] = std::sqrt(nrm);
    for (int i = 0; i < m; ++i) Q[(size_t)i * n + k] = A_out[(size_t)i * n + k] / R[(size_t)k * n + k];
#pragma omp parallel for schedule(static)
    for (int j = k + 1; j < n; ++j) {
      double r = 0.0;
      for (int i = 0; i < m; ++i) r += Q[(size_t)i * n + k] * A_out[(size_t)i * n + j];
      R[(size_t)k * n + j] = r;
      for (int i = 0; i < m; ++i) A_out[(size_t)i * n + j] = A_out[(size_t)i * n + j] - Q[(size_t)i * n + k] * r;
    }
  }
}

}  // extern "C"
