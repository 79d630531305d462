/* pbgen_host.c — host side of the shared input generator (see pbgen_core.h).
 * Build: gcc -O2 -fopenmp -ffp-contract=off -shared -fPIC (no FMA contraction,
 * so base*scale+offset rounds exactly like the device's __dmul_rn/__dadd_rn). */
#include "pbgen_core.h"

/* Fill dst[(r-row0)*cols + c] for r in [row0,row1), c in [0,cols).
 * ld = number of columns of the FULL matrix (defines the global index). */
void pbgen_fill_host(float* dst, long long row0, long long row1, long long cols, long long ld,
                     unsigned long long seed, unsigned long long stream, int mode,
                     double scale, double offset) {
  int sym = (mode & PBGEN_SYM) != 0;
  int m = mode & 0xff;
#pragma omp parallel for schedule(static)
  for (long long r = row0; r < row1; ++r) {
    for (long long c = 0; c < cols; ++c) {
      long long i = r, j = c;
      if (sym && j > i) { long long t = i; i = j; j = t; }
      uint64_t z = pbgen_bits(seed, stream, (uint64_t)(i * ld + j));
      double v = pbgen_base(z, m);
      double p = v * scale;
      double s = p + offset;
      dst[(r - row0) * cols + c] = (float)s;
    }
  }
}
