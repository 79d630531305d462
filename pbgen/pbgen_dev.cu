// pbgen_dev.cu — device side of the shared input generator (see pbgen_core.h).
// Used by the GPU harness (tests, bench) to create inputs resident in HBM; the
// values are bit-identical to pbgen_fill_host (checked in tests/test_gpu_parity.py).
#include <cuda_runtime.h>
#include "pbgen_core.h"

__global__ void pbgen_fill_kernel(float* __restrict__ dst, long long row0, long long rows,
                                  long long cols, long long ld, unsigned long long seed,
                                  unsigned long long stream, int mode, double scale,
                                  double offset) {
  const int sym = (mode & PBGEN_SYM) != 0;
  const int m = mode & 0xff;
  const long long total = rows * cols;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    long long i = row0 + e / cols, j = e % cols;
    if (sym && j > i) { long long t = i; i = j; j = t; }
    uint64_t z = pbgen_bits(seed, stream, (uint64_t)(i * ld + j));
    double v = pbgen_base(z, m);
    double s = __dadd_rn(__dmul_rn(v, scale), offset);
    dst[e] = (float)s;  // cvt.rn.f32.f64, same as the host's (float) cast
  }
}

extern "C" int pbgen_fill_device(float* dst, long long row0, long long row1, long long cols,
                                 long long ld, unsigned long long seed, unsigned long long stream,
                                 int mode, double scale, double offset, void* cuda_stream) {
  long long rows = row1 - row0;
  if (rows <= 0 || cols <= 0) return 0;
  long long total = rows * cols;
  long long blocks = (total + 255) / 256;
  if (blocks > 148 * 64) blocks = 148 * 64;
  pbgen_fill_kernel<<<(unsigned)blocks, 256, 0, (cudaStream_t)cuda_stream>>>(
      dst, row0, rows, cols, ld, seed, stream, mode, scale, offset);
  return (int)cudaGetLastError();
}
