/* pbgen_core.h — the counter-based input generator shared by the oracle
 * harness (host) and the GPU harness (device).
 *
 * This module holds NO PolyBench arithmetic: it only maps a global element
 * index to a pseudo-random fp32 value, so that the CPU oracle and the CUDA
 * path can be fed bit-identical inputs without either one producing the
 * other's inputs (task rule ③; recipe in DESIGN.md §"Input recipe", after
 * SURVEY.md §8(d) "Input generator").
 *
 *   z   = splitmix64(seed*0x9E3779B97F4A7C15 + stream*0xD1B54A32D192ED03 + idx)
 *   u01 = (z >> 40) * 2^-24            in [0,1), 24 significant bits (exact in fp32)
 *   int = z >> 61                      in {0..7}
 *   bin = z >> 63                      in {0,1}
 *   value = (float)( base * scale + offset )   computed in double, RN
 *
 * idx is the GLOBAL row-major element index (row*ld + col), so a row shard
 * generated on its own is bit-identical to the same rows of the full matrix.
 * With PBGEN_SYM the index is max(i,j)*ld + min(i,j) (a symmetric matrix).
 */
#ifndef PBGEN_CORE_H
#define PBGEN_CORE_H
#include <stdint.h>

#ifdef __CUDACC__
#define PBGEN_FN __host__ __device__ static inline
#else
#define PBGEN_FN static inline
#endif

enum { PBGEN_U01 = 0, PBGEN_INT8 = 1, PBGEN_BIN = 2 };
enum { PBGEN_SYM = 1 << 8 };

PBGEN_FN uint64_t pbgen_splitmix64(uint64_t x) {
  uint64_t z = x + 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

PBGEN_FN uint64_t pbgen_bits(uint64_t seed, uint64_t stream, uint64_t idx) {
  return pbgen_splitmix64(seed * 0x9E3779B97F4A7C15ull + stream * 0xD1B54A32D192ED03ull + idx);
}

/* base value in double (exact): u01, small int, or bit */
PBGEN_FN double pbgen_base(uint64_t z, int mode) {
  if (mode == PBGEN_INT8) return (double)(z >> 61);
  if (mode == PBGEN_BIN) return (double)(z >> 63);
  return (double)(z >> 40) * (1.0 / 16777216.0);
}

#endif
