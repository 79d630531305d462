// k_umma.cu — the 3xTF32 tcgen05 GEMM engine behind gemm / 2mm / 3mm / syrk /
// syr2k and the Gram core of covariance / correlation.
//
// Paper mapping:
//  * Loop internalization (Listing 9 at PAPER.md:404-428):
//    the per-work-item k-loop over global memory becomes a k-block loop over
//    shared-memory tiles. Here a TMA producer warp stages 128x32 fp32 tiles of
//    the hi/lo operands into a STAGES-deep smem ring; mbarriers play the role
//    of Listing 9's two group_barriers (full = "tile loaded", empty = "tile
//    consumed"), so loads of block k+1.. overlap the math on block k.
//  * Detect reduction (Listings 4-5): C[i][j] is never
//    re-read/re-written inside the k-loop; the running sum lives in a TMEM
//    accumulator (tcgen05.mma, fp32) and is written once by the epilogue.
//  * Uniformity: every barrier/mbarrier wait sits in
//    warp-uniform control flow; tails are zero-filled by TMA, not branched.
//
// Precision: x = hi + lo with hi = tf32_rna(x), lo = tf32_rna(x - hi) (split
// done by k_split.cu); acc += a_hi*b_hi + a_hi*b_lo + a_lo*b_hi (lo*lo dropped).
//
// CTA layout (192 threads, 1 CTA/SM, persistent over tiles):
//   warp 0      TMA producer (one lane)
//   warp 1      TMEM allocator + MMA issuer (one lane)
//   warps 2..5  epilogue: tcgen05.ld (warp%4 selects its 32 TMEM lanes), alpha/beta,
//               masks, fp32 / split / mirrored stores
// Tiles 128 x 128 (UMMA M=128, N=128, K=8 per instruction), BK = 32 (one 128-B
// swizzle row of fp32), 3-stage ring of {A_hi, A_lo, B_hi, B_lo} = 64 KiB/stage,
// two TMEM accumulator slots (2 x {big, small} x 128 columns = all 512) that
// alternate per 512-wide K chunk; the epilogue promotes each chunk into fp32
// registers (RN) so the tensor core's truncating accumulate cannot bias long K.
#include <math.h>

#include "pb_device.cuh"
#include "pb_internal.h"

namespace pb {
namespace {

constexpr int BM = 128;
constexpr int BN = 128;
constexpr int BK = 32;
constexpr int STAGES = 3;
constexpr int TILE_BYTES = BM * BK * 4;          // 16 KiB per operand tile
constexpr int STAGE_BYTES = 4 * TILE_BYTES;      // A_hi, A_lo, B_hi, B_lo
constexpr int NUM_THREADS = 192;
constexpr int GROUP_M = 8;                       // tile-rows per raster group (L2 reuse)
constexpr uint32_t TMEM_COLS = 4 * BN;  // 2 slots x {big, small} accumulators = 512 columns
constexpr int CHUNK_KB = 16;            // k-blocks (16 x 32 = 512 of K) per TMEM partial sum

struct Params {
  int M, N, K, npairs, nkb;  // nkb = k-blocks per pair
  uint32_t flags;
  float alpha, beta;
  const float* cin;
  int ldc;
  float* out;
  int ldo;
  int out_row0;
  float* split_hi;
  float* split_lo;
  int ld_split;
  int tm0, tm1, tiles_n;
  long long num_tiles;
};

struct __align__(8) Ctl {
  uint64_t full[STAGES];
  uint64_t empty[STAGES];
  uint64_t tfull[2];
  uint64_t tempty[2];
  uint32_t tmem_base;
};

__device__ __forceinline__ long long tri_count(long long r) { return r * (r + 1) / 2; }

// Tile t of the persistent schedule -> (tm, tn). Raster: groups of GROUP_M
// tile-rows; inside a group tn is the outer index so CTAs running together
// share B panels (and the GROUP_M A panels) in L2.
__device__ void tile_coords(const Params& p, long long t, int& tm, int& tn) {
  const bool tri = (p.flags & EPI_TRI) != 0;
  int g0 = p.tm0;
  for (;;) {
    int g1 = min(g0 + GROUP_M, p.tm1);
    long long cnt = tri ? (tri_count(g1) - tri_count(g0)) : (long long)(g1 - g0) * p.tiles_n;
    if (t < cnt || g1 >= p.tm1) {
      int gs = g1 - g0;
      if (!tri) {
        tn = (int)(t / gs);
        tm = g0 + (int)(t % gs);
      } else if (t < (long long)g0 * gs) {  // columns left of the group's diagonal block: full height
        tn = (int)(t / gs);
        tm = g0 + (int)(t % gs);
      } else {                              // diagonal block: column c has rows [c, g1)
        t -= (long long)g0 * gs;
        int c = g0;
        while (t >= g1 - c) {
          t -= g1 - c;
          ++c;
        }
        tn = c;
        tm = c + (int)t;
      }
      return;
    }
    t -= cnt;
    g0 = g1;
  }
}

__device__ __forceinline__ void store4(float* p, float a, float b, float c, float d) {
  *reinterpret_cast<float4*>(p) = make_float4(a, b, c, d);
}

__global__ void __launch_bounds__(NUM_THREADS, 1)
    umma3x_kernel(const __grid_constant__ CUtensorMap a0h, const __grid_constant__ CUtensorMap a0l,
                  const __grid_constant__ CUtensorMap b0h, const __grid_constant__ CUtensorMap b0l,
                  const __grid_constant__ CUtensorMap a1h, const __grid_constant__ CUtensorMap a1l,
                  const __grid_constant__ CUtensorMap b1h, const __grid_constant__ CUtensorMap b1l,
                  const Params p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  Ctl* ctl = reinterpret_cast<Ctl*>(smem + STAGES * STAGE_BYTES);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&ctl->full[s], 1);
      mbar_init(&ctl->empty[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&ctl->tfull[s], 1);
      mbar_init(&ctl->tempty[s], 4);  // one arrive per epilogue warp
    }
    fence_mbar_init();
  }
  if (warp == 0 && lane == 0) {
    tma_prefetch(&a0h); tma_prefetch(&a0l); tma_prefetch(&b0h); tma_prefetch(&b0l);
    if (p.npairs > 1) { tma_prefetch(&a1h); tma_prefetch(&a1l); tma_prefetch(&b1h); tma_prefetch(&b1l); }
  }
  if (warp == 1) tmem_alloc(&ctl->tmem_base, TMEM_COLS);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = ctl->tmem_base;
  const int nkb_total = p.nkb * p.npairs;

  if (warp == 0) {
    // ===================== TMA producer =====================
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (long long t = blockIdx.x; t < p.num_tiles; t += gridDim.x) {
        int tm, tn;
        tile_coords(p, t, tm, tn);
        for (int kb = 0; kb < nkb_total; ++kb) {
          mbar_wait(&ctl->empty[stage], phase ^ 1);
          uint8_t* st = smem + stage * STAGE_BYTES;
          const int pair = kb >= p.nkb;
          const int k = (kb - pair * p.nkb) * BK;
          mbar_arrive_expect_tx(&ctl->full[stage], STAGE_BYTES);
          tma_load_2d(pair ? &a1h : &a0h, &ctl->full[stage], st + 0 * TILE_BYTES, k, tm * BM);
          tma_load_2d(pair ? &a1l : &a0l, &ctl->full[stage], st + 1 * TILE_BYTES, k, tm * BM);
          tma_load_2d(pair ? &b1h : &b0h, &ctl->full[stage], st + 2 * TILE_BYTES, k, tn * BN);
          tma_load_2d(pair ? &b1l : &b0l, &ctl->full[stage], st + 3 * TILE_BYTES, k, tn * BN);
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    // ===================== MMA issuer =====================
    // The k-loop of a tile is cut into chunks of CHUNK_KB k-blocks. Each chunk
    // accumulates into one of two TMEM slots; the epilogue warps drain a
    // finished slot into fp32 registers (round-to-nearest adds) while the next
    // chunk runs in the other slot. The tensor-core accumulate truncates, so
    // this bounds the truncation bias to one chunk.
    if (lane == 0) {
      constexpr uint32_t idesc = idesc_tf32(BM, BN);
      int stage = 0;
      uint32_t phase = 0;
      int chunk_it = 0;
      for (long long t = blockIdx.x; t < p.num_tiles; t += gridDim.x) {
        for (int kb0 = 0; kb0 < nkb_total; kb0 += CHUNK_KB, ++chunk_it) {
          const int slot = chunk_it & 1;
          const uint32_t slot_phase = (chunk_it >> 1) & 1;
          mbar_wait(&ctl->tempty[slot], slot_phase ^ 1);  // epilogue drained this slot
          tc_fence_after();
          // `big` takes a_hi*b_hi, `small` the cross terms a_hi*b_lo + a_lo*b_hi
          // (2^-11 smaller): the small terms are rounded at their own scale.
          const uint32_t d_big = tmem_base + slot * 2 * BN;
          const uint32_t d_small = d_big + BN;
          const int kb1 = min(kb0 + CHUNK_KB, nkb_total);
          for (int kb = kb0; kb < kb1; ++kb) {
            mbar_wait(&ctl->full[stage], phase);
            tc_fence_after();
            const uint32_t st = smem_u32(smem + stage * STAGE_BYTES);
#pragma unroll
            for (int kk = 0; kk < BK / 8; ++kk) {
              const uint64_t ah = umma_desc_k_sw128(st + 0 * TILE_BYTES + kk * 32);
              const uint64_t al = umma_desc_k_sw128(st + 1 * TILE_BYTES + kk * 32);
              const uint64_t bh = umma_desc_k_sw128(st + 2 * TILE_BYTES + kk * 32);
              const uint64_t bl = umma_desc_k_sw128(st + 3 * TILE_BYTES + kk * 32);
              const uint32_t accum = (kb > kb0 || kk > 0) ? 1u : 0u;
              mma_tf32(d_small, al, bh, idesc, accum);
              mma_tf32(d_small, ah, bl, idesc, 1);
              mma_tf32(d_big, ah, bh, idesc, accum);
            }
            mma_commit(&ctl->empty[stage]);  // frees the smem stage when these MMAs finish
            if (++stage == STAGES) { stage = 0; phase ^= 1; }
          }
          mma_commit(&ctl->tfull[slot]);  // chunk partial sums ready for the epilogue
        }
      }
    }
  } else {
    // ===================== epilogue (warps 2..5) =====================
    const int q = warp & 3;  // TMEM lane quarter this warp may access
    const uint32_t flags = p.flags;
    int chunk_it = 0;
    for (long long t = blockIdx.x; t < p.num_tiles; t += gridDim.x) {
      int tm, tn;
      tile_coords(p, t, tm, tn);
      float acc[BN];  // this thread's output row of the tile, fp32 registers
#pragma unroll
      for (int c = 0; c < BN; ++c) acc[c] = 0.f;
      for (int kb0 = 0; kb0 < nkb_total; kb0 += CHUNK_KB, ++chunk_it) {
        const int slot = chunk_it & 1;
        const uint32_t slot_phase = (chunk_it >> 1) & 1;
        mbar_wait(&ctl->tfull[slot], slot_phase);
        tc_fence_after();
        __syncwarp();
        const uint32_t ta = tmem_base + ((uint32_t)(q * 32) << 16) + slot * 2 * BN;
#pragma unroll
        for (int c0 = 0; c0 < BN; c0 += 16) {
          uint32_t r[16], rs[16];
          tmem_ld16(ta + c0, r);
          tmem_ld16(ta + BN + c0, rs);
          tmem_wait_ld();
#pragma unroll
          for (int e = 0; e < 16; ++e) acc[c0 + e] += __uint_as_float(r[e]) + __uint_as_float(rs[e]);
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&ctl->tempty[slot]);
      }
      const int i = tm * BM + q * 32 + lane;  // output row (operand-a space)
      const bool row_ok = i < p.M;
      const bool diag_tile = (flags & EPI_TRI) && tm == tn;
      const long long orow = (long long)(i - p.out_row0);
#pragma unroll
      for (int c0 = 0; c0 < BN; c0 += 16) {
        const int j0 = tn * BN + c0;
        if (row_ok && j0 < p.N) {
          float v[16];
#pragma unroll
          for (int e = 0; e < 16; ++e) v[e] = p.alpha * acc[c0 + e];
          if (flags & EPI_CIN) {
            const float* cp = p.cin + orow * p.ldc + j0;
#pragma unroll
            for (int e = 0; e < 16; e += 4) {
              if (j0 + e < p.N) {
                float4 c = *reinterpret_cast<const float4*>(cp + e);
                v[e] += p.beta * c.x; v[e + 1] += p.beta * c.y; v[e + 2] += p.beta * c.z; v[e + 3] += p.beta * c.w;
              }
            }
          }
          if (flags & EPI_DIAG_ONE) {
#pragma unroll
            for (int e = 0; e < 16; ++e)
              if (j0 + e == i) v[e] = 1.0f;
          }
          if (!diag_tile) {
            if (flags & EPI_OUT) {
              float* op = p.out + orow * p.ldo + j0;
#pragma unroll
              for (int e = 0; e < 16; e += 4)
                if (j0 + e < p.N) store4(op + e, v[e], v[e + 1], v[e + 2], v[e + 3]);
            }
            if (flags & EPI_SPLIT) {
              float* hp = p.split_hi + (long long)i * p.ld_split + j0;
              float* lp = p.split_lo + (long long)i * p.ld_split + j0;
#pragma unroll
              for (int e = 0; e < 16; e += 4) {
                if (j0 + e < p.N) {
                  float h[4], l[4];
#pragma unroll
                  for (int u = 0; u < 4; ++u) split3x(v[e + u], h[u], l[u]);
                  store4(hp + e, h[0], h[1], h[2], h[3]);
                  store4(lp + e, l[0], l[1], l[2], l[3]);
                }
              }
            }
          } else {  // lower-triangular diagonal tile: element mask j <= i
            if (flags & EPI_OUT) {
              float* op = p.out + orow * p.ldo + j0;
#pragma unroll
              for (int e = 0; e < 16; ++e)
                if (j0 + e < p.N && j0 + e <= i) op[e] = v[e];
            }
          }
          if (flags & EPI_MIRROR) {  // out[j][i] = v for j < i
#pragma unroll
            for (int e = 0; e < 16; ++e) {
              const int j = j0 + e;
              if (j < p.N && j < i) p.out[(long long)(j - p.out_row0) * p.ldo + i] = v[e];
            }
          }
          if (flags & EPI_SPLIT_T) {
#pragma unroll
            for (int e = 0; e < 16; ++e) {
              const int j = j0 + e;
              if (j < p.N) {
                float h, l;
                split3x(v[e], h, l);
                p.split_hi[(long long)j * p.ld_split + i] = h;
                p.split_lo[(long long)j * p.ld_split + i] = l;
              }
            }
          }
        }
      }
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem_base, TMEM_COLS);
  }
}

// ---------------------------------------------------------------- host side
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn get_encode() {
  static EncodeTiledFn fn = nullptr;
  if (!fn) {
    void* ptr = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(ptr);
  }
  return fn;
}

// K-major operand (rows x K, pitch ld floats), box = 32 (K) x 128 (rows), 128-B swizzle.
bool make_map(CUtensorMap* m, const float* base, int rows, int K, int ld) {
  EncodeTiledFn enc = get_encode();
  if (!enc) return false;
  cuuint64_t dims[2] = {(cuuint64_t)K, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)ld * 4};
  cuuint32_t box[2] = {(cuuint32_t)BK, (cuuint32_t)BM};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(base), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

int num_sms() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

}  // namespace

cudaError_t launch_umma_gemm(const GemmDesc& d, cudaStream_t s, int* launches) {
  Params p{};
  p.M = d.M;
  p.N = d.N;
  p.K = d.K;
  p.npairs = d.npairs;
  p.nkb = (d.K + BK - 1) / BK;
  p.flags = d.flags;
  p.alpha = d.alpha;
  p.beta = d.beta;
  p.cin = d.cin;
  p.ldc = d.ldc;
  p.out = d.out;
  p.ldo = d.ldo;
  p.out_row0 = d.out_row0;
  p.split_hi = d.split_hi;
  p.split_lo = d.split_lo;
  p.ld_split = d.ld_split;
  const int tiles_m = (d.M + BM - 1) / BM;
  p.tiles_n = (d.N + BN - 1) / BN;
  p.tm0 = d.tm0;
  p.tm1 = d.tm1 < 0 ? tiles_m : d.tm1;
  if (p.tm1 <= p.tm0) return cudaSuccess;
  if (d.flags & EPI_TRI) {
    p.num_tiles = (long long)p.tm1 * (p.tm1 + 1) / 2 - (long long)p.tm0 * (p.tm0 + 1) / 2;
  } else {
    p.num_tiles = (long long)(p.tm1 - p.tm0) * p.tiles_n;
  }
  CUtensorMap maps[8];
  for (int q = 0; q < 2; ++q) {
    const SplitOperand& A = d.a[q < d.npairs ? q : 0];
    const SplitOperand& B = d.b[q < d.npairs ? q : 0];
    if (!make_map(&maps[4 * q + 0], A.hi, A.rows, A.K, A.ld) || !make_map(&maps[4 * q + 1], A.lo, A.rows, A.K, A.ld) ||
        !make_map(&maps[4 * q + 2], B.hi, B.rows, B.K, B.ld) || !make_map(&maps[4 * q + 3], B.lo, B.rows, B.K, B.ld))
      return cudaErrorInvalidValue;
  }
  const size_t smem = STAGES * STAGE_BYTES + 1024 + sizeof(Ctl) + 64;
  static bool attr_set = false;
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(umma3x_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    attr_set = true;
  }
  long long grid = p.num_tiles < num_sms() ? p.num_tiles : num_sms();
  umma3x_kernel<<<(unsigned)grid, NUM_THREADS, smem, s>>>(maps[0], maps[1], maps[2], maps[3], maps[4], maps[5],
                                                          maps[6], maps[7], p);
  if (launches) ++*launches;
  return cudaGetLastError();
}

}  // namespace pb
