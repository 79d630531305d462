// pb_umma.cuh — tcgen05 / TMA helpers shared by the 3xTF32 GEMM engine (k_umma.cu)
// and the fused covariance / correlation kernel (k_gram.cu). Product code.
#pragma once
#include "pb_device.cuh"

namespace pb {

// ---- cta_group-specific PTX (CG = 1: one CTA; CG = 2: an SM pair, cta_group::2)
template <int CG>
__device__ __forceinline__ void tmem_alloc_cg(uint32_t* dst, uint32_t ncols) {
  if constexpr (CG == 1) {
    tmem_alloc(dst, ncols);
  } else {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(dst)), "r"(ncols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
  }
}
template <int CG>
__device__ __forceinline__ void tmem_dealloc_cg(uint32_t taddr, uint32_t ncols) {
  if constexpr (CG == 1)
    tmem_dealloc(taddr, ncols);
  else
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols) : "memory");
}
template <int CG>
__device__ __forceinline__ void mma_cg(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  if constexpr (CG == 1) {
    mma_tf32(d, a, b, idesc, acc);
  } else {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::2.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
        "l"(a), "l"(b), "r"(idesc), "r"(acc)
        : "memory");
  }
}
// Commit this thread's MMAs to `bar` (CG=2: the barrier at the same offset in both CTAs).
template <int CG>
__device__ __forceinline__ void commit_cg(uint64_t* bar) {
  if constexpr (CG == 1) {
    mma_commit(bar);
  } else {
    asm volatile(
        "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
            smem_u32(bar)),
        "h"((uint16_t)3)
        : "memory");
  }
}
// TMA tile load; CG=2: completion is counted on the LEADER CTA's barrier.
template <int CG>
__device__ __forceinline__ void tma_load_cg(const CUtensorMap* m, uint64_t* bar, void* dst, int c0, int c1) {
  if constexpr (CG == 1) {
    tma_load_2d(m, bar, dst, c0, c1);
  } else {
    asm volatile(
        "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, "
        "%4}], [%2];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(m)), "r"(smem_u32(bar) & 0xFEFFFFFFu), "r"(c0), "r"(c1)
        : "memory");
  }
}


}  // namespace pb
