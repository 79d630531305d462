// k_peer.cu — fused peer-memory collectives: the
// reduce-scatter of atax/bicg/mvt's transposed-product partials and 3mm's
// all-gather of F, done with stores straight into the other ranks' memory
// (CUDA IPC mappings: NVLink/NVSwitch P2P between GPUs, or one GPU shared by
// several processes) instead of NCCL's multi-step protocols.
//
// Every rank owns one symmetric buffer: a header (flags[src], acks[src], two
// grid counters, a status word, the epoch) and a data region. A collective with
// epoch e (= the header's epoch + 1, read on the device: graph-replay safe):
//   push    (peer_push_kernel)    every CTA first waits until each destination
//                                 acked epoch e-1 (its data region is free), then
//                                 copies its part of the send data into the
//                                 destinations' data regions; the last CTA fences
//                                 at system scope and release-stores flags[me] = e
//                                 in every destination.
//   consume (peer_consume_kernel) waits until flags[src] >= e for every src
//                                 (acquire), reduces (slots summed in rank order:
//                                 deterministic) or copies the region out, and the
//                                 last CTA release-stores acks[me] = e in every
//                                 source.
// Two kernels, so no grid needs to be co-resident with itself; every wait is
// bounded (status word != 0 afterwards instead of a hang).
#include <algorithm>

#include "pb_device.cuh"
#include "pb_internal.h"

namespace pb {
namespace {

__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_sys(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

constexpr long long SPIN_LIMIT = 1ll << 27;  // ~ seconds with the back-off below

// Thread 0 waits until word[g] >= target for every g < n; on timeout sets *status.
__device__ void wait_all(const unsigned long long* word, int n, unsigned long long target, unsigned* status,
                         unsigned code) {
  if (threadIdx.x == 0) {
    for (int g = 0; g < n; ++g) {
      long long it = 0;
      while (ld_acquire_sys(word + g) < target) {
        __nanosleep(64);
        if (++it > SPIN_LIMIT) {
          atomicExch(status, code);
          break;
        }
      }
    }
  }
  __syncthreads();
}

// Last CTA of the grid (counter reset by that CTA) -> true in every thread of that CTA.
__device__ bool last_cta(unsigned* counter) {
  __shared__ bool last;
  __threadfence_system();
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned prev = atomicAdd(counter, 1u);
    last = prev + 1 == gridDim.x;
    if (last) atomicExch(counter, 0u);
  }
  __syncthreads();
  return last;
}

// The epoch lives in this rank's header (device memory), so captured CUDA graphs
// replay correctly: push and consume both read it at entry; consume's last CTA
// advances it once every source has been acked.
__device__ __forceinline__ unsigned long long next_epoch(const PeerView& v) {
  return *reinterpret_cast<volatile unsigned long long*>(v.epoch) + 1;
}

__global__ void __launch_bounds__(256) peer_push_kernel(PeerView v, PeerPush p) {
  const unsigned long long epoch = next_epoch(v);
  wait_all(v.acks_mine, v.nranks, epoch - 1, v.status, 1u);  // destinations consumed epoch - 1
  const long long tid = blockIdx.x * (long long)blockDim.x + threadIdx.x, nth = (long long)gridDim.x * blockDim.x;
  for (int g = 0; g < v.nranks; ++g) {
    const float4* src = reinterpret_cast<const float4*>(p.src[g]);
    float4* dst = reinterpret_cast<float4*>(v.data[g] + p.dst_off[g]);
    const long long n4 = p.count[g] >> 2;
    for (long long i = tid; i < n4; i += nth) dst[i] = src[i];
  }
  if (last_cta(v.counter + 0) && threadIdx.x < v.nranks)
    st_release_sys(v.flags[threadIdx.x] + v.rank, epoch);  // flags[me] in destination g
}

__global__ void __launch_bounds__(256) peer_consume_kernel(PeerView v, PeerConsume c) {
  const unsigned long long epoch = next_epoch(v);
  wait_all(v.flags_mine, v.nranks, epoch, v.status, 2u);
  const long long tid = blockIdx.x * (long long)blockDim.x + threadIdx.x, nth = (long long)gridDim.x * blockDim.x;
  const float4* base = reinterpret_cast<const float4*>(v.data[v.rank]);
  float4* out = reinterpret_cast<float4*>(c.out);
  const long long n4 = c.count >> 2;
  if (c.reduce) {  // out[i] = sum over sources (rank order) of slot_src[i]
    const long long s4 = c.slot >> 2;
    for (long long i = tid; i < n4; i += nth) {
      float4 a = __ldcv(base + i);
      for (int g = 1; g < v.nranks; ++g) {
        const float4 b = __ldcv(base + g * s4 + i);
        a.x += b.x; a.y += b.y; a.z += b.z; a.w += b.w;
      }
      out[i] = a;
    }
  } else {  // copy the gathered region out
    for (long long i = tid; i < n4; i += nth) out[i] = __ldcv(base + i);
  }
  if (last_cta(v.counter + 1)) {
    if (threadIdx.x < v.nranks) st_release_sys(v.acks[threadIdx.x] + v.rank, epoch);  // acks[me] in source g
    __syncthreads();
    if (threadIdx.x == 0) *v.epoch = epoch;  // the next collective uses epoch + 1
  }
}

}  // namespace

cudaError_t launch_peer_push(const PeerView& v, const PeerPush& p, cudaStream_t s) {
  long long mx = 0;
  for (int g = 0; g < v.nranks; ++g) mx = p.count[g] > mx ? p.count[g] : mx;
  const int grid = (int)std::min<long long>(64, std::max<long long>(1, (mx / 4 + 255) / 256));
  peer_push_kernel<<<grid, 256, 0, s>>>(v, p);
  return cudaGetLastError();
}

cudaError_t launch_peer_consume(const PeerView& v, const PeerConsume& c, cudaStream_t s) {
  const int grid = (int)std::min<long long>(64, std::max<long long>(1, (c.count / 4 + 255) / 256));
  peer_consume_kernel<<<grid, 256, 0, s>>>(v, c);
  return cudaGetLastError();
}

}  // namespace pb
