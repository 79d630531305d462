// pb_check.h — host-side argument validation and workspace carving shared by the
// entry points of pb_api.cu and pb_dist.cu (not part of the public ABI).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <initializer_list>
#include <string>
#include <vector>

#include "../../include/pb.h"
#include "pb_internal.h"

namespace pb {

// Records a thread-local message for pb_last_error() and returns st.
pb_status fail(pb_status st, const char* fmt, ...);
// Sets what pb_last_launch_count() reports for the current call.
void set_launches(int n);
// pb_workspace_size for the multi-GPU entry points ("<k>_dist"), pb_dist.cu.
pb_status dist_workspace_size(const std::string& name, const long long* d, int nd, size_t* bytes);

struct Range {
  const void* p;
  size_t bytes;
  bool out;
  const char* name;
};

// Validation context for one call: collects pointer ranges, checks placement,
// alignment and aliasing (outputs may not overlap anything else).
struct Check {
  std::vector<Range> r;
  pb_status st = PB_OK;
  int dev = -1;

  Check() { cudaGetDevice(&dev); }

  void arr(const void* p, long long rows, long long cols, bool out, const char* name, bool required = true) {
    if (st != PB_OK) return;
    if (p == nullptr) {
      if (required) st = fail(PB_ERR_INVALID_ARG, "%s is NULL", name);
      return;
    }
    if (reinterpret_cast<uintptr_t>(p) % 16 != 0) {
      st = fail(PB_ERR_UNSUPPORTED, "%s is not 16-byte aligned", name);
      return;
    }
    cudaPointerAttributes at;
    cudaError_t e = cudaPointerGetAttributes(&at, p);
    if (e != cudaSuccess) {
      cudaGetLastError();
      st = fail(PB_ERR_INVALID_ARG, "%s: cudaPointerGetAttributes failed (%s)", name, cudaGetErrorString(e));
      return;
    }
    if (!(at.type == cudaMemoryTypeDevice || at.type == cudaMemoryTypeManaged) || at.device != dev) {
      st = fail(PB_ERR_INVALID_ARG, "%s is not device memory on the current device", name);
      return;
    }
    r.push_back({p, (size_t)(rows * cols) * sizeof(float), out, name});
  }
  void cols4(long long cols, const char* name) {
    if (st == PB_OK && cols % 4 != 0) st = fail(PB_ERR_UNSUPPORTED, "%s: column count %lld not a multiple of 4", name, cols);
  }
  void dims(std::initializer_list<long long> ds) {
    if (st != PB_OK) return;
    for (long long d : ds)
      if (d <= 0 || d > (1ll << 30)) {
        st = fail(PB_ERR_INVALID_ARG, "dimension %lld out of range", d);
        return;
      }
  }
  pb_status finish() {
    if (st != PB_OK) return st;
    for (size_t i = 0; i < r.size(); ++i) {
      if (!r[i].out) continue;
      const char* a0 = static_cast<const char*>(r[i].p);
      const char* a1 = a0 + r[i].bytes;
      for (size_t j = 0; j < r.size(); ++j) {
        if (j == i) continue;
        const char* b0 = static_cast<const char*>(r[j].p);
        const char* b1 = b0 + r[j].bytes;
        if (a0 < b1 && b0 < a1) return st = fail(PB_ERR_ALIAS, "%s overlaps %s", r[i].name, r[j].name);
      }
    }
    return PB_OK;
  }
};

// Bump allocator over the caller's workspace (256-B aligned slices).
struct Carve {
  char* base;
  size_t cap, off = 0;
  Carve(void* b, size_t c) : base(static_cast<char*>(b)), cap(c) {}
  template <class T>
  T* take(size_t count) {
    off = align_up(off, 256);
    T* p = reinterpret_cast<T*>(base ? base + off : nullptr);
    off += count * sizeof(T);
    return p;
  }
};

}  // namespace pb
