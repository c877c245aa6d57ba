// Shared helpers for the ivfkm CUDA sources (sm_100a).
#pragma once
#include <cuda_runtime.h>
#include <cstddef>
#include <cstdint>

#include "ivfkm.h"

#define IVFKM_TRY(expr)                                  \
  do {                                                   \
    cudaError_t e_ = (expr);                             \
    if (e_ != cudaSuccess) return static_cast<int>(e_);  \
  } while (0)

#define IVFKM_TRY_RC(expr)         \
  do {                             \
    int rc_ = (expr);              \
    if (rc_ != 0) return rc_;      \
  } while (0)

#define IVFKM_CHECK_LAUNCH() IVFKM_TRY(cudaGetLastError())

namespace ivfkm {

constexpr unsigned kFull = 0xffffffffu;

// SMs of the current device (148 on a B200), queried once per device; grids
// are sized as multiples of it.
inline int num_sms() {
  static int cache[64] = {0};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return 148;
  if (!cache[dev]) {
    int n = 0;
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n < 1)
      n = 148;
    cache[dev] = n;
  }
  return cache[dev];
}

inline cudaStream_t as_stream(ivfkm_stream_t s) { return reinterpret_cast<cudaStream_t>(s); }

// Bump allocator over a caller-provided workspace.  With base == nullptr it
// only measures, so *_workspace_size() and the real carve share one code path.
struct Carver {
  char* base;
  size_t off = 0;
  explicit Carver(void* b) : base(static_cast<char*>(b)) {}
  template <class T>
  T* take(size_t count, size_t align = 256) {
    off = (off + align - 1) / align * align;
    T* p = base ? reinterpret_cast<T*>(base + off) : nullptr;
    off += count * sizeof(T);
    return p;
  }
  void* take_bytes(size_t bytes, size_t align = 256) { return take<char>(bytes, align); }
};

inline int grid_for(int64_t items, int per_block, int max_blocks = 0) {
  if (max_blocks <= 0) max_blocks = num_sms() * 32;
  int64_t g = (items + per_block - 1) / per_block;
  if (g < 1) g = 1;
  if (g > max_blocks) g = max_blocks;
  return static_cast<int>(g);
}

}  // namespace ivfkm
