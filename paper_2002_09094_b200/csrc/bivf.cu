// Bitmap-block inverted file (BIVF) of the means — the B200 layout of
// MeanSet.inverted (reference means.py:169-179, InvertedFile data.py:237-300).
//
// The reference stores term-major postings (owner id int32, value float64)
// with owners ascending inside each term.  Here the owner ids are replaced by
// one 32-bit presence mask per (term, 32-mean block) plus the offset of the
// block's first value; values keep the reference order (term-major, mean
// ascending).  A warp lane that owns mean 32*b+lane finds its posting of term
// t with one header load and a popcount, so the assign kernel accumulates in
// registers with no shared-memory scatter, no bank conflicts and no atomics,
// and the exact rescoring looks a (term, mean) value up in O(1).
//
// Build (no sort needed): atomicOr the masks, exclusive-scan the popcounts
// into offsets, scatter each value to offset + popc(mask below its bit).
#include <cub/cub.cuh>

#include "common.cuh"

using namespace ivfkm;

extern "C" int64_t ivfkm_bivf_nblk(int64_t k) {
  int64_t b = (k + 31) / 32;
  return (b + 7) / 8 * 8;
}

namespace {

struct BivfWs {
  unsigned int* err;
  unsigned int* cnt;
  unsigned int* off;
  void* cub;
  size_t cub_bytes;
};

size_t cub_scan_bytes(int64_t n) {
  size_t b = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, b, (unsigned int*)nullptr, (unsigned int*)nullptr,
                                (int)n);
  return b;
}

BivfWs carve(void* base, int64_t dim, int64_t k, size_t* total) {
  const int64_t nh = dim * ivfkm_bivf_nblk(k);
  Carver c(base);
  BivfWs w;
  w.err = c.take<unsigned int>(4);
  w.cnt = c.take<unsigned int>(nh + 1);
  w.off = c.take<unsigned int>(nh + 1);
  w.cub_bytes = cub_scan_bytes(nh + 1);
  w.cub = c.take_bytes(w.cub_bytes);
  if (total) *total = c.off;
  return w;
}

// Row owning entry q of a CSR with nrows rows: the last r with ptr[r] <= q.
__device__ __forceinline__ int64_t row_of(const int64_t* __restrict__ ptr, int64_t nrows,
                                          int64_t q) {
  int64_t lo = 0, hi = nrows;  // ptr[lo] <= q < ptr[hi]
  while (hi - lo > 1) {
    const int64_t mid = (lo + hi) >> 1;
    if (__ldg(ptr + mid) <= q) lo = mid; else hi = mid;
  }
  return lo;
}

__device__ __forceinline__ int64_t nh_of(int64_t dim, int64_t nblk) { return dim * nblk; }

// One thread per entry (grid-stride), so a few long rows (k means holding
// ~20k terms each) still spread over the whole GPU.
__global__ void bivf_mask_kernel(int major, int64_t nrows, const int64_t* __restrict__ ptr,
                                 const int32_t* __restrict__ cols, int64_t k, int64_t dim,
                                 int64_t nblk, unsigned int* __restrict__ hdr,
                                 unsigned int* __restrict__ err) {
  const int64_t nnz = ptr[nrows];
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < nnz;
       q += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = row_of(ptr, nrows, q);
    const int64_t col = cols[q];
    const int64_t c = major == 0 ? r : col;
    const int64_t t = major == 0 ? col : r;
    if (c < 0 || c >= k || t < 0 || t >= dim) {
      atomicAdd(err, 1u);
      continue;
    }
    atomicOr(&hdr[t * nblk + (c >> 5)], 1u << (c & 31));
  }
}

__global__ void bivf_popc_kernel(int64_t nh, const unsigned int* __restrict__ hdr,
                                 unsigned int* __restrict__ cnt) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i <= nh;
       i += (int64_t)gridDim.x * blockDim.x)
    cnt[i] = i < nh ? __popc(hdr[i]) : 0u;
}

__global__ void bivf_offset_kernel(int64_t nh, const unsigned int* __restrict__ off,
                                   unsigned int* __restrict__ hdr) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i <= nh;
       i += (int64_t)gridDim.x * blockDim.x)
    hdr[nh + i] = off[i];
}

__global__ void bivf_scatter_kernel(int major, int64_t nrows, const int64_t* __restrict__ ptr,
                                    const int32_t* __restrict__ cols,
                                    const double* __restrict__ vals, int64_t k, int64_t dim,
                                    int64_t nblk, const unsigned int* __restrict__ hdr,
                                    float* __restrict__ v32, double* __restrict__ v64) {
  const int64_t nnz = ptr[nrows];
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < nnz;
       q += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = row_of(ptr, nrows, q);
    const int64_t col = cols[q];
    const int64_t c = major == 0 ? r : col;
    const int64_t t = major == 0 ? col : r;
    if (c < 0 || c >= k || t < 0 || t >= dim) continue;
    const int64_t hb = t * nblk + (c >> 5);
    const unsigned pos = hdr[nh_of(dim, nblk) + hb] + __popc(hdr[hb] & ((1u << (c & 31)) - 1u));
    const double v = vals[q];
    v32[pos] = static_cast<float>(v);
    v64[pos] = v;
  }
}

}  // namespace

extern "C" size_t ivfkm_bivf_workspace_size(int64_t dim, int64_t k) {
  size_t total = 0;
  carve(nullptr, dim, k, &total);
  return total;
}

extern "C" int ivfkm_bivf_build(int64_t k, int64_t dim, int major, int64_t nrows,
                                const int64_t* ptr, const int32_t* cols, const double* vals,
                                uint32_t* headers, float* val32, double* val64, void* ws,
                                size_t ws_bytes, ivfkm_stream_t stream_) {
  if (k < 1 || dim < 1 || nrows < 0 || (major != 0 && major != 1) || !ptr || !headers)
    return IVFKM_E_ARG;
  const int64_t nblk = ivfkm_bivf_nblk(k);
  const int64_t nh = dim * nblk;
  if (nh + 1 > INT32_MAX) return IVFKM_E_UNSUPPORTED;  // cub scan length
  size_t need = 0;
  BivfWs w = carve(ws, dim, k, &need);
  if (ws_bytes < need) return IVFKM_E_WORKSPACE;
  cudaStream_t st = as_stream(stream_);
  IVFKM_TRY(cudaMemsetAsync(headers, 0, sizeof(uint32_t) * nh, st));
  IVFKM_TRY(cudaMemsetAsync(w.err, 0, sizeof(unsigned int), st));
  const int threads = 256;
  bivf_mask_kernel<<<kNumSM * 8, threads, 0, st>>>(
      major, nrows, ptr, cols, k, dim, nblk, headers, w.err);
  IVFKM_CHECK_LAUNCH();
  bivf_popc_kernel<<<grid_for(nh + 1, threads), threads, 0, st>>>(nh, headers, w.cnt);
  IVFKM_CHECK_LAUNCH();
  size_t cb = w.cub_bytes;
  IVFKM_TRY(cub::DeviceScan::ExclusiveSum(w.cub, cb, w.cnt, w.off, (int)(nh + 1), st));
  bivf_offset_kernel<<<grid_for(nh + 1, threads), threads, 0, st>>>(nh, w.off, headers);
  IVFKM_CHECK_LAUNCH();
  bivf_scatter_kernel<<<kNumSM * 8, threads, 0, st>>>(
      major, nrows, ptr, cols, vals, k, dim, nblk, headers, val32, val64);
  IVFKM_CHECK_LAUNCH();
  return IVFKM_OK;
}
