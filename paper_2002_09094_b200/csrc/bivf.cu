// Bitmap-block inverted file (BIVF) of the means — the B200 layout of
// MeanSet.inverted (reference means.py:169-179, InvertedFile data.py:237-300).
//
// The reference stores term-major postings (owner id int32, value float64)
// with owners ascending inside each term.  Here the owner ids are replaced by
// one 32-bit presence mask per (term, 32-mean block) plus the offset of the
// block's first value (layout and lookup in bivf.cuh).  A warp lane that owns
// mean 32*b+lane finds its posting of term t with one header load and a
// popcount, so the assign kernel accumulates in registers with no
// shared-memory scatter, no bank conflicts and no atomics, and the exact
// rescoring looks a (term, mean) value up in O(1).  Fully populated 256-mean
// spans are stored lane-major so the screen reads them with 16-B loads.
//
// Build (no sort needed): atomicOr the masks; count each span (padded to a
// multiple of 4 values); exclusive-scan into offsets, flag dense spans;
// scatter each value to its slot; per-term posting counts.
#include <cub/cub.cuh>

#include "bivf.cuh"
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

// One thread per (term, span): popcounts of its 8 blocks, the span total
// padded to a multiple of 4 values on the last block.
__global__ void bivf_count_kernel(int64_t nh, const unsigned int* __restrict__ masks,
                                  unsigned int* __restrict__ cnt) {
  const int64_t nspan = nh / kSpan;
  for (int64_t sp = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; sp <= nspan;
       sp += (int64_t)gridDim.x * blockDim.x) {
    if (sp == nspan) {
      cnt[nh] = 0u;
      continue;
    }
    unsigned tot = 0;
#pragma unroll
    for (int r = 0; r < kSpan; ++r) {
      const unsigned c = __popc(masks[sp * kSpan + r]);
      cnt[sp * kSpan + r] = c;
      tot += c;
    }
    cnt[sp * kSpan + kSpan - 1] += (4u - (tot & 3u)) & 3u;
  }
}

__global__ void bivf_offset_kernel(int64_t nh, const unsigned int* __restrict__ off,
                                   unsigned int* __restrict__ hdr) {
  const int64_t nspan = nh / kSpan;
  for (int64_t sp = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; sp <= nspan;
       sp += (int64_t)gridDim.x * blockDim.x) {
    if (sp == nspan) {
      hdr[nh + nh] = off[nh];
      continue;
    }
    bool dense = true;
#pragma unroll
    for (int r = 0; r < kSpan; ++r) dense &= hdr[sp * kSpan + r] == 0xffffffffu;
#pragma unroll
    for (int r = 0; r < kSpan; ++r)
      hdr[nh + sp * kSpan + r] = off[sp * kSpan + r] | (dense ? kDense : 0u);
  }
}

__global__ void bivf_scatter_kernel(int major, int64_t nrows, const int64_t* __restrict__ ptr,
                                    const int32_t* __restrict__ cols,
                                    const double* __restrict__ vals, int64_t k, int64_t dim,
                                    int64_t nblk, const unsigned int* __restrict__ hdr,
                                    float* __restrict__ v32, double* __restrict__ v64) {
  const int64_t nnz = ptr[nrows];
  const int64_t nh = bivf_nh(dim, nblk);
  BivfView view{nblk, hdr, hdr + nh, nullptr};
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < nnz;
       q += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = row_of(ptr, nrows, q);
    const int64_t col = cols[q];
    const int64_t c = major == 0 ? r : col;
    const int64_t t = major == 0 ? col : r;
    if (c < 0 || c >= k || t < 0 || t >= dim) continue;
    const int64_t pos = bivf_find(view, t, c);
    const double v = vals[q];
    v32[pos] = static_cast<float>(v);
    v64[pos] = v;
  }
}

// postings per term: nc[t] = sum_b popc(masks[t][b])
__global__ void bivf_nc_kernel(int64_t dim, int64_t nblk, const unsigned int* __restrict__ masks,
                               unsigned int* __restrict__ nc) {
  const int lane = threadIdx.x & 31;
  const int64_t wpb = blockDim.x >> 5;
  for (int64_t t = blockIdx.x * wpb + (threadIdx.x >> 5); t < dim; t += gridDim.x * wpb) {
    unsigned c = 0;
    for (int64_t b = lane; b < nblk; b += 32) c += __popc(masks[t * nblk + b]);
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) c += __shfl_xor_sync(0xffffffffu, c, off);
    if (lane == 0) nc[t] = c;
  }
}

}  // namespace

extern "C" size_t ivfkm_bivf_workspace_size(int64_t dim, int64_t k) {
  size_t total = 0;
  carve(nullptr, dim, k, &total);
  return total;
}

extern "C" int64_t ivfkm_bivf_headers_size(int64_t k, int64_t dim) {
  return 2 * bivf_nh(dim, ivfkm_bivf_nblk(k)) + 1 + dim;
}

extern "C" int64_t ivfkm_bivf_values_capacity(int64_t k, int64_t dim, int64_t nnz) {
  return nnz + 3 * dim * (ivfkm_bivf_nblk(k) / kSpan) + 4;
}

extern "C" int ivfkm_bivf_build(int64_t k, int64_t dim, int major, int64_t nrows,
                                const int64_t* ptr, const int32_t* cols, const double* vals,
                                uint32_t* headers, float* val32, double* val64, void* ws,
                                size_t ws_bytes, ivfkm_stream_t stream_) {
  if (k < 1 || dim < 1 || nrows < 0 || (major != 0 && major != 1) || !ptr || !headers)
    return IVFKM_E_ARG;
  const int64_t nblk = ivfkm_bivf_nblk(k);
  const int64_t nh = bivf_nh(dim, nblk);
  if (nh + 1 > INT32_MAX) return IVFKM_E_UNSUPPORTED;  // cub scan length, 32-bit rows
  size_t need = 0;
  BivfWs w = carve(ws, dim, k, &need);
  if (ws_bytes < need) return IVFKM_E_WORKSPACE;
  cudaStream_t st = as_stream(stream_);
  IVFKM_TRY(cudaMemsetAsync(headers, 0, sizeof(uint32_t) * nh, st));
  IVFKM_TRY(cudaMemsetAsync(w.err, 0, sizeof(unsigned int), st));
  const int threads = 256;
  bivf_mask_kernel<<<kNumSM * 8, threads, 0, st>>>(major, nrows, ptr, cols, k, dim, nblk,
                                                   headers, w.err);
  IVFKM_CHECK_LAUNCH();
  bivf_count_kernel<<<grid_for(nh / kSpan + 1, threads), threads, 0, st>>>(nh, headers, w.cnt);
  IVFKM_CHECK_LAUNCH();
  size_t cb = w.cub_bytes;
  IVFKM_TRY(cub::DeviceScan::ExclusiveSum(w.cub, cb, w.cnt, w.off, (int)(nh + 1), st));
  bivf_offset_kernel<<<grid_for(nh / kSpan + 1, threads), threads, 0, st>>>(nh, w.off, headers);
  IVFKM_CHECK_LAUNCH();
  bivf_scatter_kernel<<<kNumSM * 8, threads, 0, st>>>(major, nrows, ptr, cols, vals, k, dim,
                                                      nblk, headers, val32, val64);
  IVFKM_CHECK_LAUNCH();
  bivf_nc_kernel<<<grid_for(dim, threads / 32), threads, 0, st>>>(dim, nblk, headers,
                                                                  headers + 2 * nh + 1);
  IVFKM_CHECK_LAUNCH();
  return IVFKM_OK;
}
