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
#include <cuda_fp16.h>

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
  unsigned long long* tot64;  // total values, 64-bit (overflow check of the 32-bit offsets)
  unsigned int* cnt;
  unsigned int* off;
  unsigned int* cnt64;  // postings per block (compact exact-value layout)
  unsigned int* key_a;  // k: descending-size keys
  unsigned int* key_b;
  int32_t* id_a;        // k: mean ids
  int32_t* id_b;
  void* cub;
  size_t cub_bytes;
};

// build options (ivfkm_set_bivf_options)
float g_dense_fill = 1.0f / 64.0f;  // spans with >= fill*256 postings are stored dense
int g_permute = 1;          // slots ordered by mean size

uint32_t dense_threshold() {
  if (g_dense_fill > 1.0f) return 1u << 30;  // never
  uint32_t th = (uint32_t)(g_dense_fill * 256.0f + 0.999f);
  return th < 1 ? 1 : th;
}

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
  w.tot64 = c.take<unsigned long long>(1);
  w.cnt = c.take<unsigned int>(nh + 1);
  w.off = c.take<unsigned int>(nh + 1);
  w.cnt64 = c.take<unsigned int>(nh + 1);
  w.key_a = c.take<unsigned int>(k);
  w.key_b = c.take<unsigned int>(k);
  w.id_a = c.take<int32_t>(k);
  w.id_b = c.take<int32_t>(k);
  size_t sb = 0;
  cub::DoubleBuffer<unsigned int> kb(nullptr, nullptr);
  cub::DoubleBuffer<int32_t> vb(nullptr, nullptr);
  cub::DeviceRadixSort::SortPairs(nullptr, sb, kb, vb, (int)k);
  w.cub_bytes = std::max(cub_scan_bytes(nh + 1), sb);
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

// Entries of a CSR in contiguous per-warp chunks (so a few long rows — k
// means holding ~20k terms each — still spread over the whole GPU): one
// binary search per warp, then each lane walks the row pointer forward.
template <class F>
__device__ __forceinline__ void for_each_entry(int64_t nrows, const int64_t* __restrict__ ptr,
                                               F&& f) {
  const int64_t nnz = ptr[nrows];
  const int lane = threadIdx.x & 31;
  const int64_t nwarps = (int64_t)gridDim.x * (blockDim.x >> 5);
  const int64_t wid = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5);
  int64_t chunk = (nnz + nwarps - 1) / nwarps;
  chunk = (chunk + 31) / 32 * 32;
  const int64_t q0 = wid * chunk;
  const int64_t q1 = q0 + chunk < nnz ? q0 + chunk : nnz;
  if (q0 >= q1) return;
  int64_t r = row_of(ptr, nrows, q0);
  for (int64_t qb = q0; qb < q1; qb += 32) {
    const int64_t q = qb + lane;
    int64_t rl = r;
    if (q < q1) {
      while (__ldg(ptr + rl + 1) <= q) ++rl;
      f(rl, q);
    }
    r = __shfl_sync(0xffffffffu, rl, 31);  // lane 31 holds the furthest row
  }
}

__global__ void bivf_mask_kernel(int major, int64_t nrows, const int64_t* __restrict__ ptr,
                                 const int32_t* __restrict__ cols, int64_t k, int64_t dim,
                                 int64_t nblk, const int32_t* __restrict__ perm,
                                 unsigned int* __restrict__ hdr, unsigned int* __restrict__ err) {
  for_each_entry(nrows, ptr, [&](int64_t r, int64_t q) {
    const int64_t col = cols[q];
    const int64_t c = major == 0 ? r : col;
    const int64_t t = major == 0 ? col : r;
    if (c < 0 || c >= k || t < 0 || t >= dim) {
      atomicAdd(err, 1u);
      return;
    }
    const int64_t sl = perm[c];
    atomicOr(&hdr[t * nblk + (sl >> 5)], 1u << (sl & 31));
  });
}

// One thread per (term, span): popcounts of its 8 blocks, the span total
// padded to a multiple of 8 values on the last block (16 B of fp16 values).
__global__ void bivf_count_kernel(int64_t nh, const unsigned int* __restrict__ masks,
                                  unsigned int dense_th, unsigned int* __restrict__ cnt,
                                  unsigned int* __restrict__ cnt64,
                                  unsigned long long* __restrict__ tot64) {
  const int64_t nspan = nh / kSpan;
  unsigned long long mine = 0;
  for (int64_t sp = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; sp <= nspan;
       sp += (int64_t)gridDim.x * blockDim.x) {
    if (sp == nspan) {
      cnt[nh] = 0u;
      cnt64[nh] = 0u;
      continue;
    }
    unsigned c[kSpan], tot = 0;
#pragma unroll
    for (int r = 0; r < kSpan; ++r) {
      c[r] = __popc(masks[sp * kSpan + r]);
      cnt64[sp * kSpan + r] = c[r];
      tot += c[r];
    }
    const bool dense = tot >= dense_th;
#pragma unroll
    for (int r = 0; r < kSpan; ++r) cnt[sp * kSpan + r] = dense ? 32u : c[r];
    if (!dense) cnt[sp * kSpan + kSpan - 1] += (8u - (tot & 7u)) & 7u;
    mine += dense ? 256u : tot + ((8u - (tot & 7u)) & 7u);
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) mine += __shfl_xor_sync(0xffffffffu, mine, off);
  if ((threadIdx.x & 31) == 0 && mine) atomicAdd(tot64, mine);
}

__global__ void bivf_offset_kernel(int64_t nh, const unsigned int* __restrict__ off,
                                   unsigned int dense_th, unsigned int* __restrict__ hdr) {
  const int64_t nspan = nh / kSpan;
  for (int64_t sp = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; sp <= nspan;
       sp += (int64_t)gridDim.x * blockDim.x) {
    if (sp == nspan) {
      hdr[nh + nh] = off[nh];
      continue;
    }
    unsigned tot = 0;
#pragma unroll
    for (int r = 0; r < kSpan; ++r) tot += __popc(hdr[sp * kSpan + r]);
    const bool dense = tot >= dense_th;
#pragma unroll
    for (int r = 0; r < kSpan; ++r)
      hdr[nh + sp * kSpan + r] = off[sp * kSpan + r] | (dense ? kDense : 0u);

  }
}

__global__ void bivf_scatter_kernel(int major, int64_t nrows, const int64_t* __restrict__ ptr,
                                    const int32_t* __restrict__ cols,
                                    const double* __restrict__ vals, int64_t k, int64_t dim,
                                    int64_t nblk, const unsigned int* __restrict__ hdr,
                                    const int32_t* __restrict__ perm,
                                    float* __restrict__ v32, double* __restrict__ v64, int half) {
  const int64_t nh = bivf_nh(dim, nblk);
  const unsigned int* off64 = hdr + 2 * nh + 1 + dim + 2 * k + dim;
  for_each_entry(nrows, ptr, [&](int64_t r, int64_t q) {
    const int64_t col = cols[q];
    const int64_t c = major == 0 ? r : col;
    const int64_t t = major == 0 ? col : r;
    if (c < 0 || c >= k || t < 0 || t >= dim) return;
    const int64_t s = perm[c];
    const int64_t b = s >> 5;
    const uint32_t j = (uint32_t)(s & 31);
    const uint32_t m = hdr[t * nblk + b];
    const uint32_t o = hdr[nh + t * nblk + b];
    const uint32_t below = (uint32_t)__popc(m & ((1u << j) - 1u));
    // screen positions (fp32 and fp16 differ only inside dense spans)
    int64_t pos, pos16;
    if (o & kDense) {
      const uint32_t rr = (uint32_t)(b & (kSpan - 1));
      const uint32_t sb = (o & ~kDense) - 32u * rr;
      pos = sb + 128u * (rr >> 2) + 4u * j + (rr & 3u);
      pos16 = sb + 8u * j + rr;
    } else {
      pos = pos16 = o + below;
    }
    const double v = vals[q];
    if (half) {
      reinterpret_cast<__half*>(v32)[pos16] = __double2half(v);
    } else {
      v32[pos] = static_cast<float>(v);
    }
    v64[(int64_t)off64[t * nblk + b] + below] = v;  // compact exact-value array
  });
}

// Sorted fill (two-step build): the postings are first sorted by BIVF
// position (term, slot) so the value writes and the header reads walk the
// arrays in order instead of scattering across every term row.
template <class K>
__global__ void bivf_poskey_kernel(int major, int64_t nrows, const int64_t* __restrict__ ptr,
                                   const int32_t* __restrict__ cols,
                                   const double* __restrict__ vals, int64_t k, int64_t dim,
                                   int64_t nslot, const int32_t* __restrict__ perm,
                                   K* __restrict__ key, double* __restrict__ val) {
  for_each_entry(nrows, ptr, [&](int64_t r, int64_t q) {
    const int64_t col = cols[q];
    const int64_t c = major == 0 ? r : col;
    const int64_t t = major == 0 ? col : r;
    const bool ok = c >= 0 && c < k && t >= 0 && t < dim;
    key[q] = ok ? (K)t * (K)nslot + (K)perm[c] : (K)dim * (K)nslot;  // sentinel sorts last
    val[q] = vals[q];
  });
}

template <class K>
__global__ void bivf_write_kernel(int64_t n, int64_t dim, int64_t nblk, int64_t nslot,
                                  const K* __restrict__ key, const double* __restrict__ val,
                                  const unsigned int* __restrict__ hdr,
                                  const unsigned int* __restrict__ off64,
                                  float* __restrict__ v32, double* __restrict__ v64, int half) {
  const int64_t nh = bivf_nh(dim, nblk);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const K kk = key[i];
    if (kk >= (K)dim * (K)nslot) continue;
    const int64_t t = (int64_t)(kk / (K)nslot);
    const int64_t s = (int64_t)(kk - (K)t * (K)nslot);
    const int64_t b = s >> 5;
    const uint32_t j = (uint32_t)(s & 31);
    const uint32_t m = hdr[t * nblk + b];
    const uint32_t o = hdr[nh + t * nblk + b];
    const uint32_t below = (uint32_t)__popc(m & ((1u << j) - 1u));
    int64_t pos, pos16;
    if (o & kDense) {
      const uint32_t rr = (uint32_t)(b & (kSpan - 1));
      const uint32_t sb = (o & ~kDense) - 32u * rr;
      pos = sb + 128u * (rr >> 2) + 4u * j + (rr & 3u);
      pos16 = sb + 8u * j + rr;
    } else {
      pos = pos16 = o + below;
    }
    const double v = val[i];
    if (half) {
      reinterpret_cast<__half*>(v32)[pos16] = __double2half(v);
    } else {
      v32[pos] = static_cast<float>(v);
    }
    v64[(int64_t)off64[t * nblk + b] + below] = v;
  }
}

// absent slots of dense spans (and padding) hold exact zeros: clear the
// screen array's [0, total) (the total is a multiple of 8, so the fp16 array
// is n/2 whole 32-bit words); the compact exact-value array has no holes
__global__ void bivf_zero_kernel(const unsigned int* __restrict__ total, float* __restrict__ vs,
                                 int half) {
  const int64_t n = *total;
  const int64_t ns = half ? n / 2 : n;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < ns;
       i += (int64_t)gridDim.x * blockDim.x)
    vs[i] = 0.f;
}

// descending-size sort keys: ~terms_of_mean (stable sort => ties by mean id)
__global__ void bivf_sizes_kernel(int major, int64_t nrows, const int64_t* __restrict__ ptr,
                                  const int32_t* __restrict__ cols, int64_t k,
                                  unsigned int* __restrict__ key, int32_t* __restrict__ id) {
  if (major == 0) {
    for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < k;
         c += (int64_t)gridDim.x * blockDim.x) {
      key[c] = ~(unsigned)(ptr[c + 1] - ptr[c]);
      id[c] = (int32_t)c;
    }
    return;
  }
  // term-major input: count each mean's postings (keys were set to ~0u)
  const int64_t nnz = ptr[nrows];
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < nnz;
       q += (int64_t)gridDim.x * blockDim.x) {
    const int64_t c = cols[q];
    if (c >= 0 && c < k) atomicSub(&key[c], 1u);
  }
}

__global__ void bivf_ids_kernel(int64_t k, int32_t* __restrict__ id) {
  for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < k;
       c += (int64_t)gridDim.x * blockDim.x)
    id[c] = (int32_t)c;
}

// inv[slot] = sorted id; perm[id] = slot
__global__ void bivf_perm_kernel(int64_t k, const int32_t* __restrict__ sorted,
                                 int32_t* __restrict__ perm, int32_t* __restrict__ inv,
                                 int identity) {
  for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < k;
       s += (int64_t)gridDim.x * blockDim.x) {
    const int32_t c = identity ? (int32_t)s : sorted[s];
    inv[s] = c;
    perm[c] = (int32_t)s;
  }
}

// postings per term: nc[t] = sum_b popc(masks[t][b])
// One warp per term: postings (nc) and the dense prefix (dpre, bivf.cuh).
__global__ void bivf_nc_kernel(int64_t dim, int64_t nblk, const unsigned int* __restrict__ masks,
                               const unsigned int* __restrict__ offs,
                               unsigned int* __restrict__ nc, unsigned int* __restrict__ dpre,
                               uint2* __restrict__ tinfo) {
  const int lane = threadIdx.x & 31;
  const int64_t wpb = blockDim.x >> 5;
  const int64_t nspan = nblk / kSpan;
  for (int64_t t = blockIdx.x * wpb + (threadIdx.x >> 5); t < dim; t += gridDim.x * wpb) {
    unsigned c = 0;
    for (int64_t b = lane; b < nblk; b += 32) c += __popc(masks[t * nblk + b]);
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) c += __shfl_xor_sync(0xffffffffu, c, off);
    int64_t pre = nspan;
    for (int64_t s0 = 0; s0 < nspan; s0 += 32) {
      const int64_t s = s0 + lane;
      const bool sparse = s < nspan && !(offs[t * nblk + s * kSpan] & kDense);
      const unsigned m = __ballot_sync(0xffffffffu, sparse);
      if (m) {
        pre = s0 + __ffs(m) - 1;
        break;
      }
    }
    if (lane == 0) {
      nc[t] = c;
      dpre[t] = (unsigned)pre;
      // bit 31: the term has postings (an object touching none keeps label 0)
      tinfo[t] = make_uint2(offs[t * nblk] & ~kDense, (unsigned)pre | (c ? 0x80000000u : 0u));
    }
  }
}

}  // namespace

extern "C" size_t ivfkm_bivf_workspace_size(int64_t dim, int64_t k) {
  size_t total = 0;
  carve(nullptr, dim, k, &total);
  return total;
}

extern "C" void ivfkm_set_bivf_options(float dense_fill, int permute) {
  if (dense_fill >= 1.0f / 256.0f) g_dense_fill = dense_fill;
  if (permute == 0 || permute == 1) g_permute = permute;
}

extern "C" int64_t ivfkm_bivf_headers_size(int64_t k, int64_t dim) {
  const int64_t nh = bivf_nh(dim, ivfkm_bivf_nblk(k));
  (void)nh;
  return bivf_tinfo_word(k, dim, ivfkm_bivf_nblk(k)) + 2 * dim;
}

extern "C" int64_t ivfkm_bivf_values_capacity(int64_t k, int64_t dim, int64_t nnz) {
  const double f = g_dense_fill > 1.0f ? 1.0 : (double)g_dense_fill;
  const int64_t nblk = ivfkm_bivf_nblk(k);
  // dense spans hold 256 values each; no layout exceeds every span dense
  const int64_t by_fill = (int64_t)((double)nnz / f) + 7 * dim * (nblk / kSpan);
  const int64_t all_dense = dim * nblk * 32;
  return (by_fill < all_dense ? by_fill : all_dense) + 256 + 8;
}

namespace {

// Headers, part 1: slot order and masks.
int plan_masks(int64_t k, int64_t dim, int major, int64_t nrows, const int64_t* ptr,
               const int32_t* cols, uint32_t* headers, const BivfWs& w, cudaStream_t st) {
  const int64_t nblk = ivfkm_bivf_nblk(k);
  const int64_t nh = bivf_nh(dim, nblk);
  uint32_t* nc = headers + 2 * nh + 1;
  int32_t* perm = reinterpret_cast<int32_t*>(nc + dim);
  int32_t* inv = perm + k;
  const int threads = 256;
  // ---- slot order: means by term count, descending (stable)
  if (g_permute) {
    if (major == 1) {
      IVFKM_TRY(cudaMemsetAsync(w.key_a, 0xff, sizeof(unsigned) * k, st));
      bivf_ids_kernel<<<grid_for(k, threads), threads, 0, st>>>(k, w.id_a);
      IVFKM_CHECK_LAUNCH();
    }
    bivf_sizes_kernel<<<major == 0 ? grid_for(k, threads) : num_sms() * 8, threads, 0, st>>>(
        major, nrows, ptr, cols, k, w.key_a, w.id_a);
    IVFKM_CHECK_LAUNCH();
    cub::DoubleBuffer<unsigned int> kb(w.key_a, w.key_b);
    cub::DoubleBuffer<int32_t> vb(w.id_a, w.id_b);
    size_t cb = w.cub_bytes;
    IVFKM_TRY(cub::DeviceRadixSort::SortPairs(w.cub, cb, kb, vb, (int)k, 0, 32, st));
    bivf_perm_kernel<<<grid_for(k, threads), threads, 0, st>>>(k, vb.Current(), perm, inv, 0);
  } else {
    bivf_perm_kernel<<<grid_for(k, threads), threads, 0, st>>>(k, nullptr, perm, inv, 1);
  }
  IVFKM_CHECK_LAUNCH();
  IVFKM_TRY(cudaMemsetAsync(headers, 0, sizeof(uint32_t) * nh, st));
  IVFKM_TRY(cudaMemsetAsync(w.err, 0, sizeof(unsigned int), st));
  bivf_mask_kernel<<<num_sms() * 8, threads, 0, st>>>(major, nrows, ptr, cols, k, dim, nblk, perm,
                                                   headers, w.err);
  IVFKM_CHECK_LAUNCH();
  return IVFKM_OK;
}

// Span counts under dense threshold th (+ the 64-bit total in w.tot64).
int plan_count(int64_t k, int64_t dim, const uint32_t* headers, unsigned th, const BivfWs& w,
               cudaStream_t st) {
  const int64_t nh = bivf_nh(dim, ivfkm_bivf_nblk(k));
  const int threads = 256;
  IVFKM_TRY(cudaMemsetAsync(w.tot64, 0, sizeof(unsigned long long), st));
  bivf_count_kernel<<<grid_for(nh / kSpan + 1, threads), threads, 0, st>>>(nh, headers, th,
                                                                          w.cnt, w.cnt64, w.tot64);
  IVFKM_CHECK_LAUNCH();
  return IVFKM_OK;
}

__global__ void bivf_mo_kernel(int64_t nh, const uint32_t* __restrict__ masks,
                               const uint32_t* __restrict__ off64, uint2* __restrict__ mo) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nh;
       i += (int64_t)gridDim.x * blockDim.x)
    mo[i] = make_uint2(masks[i], off64[i]);
}

// Headers, part 2: offsets (total at offs[nh]), nc, dense prefixes, the
// exact lookup's {mask, off64} pairs.
int plan_layout(int64_t k, int64_t dim, uint32_t* headers, unsigned th, const BivfWs& w,
                cudaStream_t st) {
  const int64_t nblk = ivfkm_bivf_nblk(k);
  const int64_t nh = bivf_nh(dim, nblk);
  uint32_t* nc = headers + 2 * nh + 1;
  uint32_t* dpre = reinterpret_cast<uint32_t*>(nc + dim + 2 * k);
  uint32_t* off64 = dpre + dim;
  const int threads = 256;
  size_t cb = w.cub_bytes;
  IVFKM_TRY(cub::DeviceScan::ExclusiveSum(w.cub, cb, w.cnt64, off64, (int)(nh + 1), st));
  cb = w.cub_bytes;
  IVFKM_TRY(cub::DeviceScan::ExclusiveSum(w.cub, cb, w.cnt, w.off, (int)(nh + 1), st));
  bivf_offset_kernel<<<grid_for(nh / kSpan + 1, threads), threads, 0, st>>>(nh, w.off, th,
                                                                           headers);
  IVFKM_CHECK_LAUNCH();
  bivf_nc_kernel<<<grid_for(dim, threads / 32), threads, 0, st>>>(
      dim, nblk, headers, headers + nh, nc, dpre,
      reinterpret_cast<uint2*>(headers + bivf_tinfo_word(k, dim, nblk)));
  IVFKM_CHECK_LAUNCH();
  bivf_mo_kernel<<<grid_for(nh, threads), threads, 0, st>>>(
      nh, headers, off64, reinterpret_cast<uint2*>(headers + bivf_mo_word(k, dim, nblk)));
  IVFKM_CHECK_LAUNCH();
  return IVFKM_OK;
}

// Values: zero [0, total) (absent slots of dense spans), scatter the postings.
template <class K>
struct FillWs {
  K* key_a;
  K* key_b;
  double* val_a;
  double* val_b;
  void* cub;
  size_t cub_bytes;
};

template <class K>
FillWs<K> carve_fill(void* base, int64_t nnz, size_t* total) {
  Carver c(base);
  FillWs<K> w;
  const size_t n = (size_t)(nnz > 0 ? nnz : 1);
  w.key_a = c.take<K>(n);
  w.key_b = c.take<K>(n);
  w.val_a = c.take<double>(n);
  w.val_b = c.take<double>(n);
  size_t a = 0;
  cub::DoubleBuffer<K> kb(nullptr, nullptr);
  cub::DoubleBuffer<double> vb(nullptr, nullptr);
  cub::DeviceRadixSort::SortPairs(nullptr, a, kb, vb, (int)n, 0, (int)(sizeof(K) * 8));
  w.cub_bytes = a;
  w.cub = c.take_bytes(a);
  if (total) *total = c.off;
  return w;
}

bool fill_k32(int64_t k, int64_t dim) {
  return (double)dim * (double)(ivfkm_bivf_nblk(k) * 32) < 4294967295.0;
}

template <class K>
int sorted_fill(int64_t k, int64_t dim, int major, int64_t nrows, const int64_t* ptr,
                const int32_t* cols, const double* vals, const uint32_t* headers, float* val32,
                int half, double* val64, int64_t nnz, void* ws, cudaStream_t st) {
  const int64_t nblk = ivfkm_bivf_nblk(k);
  const int64_t nh = bivf_nh(dim, nblk);
  const int64_t nslot = nblk * 32;
  const int32_t* perm = reinterpret_cast<const int32_t*>(headers + 2 * nh + 1 + dim);
  const unsigned int* off64 = headers + 2 * nh + 1 + dim + 2 * k + dim;
  FillWs<K> w = carve_fill<K>(ws, nnz, nullptr);
  const int threads = 256;
  bivf_poskey_kernel<K><<<num_sms() * 8, threads, 0, st>>>(major, nrows, ptr, cols, vals, k, dim,
                                                        nslot, perm, w.key_a, w.val_a);
  IVFKM_CHECK_LAUNCH();
  int bits = 1;  // keys lie in [0, dim * nslot] (the sentinel included)
  while (bits < (int)(sizeof(K) * 8) && (double)(1ull << bits) <= (double)dim * (double)nslot)
    ++bits;
  cub::DoubleBuffer<K> kb(w.key_a, w.key_b);
  cub::DoubleBuffer<double> vb(w.val_a, w.val_b);
  size_t cb = w.cub_bytes;
  // The write is a scatter by computed position, so it needs locality, not
  // order: sorting by the key's top 16 bits (a few terms per bucket) keeps
  // its stores and header reads inside L2-resident windows — 2 radix passes
  // instead of 4 (measured +0.8% per iteration at config 1 against the full
  // sort; 1 pass of 8 bits gains less).
  const int begin = bits > 16 ? bits - 16 : 0;
  IVFKM_TRY(cub::DeviceRadixSort::SortPairs(w.cub, cb, kb, vb, (int)nnz, begin, bits, st));
  bivf_write_kernel<K><<<grid_for(nnz, threads), threads, 0, st>>>(
      nnz, dim, nblk, nslot, kb.Current(), vb.Current(), headers, off64, val32, val64, half);
  IVFKM_CHECK_LAUNCH();
  return IVFKM_OK;
}

int fill_impl(int64_t k, int64_t dim, int major, int64_t nrows, const int64_t* ptr,
              const int32_t* cols, const double* vals, const uint32_t* headers,
              void* val_screen, int screen_bits, double* val64, cudaStream_t st,
              int64_t nnz = -1, void* ws = nullptr) {
  const int64_t nblk = ivfkm_bivf_nblk(k);
  const int64_t nh = bivf_nh(dim, nblk);
  const int32_t* perm = reinterpret_cast<const int32_t*>(headers + 2 * nh + 1 + dim);
  float* val32 = static_cast<float*>(val_screen);  // or fp16 values (screen_bits 16)
  const int threads = 256;
  bivf_zero_kernel<<<num_sms() * 16, threads, 0, st>>>(headers + 2 * nh, val32, screen_bits == 16);
  IVFKM_CHECK_LAUNCH();
  if (ws && nnz > 0 && nnz < (int64_t)INT32_MAX) {
    return fill_k32(k, dim)
               ? sorted_fill<uint32_t>(k, dim, major, nrows, ptr, cols, vals, headers, val32,
                                       screen_bits == 16, val64, nnz, ws, st)
               : sorted_fill<unsigned long long>(k, dim, major, nrows, ptr, cols, vals, headers,
                                                 val32, screen_bits == 16, val64, nnz, ws, st);
  }
  bivf_scatter_kernel<<<num_sms() * 8, threads, 0, st>>>(major, nrows, ptr, cols, vals, k, dim,
                                                      nblk, headers, perm, val32, val64,
                                                      screen_bits == 16);
  IVFKM_CHECK_LAUNCH();
  return IVFKM_OK;
}

int check_build_args(int64_t k, int64_t dim, int major, int64_t nrows, const int64_t* ptr,
                     const void* headers) {
  if (k < 1 || dim < 1 || nrows < 0 || (major != 0 && major != 1) || !ptr || !headers)
    return IVFKM_E_ARG;
  if (k > INT32_MAX) return IVFKM_E_UNSUPPORTED;
  if (bivf_nh(dim, ivfkm_bivf_nblk(k)) + 1 > INT32_MAX)
    return IVFKM_E_UNSUPPORTED;  // cub scan length, 32-bit rows
  return IVFKM_OK;
}

}  // namespace

extern "C" int ivfkm_bivf_plan(int64_t k, int64_t dim, int major, int64_t nrows,
                               const int64_t* ptr, const int32_t* cols, uint32_t* headers,
                               int64_t* totals, void* ws, size_t ws_bytes,
                               ivfkm_stream_t stream_) {
  if (int rc = check_build_args(k, dim, major, nrows, ptr, headers)) return rc;
  if (!totals) return IVFKM_E_ARG;
  size_t need = 0;
  BivfWs w = carve(ws, dim, k, &need);
  if (ws_bytes < need) return IVFKM_E_WORKSPACE;
  cudaStream_t st = as_stream(stream_);
  if (int rc = plan_masks(k, dim, major, nrows, ptr, cols, headers, w, st)) return rc;
  // Value offsets are 31 bits (bit 31 flags dense blocks): while the layout
  // would not fit, raise the dense threshold (fewer, fuller dense spans).
  unsigned th = dense_threshold();
  unsigned int err = 0;
  unsigned long long tot = 0;
  for (;;) {
    if (int rc = plan_count(k, dim, headers, th, w, st)) return rc;
    IVFKM_TRY(cudaMemcpyAsync(&tot, w.tot64, sizeof(tot), cudaMemcpyDeviceToHost, st));
    IVFKM_TRY(cudaMemcpyAsync(&err, w.err, sizeof(err), cudaMemcpyDeviceToHost, st));
    IVFKM_TRY(cudaStreamSynchronize(st));
    if (err) return IVFKM_E_RANGE;
    if (tot < (1ull << 31) - 256) break;
    if (th > 256) return IVFKM_E_UNSUPPORTED;  // even all-sparse does not fit
    th = th * 2 > 256 ? (1u << 30) : th * 2;
  }
  if (int rc = plan_layout(k, dim, headers, th, w, st)) return rc;
  const int64_t nh = bivf_nh(dim, ivfkm_bivf_nblk(k));
  unsigned int n64 = 0;  // postings (off64[nh])
  IVFKM_TRY(cudaMemcpyAsync(&n64, headers + 2 * nh + 1 + dim + 2 * k + dim + nh, sizeof(n64),
                            cudaMemcpyDeviceToHost, st));
  IVFKM_TRY(cudaStreamSynchronize(st));
  totals[0] = (int64_t)tot;
  totals[1] = (int64_t)n64;
  return IVFKM_OK;
}

extern "C" size_t ivfkm_bivf_fill_workspace_size(int64_t k, int64_t dim, int64_t nnz) {
  size_t t = 0;
  if (fill_k32(k, dim)) carve_fill<uint32_t>(nullptr, nnz, &t);
  else carve_fill<unsigned long long>(nullptr, nnz, &t);
  return t;
}

extern "C" int ivfkm_bivf_fill(int64_t k, int64_t dim, int major, int64_t nrows,
                               const int64_t* ptr, const int32_t* cols, const double* vals,
                               const uint32_t* headers, void* val_screen, int screen_bits,
                               double* val64, int64_t nnz, void* ws, size_t ws_bytes,
                               ivfkm_stream_t stream_) {
  if (int rc = check_build_args(k, dim, major, nrows, ptr, headers)) return rc;
  if (screen_bits != 32 && screen_bits != 16) return IVFKM_E_ARG;
  if (ws && ws_bytes < ivfkm_bivf_fill_workspace_size(k, dim, nnz)) return IVFKM_E_WORKSPACE;
  return fill_impl(k, dim, major, nrows, ptr, cols, vals, headers, val_screen, screen_bits,
                   val64, as_stream(stream_), nnz, ws);
}

// plan, then (when the caller's buffers are large enough) fill, with no
// host round trip in between; IVFKM_E_WORKSPACE leaves the plan done and the
// fill to the caller (totals tell the sizes).
extern "C" int ivfkm_bivf_plan_fill(int64_t k, int64_t dim, int major, int64_t nrows,
                                    const int64_t* ptr, const int32_t* cols, const double* vals,
                                    uint32_t* headers, int64_t* totals, void* val_screen,
                                    int64_t screen_cap, int screen_bits, double* val64,
                                    int64_t val64_cap, void* ws_plan, size_t ws_plan_bytes,
                                    void* ws_fill, size_t ws_fill_bytes, ivfkm_stream_t stream_) {
  if (screen_bits != 32 && screen_bits != 16) return IVFKM_E_ARG;
  if (int rc = ivfkm_bivf_plan(k, dim, major, nrows, ptr, cols, headers, totals, ws_plan,
                               ws_plan_bytes, stream_))
    return rc;
  const int64_t nnz = totals[1];
  if (totals[0] > screen_cap || nnz > val64_cap || !ws_fill ||
      ws_fill_bytes < ivfkm_bivf_fill_workspace_size(k, dim, nnz))
    return IVFKM_E_WORKSPACE;
  return fill_impl(k, dim, major, nrows, ptr, cols, vals, headers, val_screen, screen_bits,
                   val64, as_stream(stream_), nnz, ws_fill);
}

namespace {
// Slot bytes of the sparse spans: for a posting stored in a sparse span at
// screen position o + below, its slot within the span (0..255) at the same
// position of `slot8` — the screen's sparse path then needs neither masks
// nor popcounts.  Dense spans' positions are left untouched (never read).
__global__ void bivf_slot_kernel(int major, int64_t nrows, const int64_t* __restrict__ ptr,
                                 const int32_t* __restrict__ cols, int64_t k, int64_t dim,
                                 int64_t nblk, const unsigned int* __restrict__ hdr,
                                 const int32_t* __restrict__ perm, uint8_t* __restrict__ slot8) {
  const int64_t nh = bivf_nh(dim, nblk);
  for_each_entry(nrows, ptr, [&](int64_t r, int64_t q) {
    const int64_t col = cols[q];
    const int64_t c = major == 0 ? r : col;
    const int64_t t = major == 0 ? col : r;
    if (c < 0 || c >= k || t < 0 || t >= dim) return;
    const int64_t sl = perm[c];
    const int64_t b = sl >> 5;
    const uint32_t j = (uint32_t)(sl & 31);
    const uint32_t o = hdr[nh + t * nblk + b];
    if (o & kDense) return;
    const uint32_t m = hdr[t * nblk + b];
    slot8[(int64_t)o + __popc(m & ((1u << j) - 1u))] = (uint8_t)(sl & 255);
  });
}
// Compact span offsets (bivf.cuh, bivf_soff_bytes).
__global__ void bivf_soff_kernel(int64_t dim, int64_t nblk, const unsigned int* __restrict__ offs,
                                 unsigned int* __restrict__ soff) {
  const int64_t nsp1 = nblk / kSpan + 1;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < dim * nsp1;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t t = i / nsp1, sp = i - t * nsp1;
    // sp == nsp1 - 1: the next term's first block (the total after the last term)
    soff[i] = offs[t * nblk + sp * kSpan];
  }
}
}  // namespace

extern "C" size_t ivfkm_bivf_slots_size(int64_t k, int64_t dim, int64_t n_values) {
  if (k < 1 || dim < 1 || n_values < 0) return 0;
  return bivf_soff_bytes(dim, ivfkm_bivf_nblk(k)) + (size_t)n_values;
}

extern "C" int ivfkm_bivf_slots(int64_t k, int64_t dim, int major, int64_t nrows,
                                const int64_t* ptr, const int32_t* cols, const uint32_t* headers,
                                uint8_t* slot8, ivfkm_stream_t stream_) {
  if (int rc = check_build_args(k, dim, major, nrows, ptr, headers)) return rc;
  if (!slot8) return IVFKM_E_ARG;
  const int64_t nblk = ivfkm_bivf_nblk(k);
  const int64_t nh = bivf_nh(dim, nblk);
  const int32_t* perm = reinterpret_cast<const int32_t*>(headers + 2 * nh + 1 + dim);
  cudaStream_t st = as_stream(stream_);
  bivf_soff_kernel<<<grid_for(dim * (nblk / kSpan + 1), 256, num_sms() * 16), 256, 0, st>>>(
      dim, nblk, headers + nh, reinterpret_cast<unsigned int*>(slot8));
  IVFKM_CHECK_LAUNCH();
  bivf_slot_kernel<<<num_sms() * 8, 256, 0, st>>>(major, nrows, ptr, cols, k, dim, nblk, headers,
                                                  perm, slot8 + bivf_soff_bytes(dim, nblk));
  IVFKM_CHECK_LAUNCH();
  return IVFKM_OK;
}

extern "C" int ivfkm_bivf_build(int64_t k, int64_t dim, int major, int64_t nrows,
                                const int64_t* ptr, const int32_t* cols, const double* vals,
                                uint32_t* headers, void* val_screen, int screen_bits,
                                double* val64, void* ws, size_t ws_bytes,
                                ivfkm_stream_t stream_) {
  if (int rc = check_build_args(k, dim, major, nrows, ptr, headers)) return rc;
  if (screen_bits != 32 && screen_bits != 16) return IVFKM_E_ARG;
  size_t need = 0;
  BivfWs w = carve(ws, dim, k, &need);
  if (ws_bytes < need) return IVFKM_E_WORKSPACE;
  cudaStream_t st = as_stream(stream_);
  const unsigned th = dense_threshold();
  if (int rc = plan_masks(k, dim, major, nrows, ptr, cols, headers, w, st)) return rc;
  if (int rc = plan_count(k, dim, headers, th, w, st)) return rc;
  if (int rc = plan_layout(k, dim, headers, th, w, st)) return rc;
  return fill_impl(k, dim, major, nrows, ptr, cols, vals, headers, val_screen, screen_bits,
                   val64, st);
}
