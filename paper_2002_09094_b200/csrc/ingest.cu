// Device half of ingestion: triple sort + duplicate check, tf-idf weighting
// and L2 normalisation, bit-identical to the reference (io.py:118-174):
//
//   triples.sort()                                   -> stable radix sort by (doc, term)
//   duplicate (doc, term) at the later line          -> min line of any repeated key
//   df = bincount(terms)                             -> per-term histogram
//   idf = log(n_docs / df)  (df > 0)                 -> host numpy (D values), uploaded
//   weights = counts * idf[terms - 1]; drop zeros    -> one fp64 multiply per entry
//   sq = bincount(docs - 1, weights=weights*weights) -> per document, sequential in
//                                                       entry order (bincount's loop)
//   values = weights / sqrt(sq)[docs - 1]; drop documents left empty
//
// The entries arrive sorted by (doc, term), so every document is a
// contiguous run; one thread per document adds its squares in order.
#include <cub/cub.cuh>

#include <cstdint>

#include "common.cuh"

using namespace ivfkm;

namespace {

struct BowWs {
  unsigned long long* key_a;
  unsigned long long* key_b;
  int64_t* idx_a;
  int64_t* idx_b;
  int32_t* tmp32;
  int64_t* tmp64;
  void* cub;
  size_t cub_bytes;
};

BowWs carve_bow(void* base, int64_t n, size_t* total) {
  Carver c(base);
  BowWs w;
  const size_t m = (size_t)(n > 0 ? n : 1);
  w.key_a = c.take<unsigned long long>(m);
  w.key_b = c.take<unsigned long long>(m);
  w.idx_a = c.take<int64_t>(m);
  w.idx_b = c.take<int64_t>(m);
  w.tmp32 = c.take<int32_t>(m);
  w.tmp64 = c.take<int64_t>(m);
  size_t a = 0;
  cub::DoubleBuffer<unsigned long long> kb(nullptr, nullptr);
  cub::DoubleBuffer<int64_t> vb(nullptr, nullptr);
  cub::DeviceRadixSort::SortPairs(nullptr, a, kb, vb, (int)m, 0, 64);
  w.cub_bytes = a;
  w.cub = c.take_bytes(a);
  if (total) *total = c.off;
  return w;
}

int key_bits64(int64_t n_docs, int64_t dim) {
  const double top = (double)n_docs * (double)dim;
  int b = 1;
  while (b < 64 && (double)(1ull << b) < top) ++b;
  return b;
}

__global__ void bow_keys_kernel(int64_t n, int64_t dim, const int32_t* __restrict__ docs,
                                const int32_t* __restrict__ terms,
                                unsigned long long* __restrict__ key, int64_t* __restrict__ idx) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    key[i] = (unsigned long long)(docs[i] - 1) * (unsigned long long)dim +
             (unsigned long long)(terms[i] - 1);
    idx[i] = i;
  }
}

template <class T>
__global__ void gather_kernel(int64_t n, const int64_t* __restrict__ idx, const T* __restrict__ src,
                              T* __restrict__ dst) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    dst[i] = src[idx[i]];
}

// any repeated key: its line (lines ascend within a key: the sort is stable
// over line order), minimised -> the line the reference reports
__global__ void dup_kernel(int64_t n, const unsigned long long* __restrict__ key,
                           const int64_t* __restrict__ lines, unsigned long long* __restrict__ out) {
  for (int64_t i = 1 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    if (key[i] == key[i - 1]) atomicMin(out, (unsigned long long)lines[i]);
}

__global__ void df_kernel(int64_t n, const int32_t* __restrict__ terms,
                          unsigned long long* __restrict__ df) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    atomicAdd(&df[terms[i] - 1], 1ull);
}

// doc_ptr[d] = first entry of document d+1 (entries sorted by doc)
__global__ void doc_ptr_kernel(int64_t n, int64_t n_docs, const int32_t* __restrict__ docs,
                               int64_t* __restrict__ ptr) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i <= n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t lo = i == 0 ? 0 : docs[i - 1];        // docs are 1-based
    const int64_t hi = i == n ? n_docs : docs[i] - 1;
    for (int64_t d = lo; d <= hi && d <= n_docs; ++d) ptr[d] = i;
  }
}

// One thread per document: weights, kept count, sequential sum of squares.
__global__ void doc_weights_kernel(int64_t n_docs, const int64_t* __restrict__ ptr,
                                   const int32_t* __restrict__ terms,
                                   const int32_t* __restrict__ counts,
                                   const double* __restrict__ idf, double* __restrict__ w,
                                   int64_t* __restrict__ kept, double* __restrict__ norm) {
  for (int64_t d = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; d < n_docs;
       d += (int64_t)gridDim.x * blockDim.x) {
    double sq = 0.0;
    int64_t k = 0;
    for (int64_t e = ptr[d]; e < ptr[d + 1]; ++e) {
      const double x = __dmul_rn((double)counts[e], idf[terms[e] - 1]);
      w[e] = x;
      if (x != 0.0) {
        sq = __dadd_rn(sq, __dmul_rn(x, x));
        ++k;
      }
    }
    kept[d] = k;
    norm[d] = __dsqrt_rn(sq);
  }
}

__global__ void survivor_kernel(int64_t n_docs, const int64_t* __restrict__ kept,
                                int64_t* __restrict__ alive) {
  for (int64_t d = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; d < n_docs;
       d += (int64_t)gridDim.x * blockDim.x)
    alive[d] = kept[d] > 0 ? 1 : 0;
}

// out_ptr[rank] = out_start (kept-entry offset) of each surviving document
__global__ void emit_kernel(int64_t n_docs, const int64_t* __restrict__ ptr,
                            const int32_t* __restrict__ terms, const double* __restrict__ w,
                            const double* __restrict__ norm, const int64_t* __restrict__ kept_off,
                            const int64_t* __restrict__ rank, const int64_t* __restrict__ kept,
                            int64_t* __restrict__ out_ptr, int32_t* __restrict__ out_terms,
                            double* __restrict__ out_vals, int32_t* __restrict__ dropped,
                            int64_t n_alive) {
  for (int64_t d = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; d < n_docs;
       d += (int64_t)gridDim.x * blockDim.x) {
    if (kept[d] == 0) {
      dropped[d - rank[d]] = (int32_t)(d + 1);  // 1-based, ascending
      continue;
    }
    const int64_t r = rank[d];
    int64_t o = kept_off[d];
    out_ptr[r] = o;
    if (r == n_alive - 1) out_ptr[n_alive] = o + kept[d];
    for (int64_t e = ptr[d]; e < ptr[d + 1]; ++e) {
      const double x = w[e];
      if (x == 0.0) continue;
      out_terms[o] = terms[e];
      out_vals[o] = __ddiv_rn(x, norm[d]);
      ++o;
    }
  }
}

}  // namespace

extern "C" size_t ivfkm_bow_workspace_size(int64_t n) {
  size_t t = 0;
  carve_bow(nullptr, n, &t);
  return t;
}

// Sort parsed triples by (doc, term) in place (stable over line order) and
// write the smallest line holding a repeated (doc, term) pair to *dup_line
// ([dev] uint64, UINT64_MAX when none).
extern "C" int ivfkm_bow_sort(int64_t n, int64_t n_docs, int64_t dim, int32_t* docs,
                              int32_t* terms, int32_t* counts, int64_t* lines,
                              unsigned long long* dup_line, void* ws, size_t ws_bytes,
                              ivfkm_stream_t stream_) {
  if (n < 0 || n_docs < 0 || dim < 0 || !dup_line) return IVFKM_E_ARG;
  if (n >= (int64_t)INT32_MAX) return IVFKM_E_UNSUPPORTED;
  size_t need = 0;
  BowWs w = carve_bow(ws, n, &need);
  if (ws_bytes < need) return IVFKM_E_WORKSPACE;
  cudaStream_t st = as_stream(stream_);
  IVFKM_TRY(cudaMemsetAsync(dup_line, 0xff, sizeof(unsigned long long), st));
  if (n == 0) return IVFKM_OK;
  const int T = 256;
  bow_keys_kernel<<<grid_for(n, T), T, 0, st>>>(n, dim, docs, terms, w.key_a, w.idx_a);
  IVFKM_CHECK_LAUNCH();
  cub::DoubleBuffer<unsigned long long> kb(w.key_a, w.key_b);
  cub::DoubleBuffer<int64_t> vb(w.idx_a, w.idx_b);
  size_t cb = w.cub_bytes;
  IVFKM_TRY(cub::DeviceRadixSort::SortPairs(w.cub, cb, kb, vb, (int)n, 0,
                                            key_bits64(n_docs, dim), st));
  const int64_t* idx = vb.Current();
  gather_kernel<int32_t><<<grid_for(n, T), T, 0, st>>>(n, idx, docs, w.tmp32);
  IVFKM_CHECK_LAUNCH();
  IVFKM_TRY(cudaMemcpyAsync(docs, w.tmp32, sizeof(int32_t) * n, cudaMemcpyDeviceToDevice, st));
  gather_kernel<int32_t><<<grid_for(n, T), T, 0, st>>>(n, idx, terms, w.tmp32);
  IVFKM_CHECK_LAUNCH();
  IVFKM_TRY(cudaMemcpyAsync(terms, w.tmp32, sizeof(int32_t) * n, cudaMemcpyDeviceToDevice, st));
  gather_kernel<int32_t><<<grid_for(n, T), T, 0, st>>>(n, idx, counts, w.tmp32);
  IVFKM_CHECK_LAUNCH();
  IVFKM_TRY(cudaMemcpyAsync(counts, w.tmp32, sizeof(int32_t) * n, cudaMemcpyDeviceToDevice, st));
  gather_kernel<int64_t><<<grid_for(n, T), T, 0, st>>>(n, idx, lines, w.tmp64);
  IVFKM_CHECK_LAUNCH();
  IVFKM_TRY(cudaMemcpyAsync(lines, w.tmp64, sizeof(int64_t) * n, cudaMemcpyDeviceToDevice, st));
  dup_kernel<<<grid_for(n, T), T, 0, st>>>(n, kb.Current(), lines, dup_line);
  IVFKM_CHECK_LAUNCH();
  return IVFKM_OK;
}

// Document frequencies of sorted, duplicate-free triples: df[dim] (uint64).
extern "C" int ivfkm_bow_df(int64_t n, int64_t dim, const int32_t* terms,
                            unsigned long long* df, ivfkm_stream_t stream_) {
  if (n < 0 || dim < 0 || (dim > 0 && !df)) return IVFKM_E_ARG;
  cudaStream_t st = as_stream(stream_);
  if (dim > 0) IVFKM_TRY(cudaMemsetAsync(df, 0, sizeof(unsigned long long) * dim, st));
  if (n == 0) return IVFKM_OK;
  df_kernel<<<grid_for(n, 256), 256, 0, st>>>(n, terms, df);
  IVFKM_CHECK_LAUNCH();
  return IVFKM_OK;
}

extern "C" size_t ivfkm_tfidf_workspace_size(int64_t n, int64_t n_docs) {
  Carver c(nullptr);
  c.take<int64_t>((size_t)n_docs + 1);   // doc ptr
  c.take<double>((size_t)(n > 0 ? n : 1));  // weights
  c.take<int64_t>((size_t)n_docs + 1);   // kept
  c.take<double>((size_t)n_docs + 1);    // norms
  c.take<int64_t>((size_t)n_docs + 1);   // kept offsets
  c.take<int64_t>((size_t)n_docs + 1);   // alive
  c.take<int64_t>((size_t)n_docs + 1);   // rank
  size_t a = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, a, (int64_t*)nullptr, (int64_t*)nullptr,
                                (int)(n_docs + 1));
  c.take_bytes(a);
  return c.off;
}

// tf-idf + L2 normalisation of sorted, duplicate-free triples (io.py:131-174)
// given idf[dim] (computed by the caller as the reference does).  Writes the
// surviving documents' CSR (out_ptr[n_alive+1], out_terms / out_vals with
// room for n entries) and the dropped documents (1-based, ascending);
// *counts_out = (n_alive, kept entries) on the host.  Synchronises the stream.
extern "C" int ivfkm_tfidf(int64_t n, int64_t n_docs, int64_t dim, const int32_t* docs,
                           const int32_t* terms, const int32_t* counts, const double* idf,
                           int64_t* out_ptr, int32_t* out_terms, double* out_vals,
                           int32_t* dropped, int64_t* counts_out, void* ws, size_t ws_bytes,
                           ivfkm_stream_t stream_) {
  if (n < 0 || n_docs < 0 || dim < 0 || !counts_out || !out_ptr) return IVFKM_E_ARG;
  if (n_docs >= (int64_t)INT32_MAX) return IVFKM_E_UNSUPPORTED;
  if (ws_bytes < ivfkm_tfidf_workspace_size(n, n_docs)) return IVFKM_E_WORKSPACE;
  cudaStream_t st = as_stream(stream_);
  Carver c(ws);
  int64_t* ptr = c.take<int64_t>((size_t)n_docs + 1);
  double* wts = c.take<double>((size_t)(n > 0 ? n : 1));
  int64_t* kept = c.take<int64_t>((size_t)n_docs + 1);
  double* norm = c.take<double>((size_t)n_docs + 1);
  int64_t* kept_off = c.take<int64_t>((size_t)n_docs + 1);
  int64_t* alive = c.take<int64_t>((size_t)n_docs + 1);
  int64_t* rank = c.take<int64_t>((size_t)n_docs + 1);
  size_t a = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, a, (int64_t*)nullptr, (int64_t*)nullptr,
                                (int)(n_docs + 1));
  void* cub = c.take_bytes(a);
  const int T = 256;
  if (n_docs == 0) {
    IVFKM_TRY(cudaMemsetAsync(out_ptr, 0, sizeof(int64_t), st));
    counts_out[0] = counts_out[1] = 0;
    return IVFKM_OK;
  }
  doc_ptr_kernel<<<grid_for(n + 1, T), T, 0, st>>>(n, n_docs, docs, ptr);
  IVFKM_CHECK_LAUNCH();
  doc_weights_kernel<<<grid_for(n_docs, T), T, 0, st>>>(n_docs, ptr, terms, counts, idf, wts,
                                                        kept, norm);
  IVFKM_CHECK_LAUNCH();
  IVFKM_TRY(cudaMemsetAsync(kept + n_docs, 0, sizeof(int64_t), st));
  size_t cb = a;
  IVFKM_TRY(cub::DeviceScan::ExclusiveSum(cub, cb, kept, kept_off, (int)(n_docs + 1), st));
  survivor_kernel<<<grid_for(n_docs, T), T, 0, st>>>(n_docs, kept, alive);
  IVFKM_CHECK_LAUNCH();
  IVFKM_TRY(cudaMemsetAsync(alive + n_docs, 0, sizeof(int64_t), st));
  cb = a;
  IVFKM_TRY(cub::DeviceScan::ExclusiveSum(cub, cb, alive, rank, (int)(n_docs + 1), st));
  int64_t tot[2] = {0, 0};
  IVFKM_TRY(cudaMemcpyAsync(&tot[0], rank + n_docs, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  IVFKM_TRY(cudaMemcpyAsync(&tot[1], kept_off + n_docs, sizeof(int64_t), cudaMemcpyDeviceToHost,
                            st));
  IVFKM_TRY(cudaStreamSynchronize(st));
  if (tot[0] == 0) IVFKM_TRY(cudaMemsetAsync(out_ptr, 0, sizeof(int64_t), st));
  emit_kernel<<<grid_for(n_docs, T), T, 0, st>>>(n_docs, ptr, terms, wts, norm, kept_off, rank,
                                                 kept, out_ptr, out_terms, out_vals, dropped,
                                                 tot[0]);
  IVFKM_CHECK_LAUNCH();
  IVFKM_TRY(cudaStreamSynchronize(st));
  counts_out[0] = tot[0];
  counts_out[1] = tot[1];
  return IVFKM_OK;
}
