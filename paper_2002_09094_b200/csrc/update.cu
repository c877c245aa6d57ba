// Update step of IVF spherical k-means on sm_100a, bit-identical to the
// reference update_means (reference variants.py:254-307):
//
//   for each cluster j with size > 0:
//     w = bincount(member terms, weights=member values)   # float64, entries
//                                                         # in ascending object order
//     w /= size
//     nrm = sqrt(np.sum(w * w))                           # numpy pairwise sum over
//                                                         # the dense length-D array
//     emit (t, w[t] / nrm) for w[t] != 0, terms ascending
//   empty cluster: copy the previous mean, retained = True
//
// Device plan: key every object nonzero by (label, term) and radix-sort the
// keys stably (CUB onesweep LSD, so equal keys keep ascending object order);
// one thread sums each (cluster, term) run sequentially in that order with
// __dadd_rn (bincount's order), divides by the size; one thread per cluster
// replays numpy's pairwise-summation tree over the run positions (empty
// subtrees contribute exact zeros, so only populated leaves are visited);
// scans give the new CSR offsets; the fill pass writes terms and values.
#include <cub/cub.cuh>
#include <cub/device/device_merge.cuh>
#include <thrust/iterator/counting_iterator.h>
#include <thrust/iterator/transform_iterator.h>

#include <iterator>

#include <algorithm>
#include <map>
#include <mutex>
#include <utility>
#include <vector>

#include "common.cuh"

using namespace ivfkm;

namespace {

template <class K>
struct UpdWs {
  K* key_a;
  K* key_b;
  double* val_a;  // float64 values travel with their keys through the sort
  double* val_b;
  uint32_t* head;     // run-head flags, later nonzero flags
  uint32_t* segpos;   // scan of head
  uint32_t* nzpos;    // scan of nonzero flags
  uint32_t* seg_start;
  K* seg_key;
  double* seg_w;
  uint32_t* cl_seg;   // k+1
  uint32_t* gstart;   // k * (leaf groups + 1): first run of each (cluster, leaf group)
  double* nrm;        // k
  int64_t* counts;    // k+1
  uint32_t* n_seg;    // 1
  int32_t* plan;      // pairwise-sum tree of [0, dim) (NormPlan::buf)
  void* cub;
  size_t cub_bytes;
};

template <class K>
size_t cub_bytes_for(int64_t nnz, int64_t k) {
  size_t a = 0, b = 0, c = 0;
  cub::DoubleBuffer<K> kb(nullptr, nullptr);
  cub::DoubleBuffer<double> vb(nullptr, nullptr);
  cub::DeviceRadixSort::SortPairs(nullptr, a, kb, vb, (int)nnz, 0, (int)(sizeof(K) * 8));
  cub::DeviceScan::ExclusiveSum(nullptr, b, (uint32_t*)nullptr, (uint32_t*)nullptr,
                                (int)nnz + 1);
  cub::DeviceScan::ExclusiveSum(nullptr, c, (int64_t*)nullptr, (int64_t*)nullptr, (int)(k + 1));
  return std::max(a, std::max(b, c));
}

// numpy's pairwise-summation tree over [0, D) (see norm_kernel), built once
// per D on the host: leaves left to right, internal nodes ordered by height
// so that one level can be evaluated in parallel once the lower ones are.
//   buf = leaf_lo[nleaf+1] | lv_off[nlevels+1] | node_l[nint] | node_r[nint]
// node_l/node_r index the value array: leaf j -> j, the q-th internal node
// (level order) -> nleaf + q; the root is the last value.
struct NormPlan {
  int64_t nleaf = 0, nint = 0, nlevels = 0;
  std::vector<int32_t> buf;
};

int64_t norm_plan_ints_max(int64_t dim) { return 4 * (dim / 64 + 2) + 130; }

// The norm kernel takes leaves in groups of kLeafG (one warp, one dense
// shared window of <= kLeafG * 128 positions).
constexpr int kLeafG = 4;
inline int64_t leaf_groups_max(int64_t dim) { return (dim / 64 + 2) / kLeafG + 2; }

const NormPlan& norm_plan(int64_t D) {
  static std::mutex mu;
  static std::map<int64_t, NormPlan> cache;
  std::lock_guard<std::mutex> g(mu);
  auto it = cache.find(D);
  if (it != cache.end()) return it->second;
  std::vector<int32_t> lo;
  struct Node {
    int64_t l, r;  // >= 0: leaf index; < 0: -(internal id) - 1
    int h;
  };
  std::vector<Node> nodes;
  struct Rec {
    std::vector<int32_t>& lo;
    std::vector<Node>& nodes;
    std::pair<int64_t, int> go(int64_t l, int64_t n) {
      if (n <= 128) {
        lo.push_back((int32_t)l);
        return {(int64_t)lo.size() - 1, 0};
      }
      int64_t n2 = n / 2;
      n2 -= n2 % 8;
      const auto a = go(l, n2);
      const auto b = go(l + n2, n - n2);
      const int h = std::max(a.second, b.second) + 1;
      nodes.push_back(Node{a.first, b.first, h});
      return {-(int64_t)nodes.size(), h};
    }
  } rec{lo, nodes};
  rec.go(0, D);
  NormPlan P;
  P.nleaf = (int64_t)lo.size();
  P.nint = (int64_t)nodes.size();
  int H = 0;
  for (const Node& n : nodes) H = std::max(H, n.h);
  P.nlevels = H;
  std::vector<int64_t> order(nodes.size());
  for (size_t i = 0; i < order.size(); ++i) order[i] = (int64_t)i;
  std::stable_sort(order.begin(), order.end(),
                   [&](int64_t a, int64_t b) { return nodes[a].h < nodes[b].h; });
  std::vector<int64_t> pos(nodes.size());
  for (size_t q = 0; q < order.size(); ++q) pos[order[q]] = (int64_t)q;
  auto ref = [&](int64_t r) -> int32_t {
    return (int32_t)(r >= 0 ? r : P.nleaf + pos[-r - 1]);
  };
  P.buf.reserve(P.nleaf + 1 + H + 1 + 2 * P.nint);
  for (int32_t x : lo) P.buf.push_back(x);
  P.buf.push_back((int32_t)D);
  std::vector<int32_t> off(H + 1, 0);
  for (const Node& n : nodes) off[n.h]++;  // heights 1..H -> levels 0..H-1
  int32_t run = 0;
  for (int h = 1; h <= H; ++h) {
    P.buf.push_back(run);
    run += off[h];
  }
  P.buf.push_back(run);
  for (size_t q = 0; q < order.size(); ++q) P.buf.push_back(ref(nodes[order[q]].l));
  for (size_t q = 0; q < order.size(); ++q) P.buf.push_back(ref(nodes[order[q]].r));
  return cache.emplace(D, std::move(P)).first->second;
}

template <class K>
UpdWs<K> carve_upd(void* base, int64_t nnz, int64_t k, int64_t dim, size_t* total) {
  Carver c(base);
  UpdWs<K> w;
  const size_t n = (size_t)(nnz > 0 ? nnz : 1);
  w.key_a = c.take<K>(n);
  w.key_b = c.take<K>(n);
  w.val_a = c.take<double>(n);
  w.val_b = c.take<double>(n);
  w.head = c.take<uint32_t>(n + 1);  // + the closing flag of the nonzero scan
  w.segpos = c.take<uint32_t>(n);
  w.nzpos = c.take<uint32_t>(n + 1);
  w.seg_start = c.take<uint32_t>(n + 1);
  w.seg_key = c.take<K>(n);
  w.seg_w = c.take<double>(n);
  w.cl_seg = c.take<uint32_t>(k + 1);
  w.gstart = c.take<uint32_t>((size_t)k * (size_t)(leaf_groups_max(dim) + 1));
  w.nrm = c.take<double>(k);
  w.counts = c.take<int64_t>(k + 1);
  w.n_seg = c.take<uint32_t>(4);
  w.plan = c.take<int32_t>((size_t)norm_plan_ints_max(dim));
  w.cub_bytes = cub_bytes_for<K>((int64_t)n, k);
  w.cub = c.take_bytes(w.cub_bytes);
  if (total) *total = c.off;
  return w;
}

bool use_k32(int64_t k, int64_t dim) { return (double)k * (double)dim < 4294967295.0; }

int key_bits(int64_t k, int64_t dim) {
  const double top = (double)k * (double)dim;
  int b = 1;
  while ((double)(1ull << b) < top && b < 63) ++b;
  return b;
}

template <class K>
__global__ void keys_kernel(int64_t n_obj, const int64_t* __restrict__ row_ptr,
                            const int32_t* __restrict__ terms, const double* __restrict__ val64,
                            const int32_t* __restrict__ labels, int64_t dim,
                            K* __restrict__ key, double* __restrict__ val) {
  const int lane = threadIdx.x & 31;
  const int64_t wpb = blockDim.x >> 5;
  for (int64_t i = blockIdx.x * wpb + (threadIdx.x >> 5); i < n_obj; i += gridDim.x * wpb) {
    const K base = (K)labels[i] * (K)dim;
    for (int64_t e = row_ptr[i] + lane; e < row_ptr[i + 1]; e += 32) {
      key[e] = base + (K)terms[e];
      val[e] = val64[e];
    }
  }
}

// Sorted (cluster * D + term) keys, read from the key array (full sort) or
// derived from the composite (cluster, term, object) keys of the label-delta
// sort.
template <class K>
struct ArrKey {
  const K* p;
  __device__ __forceinline__ K operator()(int64_t e) const { return p[e]; }
};

template <class K, class R>
__global__ void head_kernel(int64_t nnz, R key, uint32_t* __restrict__ head) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < nnz;
       e += (int64_t)gridDim.x * blockDim.x)
    head[e] = (e == 0 || key(e) != key(e - 1)) ? 1u : 0u;
}

// One thread per (cluster, term) run: sequential float64 sum in ascending
// object order (bincount), then w = sum / size.  Reuses `head` as the
// nonzero flag array, [0, n_seg] (nz[n_seg] = 0 closes the scan).  Runs
// longer than kLongRun (the hot terms: hundreds of members each) go to a
// list summed a warp per run (segsum_long_kernel), so no thread walks a
// long run four loads at a time (split measured best at 64 of 28-128).
// The same pass writes the run tables the norm reads: the first run of
// every cluster (cl_seg) and of every (cluster, leaf group) (gstart) — at
// the runs where the cluster or the group changes, groups and clusters
// holding no run pointing at the next run.
constexpr uint32_t kLongRun = 64;

__device__ __forceinline__ int group_of(int64_t pos, const int32_t* glo, int ng);

template <class K>
__global__ void __launch_bounds__(256) segsum_kernel(
    int64_t n_seg, const uint32_t* __restrict__ seg_start, const K* __restrict__ seg_key,
    const double* __restrict__ sval, const unsigned long long* __restrict__ sizes, int64_t k,
    int64_t dim, const int32_t* __restrict__ plan, int64_t nleaf, double* __restrict__ seg_w,
    uint32_t* __restrict__ nz, uint32_t* __restrict__ long_list, uint32_t* __restrict__ n_long,
    uint32_t* __restrict__ cl_seg, uint32_t* __restrict__ gstart) {
  // glo[ng]: group start positions; tab[pos >> 8]: the group holding the
  // bucket's first position (a group spans >= 256 positions when D > 128, so
  // at most two more starts fall in one bucket)
  extern __shared__ int32_t glo[];
  const int ng = (int)((nleaf + kLeafG - 1) / kLeafG);
  const int nb = (int)(dim >> 8) + 1;
  int32_t* tab = glo + ng;
  for (int g = threadIdx.x; g < ng; g += blockDim.x) glo[g] = plan[(int64_t)g * kLeafG];
  __syncthreads();
  for (int b = threadIdx.x; b < nb; b += blockDim.x) tab[b] = group_of((int64_t)b << 8, glo, ng);
  __syncthreads();
  auto gof = [&](int64_t pos) {
    int g = tab[pos >> 8];
    while (g + 1 < ng && glo[g + 1] <= pos) ++g;
    return g;
  };
  const int64_t stride = ng + 1;
  for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s <= n_seg;
       s += (int64_t)gridDim.x * blockDim.x) {
    if (s == n_seg) {
      nz[s] = 0u;
      continue;
    }
    uint32_t e = seg_start[s];
    const uint32_t end = seg_start[s + 1];
    const K key = seg_key[s];
    const int64_t c = (int64_t)(key / (K)dim);
    // run tables
    {
      const int g = gof((int64_t)(key - (K)c * (K)dim));
      uint32_t* gs = gstart + c * stride;
      int from = 0;
      int64_t pc = -1;
      if (s > 0) {
        const K pk = seg_key[s - 1];
        pc = (int64_t)(pk / (K)dim);
        if (pc == c) from = gof((int64_t)(pk - (K)pc * (K)dim)) + 1;
      }
      for (int q = from; q <= g; ++q) gs[q] = (uint32_t)s;
      for (int64_t q = pc + 1; q <= c; ++q) cl_seg[q] = (uint32_t)s;
      int64_t nc = k;  // the next run's cluster
      if (s + 1 < n_seg) nc = (int64_t)(seg_key[s + 1] / (K)dim);
      if (nc != c) {
        for (int q = g + 1; q <= ng; ++q) gs[q] = (uint32_t)(s + 1);
        if (s + 1 == n_seg)
          for (int64_t q = c + 1; q <= k; ++q) cl_seg[q] = (uint32_t)n_seg;
      }
    }
    if (end - e > kLongRun) {
      long_list[atomicAdd(n_long, 1u)] = (uint32_t)s;
      continue;
    }
    double acc = 0.0;
    for (; e + 4 <= end; e += 4) {  // four loads in flight, adds in order
      const double a = sval[e], b = sval[e + 1], c2 = sval[e + 2], d = sval[e + 3];
      acc = __dadd_rn(__dadd_rn(__dadd_rn(__dadd_rn(acc, a), b), c2), d);
    }
    for (; e < end; ++e) acc = __dadd_rn(acc, sval[e]);
    const double w = __ddiv_rn(acc, (double)sizes[c]);
    seg_w[s] = w;
    nz[s] = (w != 0.0) ? 1u : 0u;
  }
}

// A warp per long run: lanes stage 64 values at a time in shared memory
// (the next 64 already in flight) and lane 0 adds them in order.
template <class K>
__global__ void __launch_bounds__(256) segsum_long_kernel(
    const uint32_t* __restrict__ seg_start, const K* __restrict__ seg_key,
    const double* __restrict__ sval, const unsigned long long* __restrict__ sizes, int64_t dim,
    double* __restrict__ seg_w, uint32_t* __restrict__ nz, const uint32_t* __restrict__ long_list,
    const uint32_t* __restrict__ n_long) {
  __shared__ __align__(16) double s_buf[8][64];
  const int lane = threadIdx.x & 31;
  double* buf = s_buf[threadIdx.x >> 5];
  const double2* buf2 = reinterpret_cast<const double2*>(buf);
  const uint32_t n = *n_long;
  const int64_t wpb = blockDim.x >> 5;
  for (int64_t q = blockIdx.x * wpb + (threadIdx.x >> 5); q < n; q += gridDim.x * wpb) {
    const uint32_t s = long_list[q];
    const uint32_t b = seg_start[s], end = seg_start[s + 1];
    double acc = 0.0;
    double x0 = b + lane < end ? sval[b + lane] : 0.0;
    double x1 = b + 32 + lane < end ? sval[b + 32 + lane] : 0.0;
    for (uint32_t e0 = b; e0 < end; e0 += 64) {
      buf[lane] = x0;
      buf[32 + lane] = x1;
      __syncwarp();
      const uint32_t e1 = e0 + 64;
      x0 = e1 + lane < end ? sval[e1 + lane] : 0.0;
      x1 = e1 + 32 + lane < end ? sval[e1 + 32 + lane] : 0.0;
      if (lane == 0) {
        const uint32_t m = end - e0 < 64 ? end - e0 : 64;
        if (m == 64) {
#pragma unroll
          for (int j = 0; j < 32; ++j) {
            const double2 v = buf2[j];
            acc = __dadd_rn(__dadd_rn(acc, v.x), v.y);
          }
        } else {
          for (uint32_t j = 0; j < m; ++j) acc = __dadd_rn(acc, buf[j]);
        }
      }
      __syncwarp();
    }
    if (lane == 0) {
      const int64_t c = (int64_t)(seg_key[s] / (K)dim);
      const double w = __ddiv_rn(acc, (double)sizes[c]);
      seg_w[s] = w;
      nz[s] = (w != 0.0) ? 1u : 0u;
    }
  }
}

template <class K>
__global__ void clseg_kernel(int64_t k, int64_t dim, const uint32_t* __restrict__ n_seg_p,
                             const K* __restrict__ seg_key, uint32_t* __restrict__ cl_seg) {
  const uint32_t n_seg = *n_seg_p;
  for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c <= k;
       c += (int64_t)gridDim.x * blockDim.x) {
    const K target = (K)c * (K)dim;
    uint32_t lo = 0, hi = n_seg;
    while (lo < hi) {
      const uint32_t mid = (lo + hi) >> 1;
      if (seg_key[mid] < target) lo = mid + 1; else hi = mid;
    }
    cl_seg[c] = c == k ? n_seg : lo;
  }
}

// numpy's pairwise summation (numpy/_core/src/umath/loops_utils.h.src,
// pairwise_sum) over the dense length-D array w*w, replayed on the sparse
// support.  The recursion splits a range of n > 128 elements at
// n2 = n/2 - (n/2)%8, so its leaves (64..128 elements, or the whole array
// when D <= 128) depend on D only; a leaf of >= 8 elements sums into 8
// strided accumulators combined as ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)) plus a
// sequential tail, a leaf under 8 elements is a plain sequential sum.  Zeros
// add exact +0.0, so only the cluster's nonzeros need visiting (scattered
// into a zeroed window by norm_kernel).
// (test_gpu_parity.py::test_update_norm_across_dims checks it at many D.)

// First run of every (cluster, leaf group): runs are sorted by (cluster,
// term), so group boundaries are where the group of consecutive runs'
// positions changes; groups holding no run point at the next run.
__device__ __forceinline__ int group_of(int64_t pos, const int32_t* glo, int ng) {
  int lo = 0, hi = ng - 1;  // last g with glo[g] <= pos
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (glo[mid] <= pos) lo = mid; else hi = mid - 1;
  }
  return lo;
}

template <class K, class R>
__global__ void segstart_kernel(int64_t nnz, R key, const uint32_t* __restrict__ head,
                                const uint32_t* __restrict__ segpos,
                                uint32_t* __restrict__ seg_start, K* __restrict__ seg_key,
                                uint32_t* __restrict__ n_seg) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < nnz;
       e += (int64_t)gridDim.x * blockDim.x) {
    if (head[e]) {
      seg_start[segpos[e]] = (uint32_t)e;
      seg_key[segpos[e]] = key(e);
    }
    if (e == nnz - 1) {
      const uint32_t ns = segpos[e] + head[e];
      *n_seg = ns;
      seg_start[ns] = (uint32_t)nnz;
    }
  }
}

// One CTA per cluster, one warp per group of kLeafG leaves: the group's runs
// (a contiguous range, gstart) put w*w into the warp's zeroed dense window
// (absent terms stay 0.0); lane 8i+j sums leaf i's strided accumulator j,
// shuffles combine them in numpy's order, lane 8i adds the tail.  The
// internal nodes are then evaluated level by level.
constexpr int kNormWarps = 16;

template <class K>
__global__ void __launch_bounds__(kNormWarps * 32) norm_kernel(
    int64_t k, int64_t dim, int64_t nleaf, int64_t nint, int64_t nlevels,
    const int32_t* __restrict__ plan, const unsigned long long* __restrict__ sizes,
    const int64_t* __restrict__ prev_ptr, const uint32_t* __restrict__ cl_seg,
    const uint32_t* __restrict__ gstart, const K* __restrict__ seg_key,
    const double* __restrict__ seg_w, const uint32_t* __restrict__ nzpos,
    double* __restrict__ nrm, int64_t* __restrict__ counts) {
  extern __shared__ __align__(16) unsigned char smem[];
  double* win_all = reinterpret_cast<double*>(smem);              // warps * kLeafG * 128
  double* val = win_all + kNormWarps * kLeafG * 128;               // nleaf + nint
  int32_t* leaf_lo = reinterpret_cast<int32_t*>(val + nleaf + nint);  // nleaf + 1
  const int32_t* lv_off = plan + nleaf + 1;
  const int32_t* node_l = lv_off + nlevels + 1;
  const int32_t* node_r = node_l + nint;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double* win = win_all + warp * kLeafG * 128;
  const int ng = (int)((nleaf + kLeafG - 1) / kLeafG);
  for (int64_t j = threadIdx.x; j <= nleaf; j += blockDim.x) leaf_lo[j] = plan[j];
  if (blockIdx.x == 0 && threadIdx.x == 0) counts[k] = 0;
  __syncthreads();
  for (int64_t c = blockIdx.x; c < k; c += gridDim.x) {
    if (sizes[c] == 0) {  // retained: previous mean, count only
      if (threadIdx.x == 0) {
        counts[c] = prev_ptr[c + 1] - prev_ptr[c];
        nrm[c] = 1.0;
      }
      continue;
    }
    const uint32_t* gs = gstart + c * (int64_t)(ng + 1);
    const K base = (K)c * (K)dim;
    const bool no_runs = cl_seg[c] == cl_seg[c + 1];  // members with empty rows only
    for (int g = warp; g < ng; g += kNormWarps) {
      const uint32_t s0 = no_runs ? 0u : gs[g], s1 = no_runs ? 0u : gs[g + 1];
      const int l0 = g * kLeafG;
      const int nl = (int)(nleaf - l0 < kLeafG ? nleaf - l0 : kLeafG);
      const int p0 = leaf_lo[l0], np = leaf_lo[l0 + nl] - p0;
      for (int i = lane; i < np; i += 32) win[i] = 0.0;
      __syncwarp();
      for (uint32_t sidx = s0 + lane; sidx < s1; sidx += 32) {
        const double w = seg_w[sidx];
        win[(int64_t)(seg_key[sidx] - base) - p0] = __dmul_rn(w, w);
      }
      __syncwarp();
      const int li = lane >> 3, j = lane & 7;
      const bool has = li < nl;
      const int lo = has ? leaf_lo[l0 + li] - p0 : 0;
      const int n = has ? leaf_lo[l0 + li + 1] - leaf_lo[l0 + li] : 0;
      double r = 0.0;
      if (n < 8) {
        if (j == 0)
          for (int i = 0; i < n; ++i) r = __dadd_rn(r, win[lo + i]);
      } else {
        const int lim = n - (n & 7);
        for (int i = j; i < lim; i += 8) r = __dadd_rn(r, win[lo + i]);
      }
      // ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7))
      const double r1 = __shfl_down_sync(kFull, r, 1);
      const double a = __dadd_rn(r, r1);
      const double a2 = __shfl_down_sync(kFull, a, 2);
      const double b2 = __dadd_rn(a, a2);
      const double b4 = __shfl_down_sync(kFull, b2, 4);
      const double c8 = __dadd_rn(b2, b4);
      if (has && j == 0) {
        double res;
        if (n < 8) {
          res = r;
        } else {
          res = c8;
          for (int i = n - (n & 7); i < n; ++i) res = __dadd_rn(res, win[lo + i]);
        }
        val[l0 + li] = res;
      }
      __syncwarp();
    }
    __syncthreads();
    // internal nodes level by level: pw(node) = pw(left) + pw(right)
    for (int64_t l = 0; l < nlevels; ++l) {
      for (int64_t q = lv_off[l] + threadIdx.x; q < lv_off[l + 1]; q += blockDim.x)
        val[nleaf + q] = __dadd_rn(val[node_l[q]], val[node_r[q]]);
      __syncthreads();
    }
    if (threadIdx.x == 0) {
      const uint32_t b = cl_seg[c], e = cl_seg[c + 1];
      counts[c] = (int64_t)nzpos[e] - (int64_t)nzpos[b];
      nrm[c] = __dsqrt_rn(val[nleaf + nint - 1]);
    }
    __syncthreads();
  }
}

template <class K>
__global__ void fill_kernel(int64_t nnz, int64_t dim, const uint32_t* __restrict__ n_seg_p,
                            const K* __restrict__ seg_key, const double* __restrict__ seg_w,
                            const uint32_t* __restrict__ nz, const uint32_t* __restrict__ nzpos,
                            const uint32_t* __restrict__ cl_seg, const double* __restrict__ nrm,
                            const int64_t* __restrict__ new_ptr, int32_t* __restrict__ new_terms,
                            double* __restrict__ new_vals, int64_t capacity) {
  const uint32_t n_seg = *n_seg_p;
  for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < n_seg;
       s += (int64_t)gridDim.x * blockDim.x) {
    if (!nz[s]) continue;
    const int64_t c = (int64_t)(seg_key[s] / (K)dim);
    const int64_t t = (int64_t)(seg_key[s] - (K)c * (K)dim);
    const int64_t pos = new_ptr[c] + (int64_t)(nzpos[s] - nzpos[cl_seg[c]]);
    if (pos >= capacity) continue;  // caller's buffer too small: never write past it
    new_terms[pos] = (int32_t)t;
    new_vals[pos] = __ddiv_rn(seg_w[s], nrm[c]);
  }
}

__global__ void retain_kernel(int64_t k, const unsigned long long* __restrict__ sizes,
                              const int64_t* __restrict__ prev_ptr,
                              const int32_t* __restrict__ prev_terms,
                              const double* __restrict__ prev_vals,
                              const int64_t* __restrict__ new_ptr, int32_t* __restrict__ new_terms,
                              double* __restrict__ new_vals, uint8_t* __restrict__ retained,
                              int64_t capacity) {
  const int lane = threadIdx.x & 31;
  const int64_t wpb = blockDim.x >> 5;
  for (int64_t c = blockIdx.x * wpb + (threadIdx.x >> 5); c < k; c += gridDim.x * wpb) {
    const bool empty = sizes[c] == 0;
    if (lane == 0) retained[c] = empty ? 1 : 0;
    if (!empty) continue;
    const int64_t pb = prev_ptr[c], nb = new_ptr[c];
    int64_t n = prev_ptr[c + 1] - pb;
    if (nb + n > capacity) n = capacity > nb ? capacity - nb : 0;
    for (int64_t q = lane; q < n; q += 32) {
      new_terms[nb + q] = prev_terms[pb + q];
      new_vals[nb + q] = prev_vals[pb + q];
    }
  }
}

// ---------------------------------------------------------------------------
// Label-delta sort (optional state, ivfkm_update_count_delta).  After the
// first iterations only a few percent of the objects change cluster, so the
// previous iteration's sorted entries are kept as composite keys
// (label, term, object) — unique, so every order is the stable order — and
// updated by (1) dropping the changed objects' entries (stable compaction),
// (2) keying and sorting those entries under their new labels, (3) merging
// the two sorted runs.  Iterations where more than a quarter of the entries
// move fall back to one full sort of the composite keys.

struct DeltaHdr {
  long long magic, n_obj, nnz, k, dim, valid, cur, pad;
};
constexpr long long kDeltaMagic = 0x69766b6d64656c74ll;

struct DeltaState {
  DeltaHdr* hdr;
  int32_t* labels;               // the labels S was built with
  unsigned long long* key[2];    // S: composite keys
  double* val[2];                // S: values
  unsigned long long* bkey[2];   // changed entries (B), capacity nnz/4
  double* bval[2];
  uint8_t* oflag;                // n_obj: changed
  uint32_t* obits;               // n_obj bits: changed (the merge's lookups stay in L1)
  int32_t* clist;                // n_obj: changed objects
  int64_t* cptr;                 // n_obj+1: their entry offsets in B
  unsigned long long* counts;    // [0] changed objects, [1] their entries, [2] selected
  int32_t* plan;                 // the norm's tree plan, uploaded once (hdr.pad = its dim)
  int64_t* tcnt;                 // merge with deletions: kept entries per tile, scanned
  int64_t* tb;                   // B entries below each tile's first key
  void* cub;
  size_t cub_bytes;
};

struct KeptFlag {
  const unsigned long long* key;
  const uint8_t* oflag;
  unsigned long long omask;
  __device__ __forceinline__ uint8_t operator()(int64_t e) const {
    return oflag[key[e] & omask] ? 0 : 1;
  }
};

int64_t delta_cap(int64_t nnz) { return nnz / 4 + 1024; }

// 0: one fused merge with deletions (mdel_*_kernel); 1: round 1's two CUB
// stable selects + CUB merge (A/B and tests; ivfkm_set_update_option)
int g_delta_cub_merge = 0;

DeltaState carve_delta(void* base, int64_t n_obj, int64_t nnz, int64_t dim, size_t* total) {
  Carver c(base);
  DeltaState d;
  const size_t n = (size_t)(nnz > 0 ? nnz : 1), no = (size_t)(n_obj > 0 ? n_obj : 1);
  const size_t nb = (size_t)delta_cap(nnz);
  d.hdr = c.take<DeltaHdr>(1);
  d.labels = c.take<int32_t>(no);
  for (int b = 0; b < 2; ++b) {
    d.key[b] = c.take<unsigned long long>(n);
    d.val[b] = c.take<double>(n);
    d.bkey[b] = c.take<unsigned long long>(nb);
    d.bval[b] = c.take<double>(nb);
  }
  d.oflag = c.take<uint8_t>(no);
  d.obits = c.take<uint32_t>(no / 32 + 1);
  d.clist = c.take<int32_t>(no);
  d.cptr = c.take<int64_t>(no + 1);
  d.counts = c.take<unsigned long long>(4);
  d.plan = c.take<int32_t>((size_t)norm_plan_ints_max(dim));
  d.tcnt = c.take<int64_t>((size_t)n / 2048 + 2);
  d.tb = c.take<int64_t>((size_t)n / 2048 + 2);
  size_t a = 0, b = 0, m = 0, sc = 0, so = 0, st = 0;
  cub::DoubleBuffer<unsigned long long> kb(nullptr, nullptr);
  cub::DoubleBuffer<double> vb(nullptr, nullptr);
  cub::DeviceRadixSort::SortPairs(nullptr, a, kb, vb, (int)n, 0, 64);
  {
    auto kept = thrust::make_transform_iterator(thrust::counting_iterator<int64_t>(0),
                                                KeptFlag{nullptr, nullptr, 0ull});
    size_t b1 = 0, b2 = 0;
    cub::DeviceSelect::Flagged(nullptr, b1, (unsigned long long*)nullptr, kept,
                               (unsigned long long*)nullptr, (unsigned long long*)nullptr, (int)n);
    cub::DeviceSelect::Flagged(nullptr, b2, (double*)nullptr, kept, (double*)nullptr,
                               (unsigned long long*)nullptr, (int)n);
    b = std::max(b1, b2);
  }
  cub::DeviceMerge::MergePairs(nullptr, m, (unsigned long long*)nullptr, (double*)nullptr, (int)n,
                               (unsigned long long*)nullptr, (double*)nullptr, (int)nb,
                               (unsigned long long*)nullptr, (double*)nullptr);
  cub::DeviceScan::ExclusiveSum(nullptr, sc, (int64_t*)nullptr, (int64_t*)nullptr, (int)no + 1);
  cub::DeviceSelect::Flagged(nullptr, so, (int32_t*)nullptr, (uint8_t*)nullptr,
                             (int32_t*)nullptr, (unsigned long long*)nullptr, (int)no);
  cub::DeviceScan::ExclusiveSum(nullptr, st, (int64_t*)nullptr, (int64_t*)nullptr,
                                (int)(n / 2048 + 2));
  d.cub_bytes = std::max(std::max(std::max(a, b), st), std::max(std::max(m, sc), so));
  d.cub = c.take_bytes(d.cub_bytes);
  if (total) *total = c.off;
  return d;
}

struct Bits {
  int ob, tb, lb;
  unsigned long long omask, tmask;
};

inline int bits_for(int64_t n) {
  int b = 1;
  while (b < 63 && (1ll << b) < n) ++b;
  return b;
}

Bits comp_bits(int64_t n_obj, int64_t dim, int64_t k) {
  Bits b;
  b.ob = bits_for(n_obj);
  b.tb = bits_for(dim);
  b.lb = bits_for(k);
  b.omask = (1ull << b.ob) - 1ull;
  b.tmask = (1ull << b.tb) - 1ull;
  return b;
}

__global__ void comp_keys_kernel(int64_t n_obj, const int64_t* __restrict__ row_ptr,
                                 const int32_t* __restrict__ terms,
                                 const double* __restrict__ val64,
                                 const int32_t* __restrict__ labels,
                                 const int32_t* __restrict__ objs, int64_t n_list,
                                 const int64_t* __restrict__ out_ptr, Bits bt,
                                 unsigned long long* __restrict__ key, double* __restrict__ val) {
  // one warp per object: all objects (objs == nullptr) or the listed ones
  const int lane = threadIdx.x & 31;
  const int64_t wpb = blockDim.x >> 5;
  const int64_t n = objs ? n_list : n_obj;
  for (int64_t q = blockIdx.x * wpb + (threadIdx.x >> 5); q < n; q += gridDim.x * wpb) {
    const int64_t i = objs ? objs[q] : q;
    const int64_t rb = row_ptr[i], re = row_ptr[i + 1];
    const int64_t o = objs ? out_ptr[q] : rb;
    const unsigned long long hi = ((unsigned long long)labels[i] << (bt.tb + bt.ob)) |
                                  (unsigned long long)i;
    for (int64_t e = rb + lane; e < re; e += 32) {
      key[o + (e - rb)] = hi | ((unsigned long long)terms[e] << bt.ob);
      val[o + (e - rb)] = val64[e];
    }
  }
}

__global__ void changed_kernel(int64_t n_obj, const int32_t* __restrict__ labels,
                               const int32_t* __restrict__ old, const int64_t* __restrict__ row_ptr,
                               uint8_t* __restrict__ oflag, uint32_t* __restrict__ obits,
                               int64_t* __restrict__ len, unsigned long long* __restrict__ counts) {
  unsigned long long co = 0, ce = 0;
  // whole warps walk 32 consecutive objects (the ballot is one mask word)
  const int64_t n32 = (n_obj + 31) & ~31ll;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n32;
       i += (int64_t)gridDim.x * blockDim.x) {
    const bool in = i < n_obj;
    const bool ch = in && labels[i] != old[i];
    const unsigned m = __ballot_sync(0xffffffffu, ch);
    if ((threadIdx.x & 31) == 0) obits[i >> 5] = m;
    if (in) {
      oflag[i] = ch ? 1 : 0;
      const int64_t l = ch ? row_ptr[i + 1] - row_ptr[i] : 0;
      len[i] = l;
      co += ch;
      ce += (unsigned long long)l;
    }
  }
  for (int off = 16; off > 0; off >>= 1) {
    co += __shfl_xor_sync(0xffffffffu, co, off);
    ce += __shfl_xor_sync(0xffffffffu, ce, off);
  }
  if ((threadIdx.x & 31) == 0 && (co | ce)) {
    atomicAdd(&counts[0], co);
    atomicAdd(&counts[1], ce);
  }
}

// lens of the listed changed objects (in list order) for the B offsets
__global__ void list_len_kernel(int64_t n_list, const int32_t* __restrict__ objs,
                                const int64_t* __restrict__ row_ptr, int64_t* __restrict__ len) {
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < n_list;
       q += (int64_t)gridDim.x * blockDim.x)
    len[q] = row_ptr[objs[q] + 1] - row_ptr[objs[q]];
}

// composite (label, term, obj) -> the (label * dim + term) key of the classic path
template <class K>
struct CompKey {
  const unsigned long long* p;
  Bits bt;
  int64_t dim;
  __device__ __forceinline__ K operator()(int64_t e) const {
    const unsigned long long c = p[e];
    return (K)(c >> (bt.tb + bt.ob)) * (K)dim + (K)((c >> bt.ob) & bt.tmask);
  }
};

__global__ void set_hdr_kernel(DeltaHdr* hdr, DeltaHdr v) { *hdr = v; }

// Merge with deletions: O = merge(S minus the changed objects' entries, B),
// every output position computed directly (keys are unique, so the order is
// the full sort's).  S is cut into tiles of kMTile entries; tile t's output
// starts after the kept entries of the tiles before it (scan of the tile
// counts) and the B entries below its first key (tb[t], a binary search).
// Inside a tile every B entry finds its insertion point L among the tile's
// keys (binary search in shared memory) and bumps a count at L; one block
// scan over (kept flag, B count) pairs packed in 16-bit halves then places
// both: a kept entry at i after the kept entries and the B entries inserted
// at or before i, a B entry after the kept entries below L and the B entries
// before it.  A tile holding more than kMBCap B entries (movers piled into
// one region) places its kept entries by binary searches in global B
// instead.  Keys and values are read once into registers, the changed
// objects are one bit each (an L1-resident mask where the objects are a few
// hundred thousand): one read of S's keys for the tile counts, one read of
// keys + values and one write — where two stable selects and a merge path
// read and wrote S twice.
constexpr int kMT = 256, kMPer = 8, kMTile = kMT * kMPer, kMBPer = 4, kMBCap = kMT * kMBPer;

int64_t mdel_tiles(int64_t n) { return (n + kMTile - 1) / kMTile; }

__device__ __forceinline__ bool mdel_kept(const uint32_t* __restrict__ obits,
                                          unsigned long long k, unsigned long long omask) {
  const unsigned long long o = k & omask;
  return !((__ldg(obits + (o >> 5)) >> (o & 31)) & 1u);
}

__global__ void __launch_bounds__(kMT) mdel_count_kernel(
    int64_t n, const unsigned long long* __restrict__ key, const uint32_t* __restrict__ obits,
    unsigned long long omask, int64_t* __restrict__ tcnt) {
  __shared__ int wsum[kMT / 32];
  const int64_t t = blockIdx.x, i0 = t * kMTile;
  const int len = (int)min((int64_t)kMTile, n - i0);
  unsigned long long kk[kMPer];
#pragma unroll
  for (int r = 0; r < kMPer; ++r) {
    const int i = r * kMT + threadIdx.x;
    kk[r] = i < len ? __ldcs(key + i0 + i) : 0ull;
  }
  int c = 0;
#pragma unroll
  for (int r = 0; r < kMPer; ++r)
    if (r * kMT + (int)threadIdx.x < len) c += mdel_kept(obits, kk[r], omask) ? 1 : 0;
  c = __reduce_add_sync(0xffffffffu, c);
  if ((threadIdx.x & 31) == 0) wsum[threadIdx.x >> 5] = c;
  __syncthreads();
  if (threadIdx.x == 0) {
    int s = 0;
#pragma unroll
    for (int w = 0; w < kMT / 32; ++w) s += wsum[w];
    tcnt[t] = s;
    if (t == gridDim.x - 1) tcnt[t + 1] = 0;
  }
}

// tb[t] = B entries below tile t's first key (one thread per tile: the
// binary searches' dependent loads overlap across tiles instead of holding
// a counting CTA each)
__global__ void mdel_tb_kernel(int64_t n, int64_t nt, const unsigned long long* __restrict__ key,
                               const unsigned long long* __restrict__ bkey, int64_t nb,
                               int64_t* __restrict__ tb) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t > nt) return;
  int64_t lo = 0;
  if (t == nt) {
    lo = nb;
  } else if (t > 0) {
    const unsigned long long k0 = key[t * kMTile];
    int64_t hi = nb;
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      if (bkey[mid] < k0) lo = mid + 1;
      else hi = mid;
    }
  }
  tb[t] = lo;
}

__global__ void __launch_bounds__(kMT, 4) mdel_merge_kernel(
    int64_t n, const unsigned long long* __restrict__ key, const double* __restrict__ val,
    const uint32_t* __restrict__ obits, unsigned long long omask,
    const unsigned long long* __restrict__ bkey, const double* __restrict__ bval,
    const int64_t* __restrict__ tpre, const int64_t* __restrict__ tb,
    unsigned long long* __restrict__ okey, double* __restrict__ oval) {
  __shared__ unsigned long long sk[kMTile];
  // per position: kept flag (low half) + B entries inserted there (high
  // half), scanned in place to the exclusive prefix; [kMTile] = the totals
  __shared__ __align__(16) uint32_t sv[kMTile + 1];
  __shared__ uint32_t wsum[kMT / 32];
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int64_t t = blockIdx.x, i0 = t * kMTile;
  const int len = (int)min((int64_t)kMTile, n - i0);
  const int64_t jb = tb[t], je = tb[t + 1];
  const int nbt = (int)(je - jb);
  const bool fits = nbt <= kMBCap;
  unsigned long long kk[kMPer];
  double vv[kMPer];
#pragma unroll
  for (int r = 0; r < kMPer; ++r) {
    const int i = r * kMT + tid;
    kk[r] = i < len ? __ldcs(key + i0 + i) : ~0ull;
    vv[r] = i < len ? __ldcs(val + i0 + i) : 0.0;
  }
  unsigned long long bk[kMBPer];
  if (fits) {
#pragma unroll
    for (int r = 0; r < kMBPer; ++r) {
      const int j = r * kMT + tid;
      bk[r] = j < nbt ? __ldcs(bkey + jb + j) : 0ull;
    }
  }
  unsigned kept = 0;
#pragma unroll
  for (int r = 0; r < kMPer; ++r) {
    const int i = r * kMT + tid;
    const bool f = i < len && mdel_kept(obits, kk[r], omask);
    kept |= (f ? 1u : 0u) << r;
    sk[i] = kk[r];
    sv[i] = f ? 1u : 0u;
  }
  __syncthreads();
  int bl[kMBPer];
  if (fits) {
#pragma unroll
    for (int r = 0; r < kMBPer; ++r) {
      const int j = r * kMT + tid;
      int lo = 0;
      if (j < nbt) {
        int hi = len;
        while (lo < hi) {
          const int mid = (lo + hi) >> 1;
          if (sk[mid] < bk[r]) lo = mid + 1;
          else hi = mid;
        }
        if (lo < kMTile) atomicAdd(&sv[lo], 1u << 16);
      }
      bl[r] = lo;
    }
    __syncthreads();
  }
  // blocked exclusive scan: thread tid owns [tid*kMPer, tid*kMPer + kMPer)
  uint4 a = *reinterpret_cast<const uint4*>(sv + tid * kMPer);
  uint4 b = *reinterpret_cast<const uint4*>(sv + tid * kMPer + 4);
  uint32_t e[kMPer] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
  uint32_t c = 0;
#pragma unroll
  for (int q = 0; q < kMPer; ++q) c += e[q];
  uint32_t inc = c;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t v = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += v;
  }
  if (lane == 31) wsum[wid] = inc;
  __syncthreads();
  uint32_t run = 0, total = 0;
#pragma unroll
  for (int w = 0; w < kMT / 32; ++w) {
    run += w < wid ? wsum[w] : 0u;
    total += wsum[w];
  }
  run += inc - c;
#pragma unroll
  for (int q = 0; q < kMPer; ++q) {
    const uint32_t x = e[q];
    e[q] = run;
    run += x;
  }
  *reinterpret_cast<uint4*>(sv + tid * kMPer) = make_uint4(e[0], e[1], e[2], e[3]);
  *reinterpret_cast<uint4*>(sv + tid * kMPer + 4) = make_uint4(e[4], e[5], e[6], e[7]);
  if (tid == 0) sv[kMTile] = total;
  __syncthreads();
  const int64_t base = tpre[t];
  // kept entries (striped: near-contiguous writes)
#pragma unroll
  for (int r = 0; r < kMPer; ++r) {
    if (!((kept >> r) & 1u)) continue;
    const int i = r * kMT + tid;
    int64_t nbelow;  // this tile's B entries below the key
    if (fits) {
      nbelow = (int64_t)(sv[i + 1] >> 16);  // inserted at positions <= i
    } else {
      int64_t lo = 0, hi = nbt;
      while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if (bkey[jb + mid] < kk[r]) lo = mid + 1;
        else hi = mid;
      }
      nbelow = lo;
    }
    const int64_t pos = base + jb + (int64_t)(sv[i] & 0xffffu) + nbelow;
    __stcs(okey + pos, kk[r]);
    __stcs(oval + pos, vv[r]);
  }
  // this tile's B entries
  if (fits) {
#pragma unroll
    for (int r = 0; r < kMBPer; ++r) {
      const int j = r * kMT + tid;
      if (j < nbt) {
        const int64_t pos = base + (int64_t)(sv[bl[r]] & 0xffffu) + jb + j;
        __stcs(okey + pos, bk[r]);
        __stcs(oval + pos, __ldcs(bval + jb + j));
      }
    }
  } else {
    for (int j = tid; j < nbt; j += kMT) {
      const unsigned long long k = bkey[jb + j];
      int lo = 0, hi = len;
      while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (sk[mid] < k) lo = mid + 1;
        else hi = mid;
      }
      const int64_t pos = base + (int64_t)(sv[lo] & 0xffffu) + jb + j;
      okey[pos] = k;
      oval[pos] = bval[jb + j];
    }
  }
}

// Sorted (key, value) for this update: the composite-key state S brought up to
// the current labels (incrementally when few objects moved); returns the S
// buffers through *sk / *sv.
int delta_sort(int64_t n_obj, const int64_t* row_ptr, const int32_t* terms, const double* val64,
               int64_t nnz, int64_t k, int64_t dim, const int32_t* labels, DeltaState& d,
               const unsigned long long** sk, const double** sv, int64_t* moved,
               bool* plan_ok, cudaStream_t st) {
  const Bits bt = comp_bits(n_obj, dim, k);
  const int total_bits = bt.ob + bt.tb + bt.lb;
  const int T = 256;
  // the header and the movers' counts come back in one read (on a fresh
  // state the counts are computed against zeros and ignored)
  DeltaHdr h;
  unsigned long long cnt[2] = {0, 0};
  IVFKM_TRY(cudaMemsetAsync(d.counts, 0, sizeof(unsigned long long) * 4, st));
  changed_kernel<<<grid_for(n_obj, T), T, 0, st>>>(n_obj, labels, d.labels, row_ptr, d.oflag,
                                                  d.obits, d.cptr, d.counts);
  IVFKM_CHECK_LAUNCH();
  IVFKM_TRY(cudaMemcpyAsync(&h, d.hdr, sizeof(h), cudaMemcpyDeviceToHost, st));
  IVFKM_TRY(cudaMemcpyAsync(cnt, d.counts, sizeof(cnt), cudaMemcpyDeviceToHost, st));
  IVFKM_TRY(cudaStreamSynchronize(st));
  bool full = !(h.magic == kDeltaMagic && h.valid == 1 && h.n_obj == n_obj && h.nnz == nnz &&
                h.k == k && h.dim == dim && (h.cur == 0 || h.cur == 1));
  int cur = full ? 0 : (int)h.cur;
  *plan_ok = !full && h.pad == dim;  // same layout, plan already uploaded
  if (!full && (int64_t)cnt[1] > delta_cap(nnz) - 1024) full = true;
  if (full) {
    comp_keys_kernel<<<grid_for(n_obj, T / 32), T, 0, st>>>(n_obj, row_ptr, terms, val64, labels,
                                                           nullptr, 0, nullptr, bt, d.key[0],
                                                           d.val[0]);
    IVFKM_CHECK_LAUNCH();
    cub::DoubleBuffer<unsigned long long> kb(d.key[0], d.key[1]);
    cub::DoubleBuffer<double> vb(d.val[0], d.val[1]);
    size_t cb = d.cub_bytes;
    // the entries are produced in object order and the radix sort is stable,
    // so sorting the (label, term) bits alone leaves equal pairs in object
    // order: the object bits need no passes
    IVFKM_TRY(cub::DeviceRadixSort::SortPairs(d.cub, cb, kb, vb, (int)nnz, bt.ob, total_bits,
                                              st));
    cur = kb.selector;
    *moved = nnz;
  } else if (cnt[1] > 0) {
    const int oth = cur ^ 1;
    const int64_t nb = (int64_t)cnt[1], nc = (int64_t)cnt[0];
    size_t cb = d.cub_bytes;
    // B: the changed objects' entries under their new labels, sorted
    {
      // list the changed objects (ascending ids)
      cub::CountingInputIterator<int32_t> it(0);
      cb = d.cub_bytes;
      IVFKM_TRY(cub::DeviceSelect::Flagged(d.cub, cb, it, d.oflag, d.clist, d.counts + 3,
                                           (int)n_obj, st));
    }
    list_len_kernel<<<grid_for(nc, T), T, 0, st>>>(nc, d.clist, row_ptr, d.cptr);
    IVFKM_CHECK_LAUNCH();
    IVFKM_TRY(cudaMemsetAsync(d.cptr + nc, 0, sizeof(int64_t), st));
    cb = d.cub_bytes;
    IVFKM_TRY(cub::DeviceScan::ExclusiveSum(d.cub, cb, d.cptr, d.cptr, (int)nc + 1, st));
    comp_keys_kernel<<<grid_for(nc, T / 32), T, 0, st>>>(n_obj, row_ptr, terms, val64, labels,
                                                        d.clist, nc, d.cptr, bt, d.bkey[0],
                                                        d.bval[0]);
    IVFKM_CHECK_LAUNCH();
    cub::DoubleBuffer<unsigned long long> kb(d.bkey[0], d.bkey[1]);
    cub::DoubleBuffer<double> vb(d.bval[0], d.bval[1]);
    cb = d.cub_bytes;
    // movers listed in ascending object order: (label, term) bits only, as above
    IVFKM_TRY(cub::DeviceRadixSort::SortPairs(d.cub, cb, kb, vb, (int)nb, bt.ob, total_bits,
                                              st));
    if (g_delta_cub_merge) {
      // A: the unchanged objects' entries, in order (the kept flags computed
      // from the keys inside both selects: no flag pass); merge A (oth) and
      // B into cur (keys are unique: no ties to order)
      auto kept = thrust::make_transform_iterator(thrust::counting_iterator<int64_t>(0),
                                                  KeptFlag{d.key[cur], d.oflag, bt.omask});
      cb = d.cub_bytes;
      IVFKM_TRY(cub::DeviceSelect::Flagged(d.cub, cb, d.key[cur], kept, d.key[oth],
                                           d.counts + 2, (int)nnz, st));
      cb = d.cub_bytes;
      IVFKM_TRY(cub::DeviceSelect::Flagged(d.cub, cb, d.val[cur], kept, d.val[oth],
                                           d.counts + 2, (int)nnz, st));
      cb = d.cub_bytes;
      IVFKM_TRY(cub::DeviceMerge::MergePairs(d.cub, cb, d.key[oth], d.val[oth], (int)(nnz - nb),
                                             kb.Current(), vb.Current(), (int)nb, d.key[cur],
                                             d.val[cur], ::cuda::std::less<>{}, st));
    } else {
      // one fused merge with deletions, S (cur) -> oth
      const int64_t nt = mdel_tiles(nnz);
      mdel_tb_kernel<<<grid_for(nt + 1, T), T, 0, st>>>(nnz, nt, d.key[cur], kb.Current(), nb,
                                                         d.tb);
      IVFKM_CHECK_LAUNCH();
      mdel_count_kernel<<<(unsigned)nt, kMT, 0, st>>>(nnz, d.key[cur], d.obits, bt.omask, d.tcnt);
      IVFKM_CHECK_LAUNCH();
      cb = d.cub_bytes;
      IVFKM_TRY(cub::DeviceScan::ExclusiveSum(d.cub, cb, d.tcnt, d.tcnt, (int)nt + 1, st));
      mdel_merge_kernel<<<(unsigned)nt, kMT, 0, st>>>(nnz, d.key[cur], d.val[cur], d.obits,
                                                      bt.omask, kb.Current(), vb.Current(),
                                                      d.tcnt, d.tb, d.key[oth], d.val[oth]);
      IVFKM_CHECK_LAUNCH();
      cur = oth;
    }
    *moved = nb;
  } else {
    *moved = 0;
  }
  // remember the labels S now holds
  IVFKM_TRY(cudaMemcpyAsync(d.labels, labels, sizeof(int32_t) * n_obj, cudaMemcpyDeviceToDevice,
                            st));
  set_hdr_kernel<<<1, 1, 0, st>>>(d.hdr, DeltaHdr{kDeltaMagic, n_obj, nnz, k, dim, 1, cur, dim});
  IVFKM_CHECK_LAUNCH();
  *sk = d.key[cur];
  *sv = d.val[cur];
  return IVFKM_OK;
}

// Fused run detection: one CUB exclusive scan whose input is the head flag
// computed from the sorted keys on the fly and whose output, instead of
// being stored, writes the run start and key at every head (and the run
// count at the last entry) — no flag array, no position array, no extra pass.
template <class R>
struct HeadFlag {
  R key;
  __device__ __forceinline__ uint32_t operator()(int64_t e) const {
    return (e == 0 || key(e) != key(e - 1)) ? 1u : 0u;
  }
};

template <class K, class R>
struct RunStartOut {
  R key;
  uint32_t* seg_start;
  K* seg_key;
  uint32_t* n_seg;
  int64_t nnz;
  int64_t base = 0;
  struct Ref {
    R key;
    uint32_t* seg_start;
    K* seg_key;
    uint32_t* n_seg;
    int64_t nnz, e;
    __device__ __forceinline__ void operator=(uint32_t pos) const {
      const K k = key(e);
      const bool head = e == 0 || k != key(e - 1);
      if (head) {
        seg_start[pos] = (uint32_t)e;
        seg_key[pos] = k;
      }
      if (e == nnz - 1) {
        const uint32_t ns = pos + (head ? 1u : 0u);
        *n_seg = ns;
        seg_start[ns] = (uint32_t)nnz;
      }
    }
  };
  using iterator_category = std::random_access_iterator_tag;
  using value_type = uint32_t;
  using difference_type = int64_t;
  using pointer = void;
  using reference = Ref;
  __host__ __device__ RunStartOut operator+(int64_t d) const {
    RunStartOut o = *this;
    o.base += d;
    return o;
  }
  __device__ __forceinline__ Ref operator[](int64_t i) const {
    return Ref{key, seg_start, seg_key, n_seg, nnz, base + i};
  }
  __device__ __forceinline__ Ref operator*() const { return (*this)[0]; }
};

// Run heads, their scan and the run starts / keys / leaf-group starts.
template <class K, class R>
int runs_impl(int64_t nnz, R rd, const UpdWs<K>& w, int64_t dim, int64_t nleaf,
              const int32_t* plan, cudaStream_t st) {
  const int T = 256;
  {
    auto in = thrust::make_transform_iterator(thrust::counting_iterator<int64_t>(0),
                                              HeadFlag<R>{rd});
    RunStartOut<K, R> out{rd, w.seg_start, w.seg_key, w.n_seg, nnz, 0};
    size_t need = 0;
    IVFKM_TRY(cub::DeviceScan::ExclusiveSum(nullptr, need, in, out, (int)nnz, st));
    if (need <= w.cub_bytes) {
      size_t cb = w.cub_bytes;
      IVFKM_TRY(cub::DeviceScan::ExclusiveSum(w.cub, cb, in, out, (int)nnz, st));
    } else {
      head_kernel<K, R><<<grid_for(nnz, T), T, 0, st>>>(nnz, rd, w.head);
      IVFKM_CHECK_LAUNCH();
      size_t cb = w.cub_bytes;
      IVFKM_TRY(cub::DeviceScan::ExclusiveSum(w.cub, cb, w.head, w.segpos, (int)nnz, st));
      segstart_kernel<K, R><<<grid_for(nnz, T), T, 0, st>>>(
          nnz, rd, w.head, w.segpos, w.seg_start, w.seg_key, w.n_seg);
      IVFKM_CHECK_LAUNCH();
    }
  }
  return IVFKM_OK;
}

template <class K>
int update_count_impl(int64_t n_obj, const int64_t* row_ptr, const int32_t* terms,
                      const double* val64, int64_t nnz, int64_t k, int64_t dim,
                      const int32_t* labels, const unsigned long long* sizes,
                      const int64_t* prev_ptr, int64_t* new_ptr, void* ws, size_t ws_bytes,
                      DeltaState* delta, cudaStream_t st) {
  size_t need = 0;
  UpdWs<K> w = carve_upd<K>(ws, nnz, k, dim, &need);
  if (ws_bytes < need) return IVFKM_E_WORKSPACE;
  const int T = 256;
  const NormPlan& P = norm_plan(dim);
  const int64_t nleaf = P.nleaf, nint = P.nint;
  const size_t nsmem = (size_t)kNormWarps * kLeafG * 128 * 8 + (size_t)(nleaf + nint) * 8 +
                       (size_t)(nleaf + 1) * 4;
  if (nsmem > 200 * 1024) return IVFKM_E_UNSUPPORTED;  // D beyond ~1M terms
  // The plan lives in a process-lifetime cache.  It is uploaded from pageable
  // memory (a small copy the driver stages itself; a page-locked async copy
  // would queue behind a concurrent bulk upload on the copy engine), and
  // kept in the label-delta state across calls when there is one.
  const size_t plan_bytes = P.buf.size() * sizeof(int32_t);
  const int32_t* plan = w.plan;
  if (!(delta && nnz > 0))
    IVFKM_TRY(cudaMemcpyAsync(w.plan, P.buf.data(), plan_bytes, cudaMemcpyHostToDevice, st));
  if (nnz > 0) {
    const double* sval;
    if (delta) {
      const unsigned long long* ck;
      int64_t moved = 0;
      bool plan_ok = false;
      IVFKM_TRY_RC(delta_sort(n_obj, row_ptr, terms, val64, nnz, k, dim, labels, *delta, &ck,
                              &sval, &moved, &plan_ok, st));
      plan = delta->plan;
      if (!plan_ok)
        IVFKM_TRY(cudaMemcpyAsync(delta->plan, P.buf.data(), plan_bytes, cudaMemcpyHostToDevice,
                                  st));
      IVFKM_TRY_RC(runs_impl<K>(nnz, CompKey<K>{ck, comp_bits(n_obj, dim, k), dim}, w, dim,
                                nleaf, plan, st));
    } else {
      keys_kernel<K><<<grid_for(n_obj, T / 32), T, 0, st>>>(n_obj, row_ptr, terms, val64, labels,
                                                            dim, w.key_a, w.val_a);
      IVFKM_CHECK_LAUNCH();
      cub::DoubleBuffer<K> kb(w.key_a, w.key_b);
      cub::DoubleBuffer<double> vb(w.val_a, w.val_b);
      size_t cb = w.cub_bytes;
      IVFKM_TRY(cub::DeviceRadixSort::SortPairs(w.cub, cb, kb, vb, (int)nnz, 0, key_bits(k, dim),
                                                st));
      sval = vb.Current();
      IVFKM_TRY_RC(runs_impl<K>(nnz, ArrKey<K>{kb.Current()}, w, dim, nleaf, plan, st));
    }
    // the run count sizes the rest of the update (one 4-byte read-back)
    uint32_t n_seg = 0;
    IVFKM_TRY(cudaMemcpyAsync(&n_seg, w.n_seg, sizeof(n_seg), cudaMemcpyDeviceToHost, st));
    IVFKM_TRY(cudaStreamSynchronize(st));
    IVFKM_TRY(cudaMemsetAsync(w.n_seg + 1, 0, sizeof(uint32_t), st));
    // segpos is free again: it holds the long-run list
    {
      const int ng = (int)((nleaf + kLeafG - 1) / kLeafG);
      segsum_kernel<K><<<grid_for((int64_t)n_seg + 1, T), T, (size_t)(ng + (dim >> 8) + 1) * 4,
                         st>>>(n_seg, w.seg_start, w.seg_key, sval, sizes, k, dim, plan, nleaf,
                               w.seg_w, w.head, w.segpos, w.n_seg + 1, w.cl_seg, w.gstart);
      IVFKM_CHECK_LAUNCH();
    }
    segsum_long_kernel<K><<<num_sms() * 8, 256, 0, st>>>(w.seg_start, w.seg_key, sval, sizes, dim,
                                                      w.seg_w, w.head, w.segpos, w.n_seg + 1);
    IVFKM_CHECK_LAUNCH();
    size_t cb = w.cub_bytes;
    IVFKM_TRY(cub::DeviceScan::ExclusiveSum(w.cub, cb, w.head, w.nzpos, (int)n_seg + 1, st));
  } else {
    IVFKM_TRY(cudaMemsetAsync(w.n_seg, 0, sizeof(uint32_t), st));
    clseg_kernel<K><<<grid_for(k + 1, T), T, 0, st>>>(k, dim, w.n_seg, w.seg_key, w.cl_seg);
    IVFKM_CHECK_LAUNCH();
  }
  IVFKM_TRY(cudaFuncSetAttribute(norm_kernel<K>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)nsmem));
  norm_kernel<K><<<(int)std::min<int64_t>(k, num_sms() * 4), kNormWarps * 32, nsmem, st>>>(
      k, dim, nleaf, nint, P.nlevels, plan, sizes, prev_ptr, w.cl_seg, w.gstart, w.seg_key,
      w.seg_w, w.nzpos, w.nrm, w.counts);
  IVFKM_CHECK_LAUNCH();
  size_t cb = w.cub_bytes;
  IVFKM_TRY(cub::DeviceScan::ExclusiveSum(w.cub, cb, w.counts, new_ptr, (int)(k + 1), st));
  return IVFKM_OK;
}

template <class K>
int update_fill_impl(int64_t nnz, int64_t k, int64_t dim, const unsigned long long* sizes,
                     const int64_t* prev_ptr, const int32_t* prev_terms,
                     const double* prev_vals, const int64_t* new_ptr, int32_t* new_terms,
                     double* new_vals, uint8_t* retained, int64_t capacity, void* ws,
                     size_t ws_bytes, cudaStream_t st) {
  size_t need = 0;
  UpdWs<K> w = carve_upd<K>(ws, nnz, k, dim, &need);
  if (ws_bytes < need) return IVFKM_E_WORKSPACE;
  const int T = 256;
  if (nnz > 0) {
    fill_kernel<K><<<grid_for(nnz, T), T, 0, st>>>(nnz, dim, w.n_seg, w.seg_key, w.seg_w, w.head,
                                                   w.nzpos, w.cl_seg, w.nrm, new_ptr, new_terms,
                                                   new_vals, capacity);
    IVFKM_CHECK_LAUNCH();
  }
  retain_kernel<<<grid_for(k, T / 32), T, 0, st>>>(k, sizes, prev_ptr, prev_terms, prev_vals,
                                                   new_ptr, new_terms, new_vals, retained,
                                                   capacity);
  IVFKM_CHECK_LAUNCH();
  return IVFKM_OK;
}

}  // namespace

extern "C" size_t ivfkm_update_workspace_size(int64_t /*n_obj*/, int64_t nnz, int64_t k,
                                              int64_t dim) {
  size_t total = 0;
  if (use_k32(k, dim)) carve_upd<uint32_t>(nullptr, nnz, k, dim, &total);
  else carve_upd<unsigned long long>(nullptr, nnz, k, dim, &total);
  return total;
}

extern "C" int ivfkm_update_count(int64_t n_obj, int64_t nnz, const int64_t* row_ptr,
                                  const int32_t* terms,
                                  const double* val64, int64_t k, int64_t dim,
                                  const int32_t* labels, const unsigned long long* sizes,
                                  const int64_t* prev_ptr, int64_t* new_ptr, void* ws,
                                  size_t ws_bytes, ivfkm_stream_t stream_) {
  if (n_obj < 0 || k < 1 || dim < 1 || !row_ptr || !sizes || !prev_ptr || !new_ptr)
    return IVFKM_E_ARG;
  if (nnz < 0) return IVFKM_E_ARG;
  if (nnz >= (int64_t)INT32_MAX) return IVFKM_E_UNSUPPORTED;  // cub length / uint32 indices
  cudaStream_t st = as_stream(stream_);
  if (use_k32(k, dim))
    return update_count_impl<uint32_t>(n_obj, row_ptr, terms, val64, nnz, k, dim, labels, sizes,
                                       prev_ptr, new_ptr, ws, ws_bytes, nullptr, st);
  return update_count_impl<unsigned long long>(n_obj, row_ptr, terms, val64, nnz, k, dim, labels,
                                               sizes, prev_ptr, new_ptr, ws, ws_bytes, nullptr, st);
}

extern "C" int ivfkm_set_update_option(int which, int value) {
  switch (which) {
    case 1: g_delta_cub_merge = value ? 1 : 0; return IVFKM_OK;
    default: return IVFKM_E_ARG;
  }
}

extern "C" size_t ivfkm_update_state_size(int64_t n_obj, int64_t nnz, int64_t k, int64_t dim) {
  if (n_obj < 0 || nnz < 0 || k < 1 || dim < 1 || nnz >= (int64_t)INT32_MAX) return 0;
  const Bits bt = comp_bits(n_obj, dim, k);
  if (bt.ob + bt.tb + bt.lb > 64) return 0;
  size_t total = 0;
  carve_delta(nullptr, n_obj, nnz, dim, &total);
  return total;
}

extern "C" int ivfkm_update_count_delta(int64_t n_obj, int64_t nnz, const int64_t* row_ptr,
                                        const int32_t* terms, const double* val64, int64_t k,
                                        int64_t dim, const int32_t* labels,
                                        const unsigned long long* sizes, const int64_t* prev_ptr,
                                        int64_t* new_ptr, void* ws, size_t ws_bytes, void* state,
                                        size_t state_bytes, ivfkm_stream_t stream_) {
  if (n_obj < 0 || k < 1 || dim < 1 || !row_ptr || !sizes || !prev_ptr || !new_ptr || !state)
    return IVFKM_E_ARG;
  if (nnz < 0) return IVFKM_E_ARG;
  const size_t need = ivfkm_update_state_size(n_obj, nnz, k, dim);
  if (need == 0) return IVFKM_E_UNSUPPORTED;
  if (state_bytes < need) return IVFKM_E_WORKSPACE;
  DeltaState d = carve_delta(state, n_obj, nnz, dim, nullptr);
  cudaStream_t st = as_stream(stream_);
  if (use_k32(k, dim))
    return update_count_impl<uint32_t>(n_obj, row_ptr, terms, val64, nnz, k, dim, labels, sizes,
                                       prev_ptr, new_ptr, ws, ws_bytes, &d, st);
  return update_count_impl<unsigned long long>(n_obj, row_ptr, terms, val64, nnz, k, dim, labels,
                                               sizes, prev_ptr, new_ptr, ws, ws_bytes, &d, st);
}

extern "C" int ivfkm_update_fill(int64_t /*n_obj*/, int64_t nnz, int64_t k, int64_t dim,
                                 const unsigned long long* sizes, const int64_t* prev_ptr,
                                 const int32_t* prev_terms, const double* prev_vals,
                                 const int64_t* new_ptr, int32_t* new_terms, double* new_vals,
                                 uint8_t* retained, int64_t capacity, void* ws, size_t ws_bytes,
                                 ivfkm_stream_t stream_) {
  if (k < 1 || dim < 1 || !new_ptr || !retained || capacity < 0) return IVFKM_E_ARG;
  if (capacity > 0 && (!new_terms || !new_vals)) return IVFKM_E_ARG;
  cudaStream_t st = as_stream(stream_);
  if (use_k32(k, dim))
    return update_fill_impl<uint32_t>(nnz, k, dim, sizes, prev_ptr, prev_terms, prev_vals, new_ptr,
                                      new_terms, new_vals, retained, capacity, ws, ws_bytes, st);
  return update_fill_impl<unsigned long long>(nnz, k, dim, sizes, prev_ptr, prev_terms, prev_vals,
                                              new_ptr, new_terms, new_vals, retained, capacity, ws,
                                              ws_bytes, st);
}
