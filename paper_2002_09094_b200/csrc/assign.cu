// Assignment step of IVF spherical k-means on sm_100a.
//
// Reference semantics (file:line under /root/reference/pkg/src/sparse_kmeans):
//   _kernels.pyx:106-128  for each object i: rho[0..k) = 0; for each nonzero
//                         (t, v) in row order, for each mean posting (c, u) of
//                         term t: rho[c] += v * u  (float64, mul then add);
//   _kernels.pyx:17-26    label = argmax, strict '>' from -inf, so the
//                         smallest index among maximizers wins;
//   clustering.py:105-119 objective = fsum_i sum_h v_h * mu_{a(i)}[t_h]
//                         (= rho_i[a(i)] bit for bit: same products, same order);
//   clustering.py:286     convergence = labels unchanged;
//   variants.py:56-59     sizes = bincount(labels).
//
// B200 design:
//   1. screen (fp32, registers): one CTA (or a thread-block cluster of CTAs
//      when k outgrows one SM's shared memory) per object.  Lane `l` of a warp
//      owns means 32*b + l of RR consecutive 32-mean blocks b and accumulates
//      rho in registers: for each object nonzero the warp loads the RR block
//      headers of the term (one coalesced 8*RR-byte load), and each lane whose
//      mask bit is set loads its value at offset + popc(mask below the lane).
//      No shared-memory scatter, no bank conflicts, no atomics, fixed FMA order.
//      Finished spans are parked in shared memory (cluster: distributed
//      shared memory) for the block argmax.
//   2. window: |rho32 - rho64| <= eps_i is a rigorous bound (n_i+3 roundings
//      of size 2^-24 on a sum bounded by |x_i| * max|mu|), so the reference
//      winner is within 2*eps_i of the fp32 max.  A single candidate is
//      certified; several are queued for exact rescoring.
//   3. finalize (fp64, one warp per object): rescore the candidates (or the
//      certified winner, whose similarity is the objective summand) with
//      __dmul_rn/__dadd_rn in the reference's h order — bit-identical to the
//      reference's float64 rho — pick the max with the smallest index.
//   4. accumulate: changed labels, sizes, and the exact objective (a
//      fixed-point superaccumulator, so the host can round the exact sum once,
//      like math.fsum).
#include <cooperative_groups.h>
#include <cuda_fp16.h>

#include <cub/cub.cuh>
#include <map>
#include <mutex>
#include <utility>

#include <cfloat>
#include <climits>
#include <cmath>

#include "bivf.cuh"
#include "common.cuh"

namespace cg = cooperative_groups;
using namespace ivfkm;

namespace {

constexpr int kMaxC = IVFKM_MAXC;
constexpr int kLimbs = IVFKM_OBJ_LIMBS;
constexpr int kMaxSplit = 8;           // portable cluster size
constexpr int kSmemLimit = 227 * 1024;  // opt-in dynamic shared memory per CTA
constexpr int kMaxLocalSpans = 63;      // dense-prefix buckets per CTA (screen_kernel)
constexpr int kMaxChunks = 32;          // 32-entry chunks per staged row piece (rowcap 1024)
constexpr int kEntryBytes = 20;         // screen_kernel staging per row entry

struct ScreenParams {
  int64_t n_obj;
  const int64_t* row_ptr;
  const int32_t* terms;
  const float* val32;
  const double* xnorm;
  int64_t k;
  int64_t nblk;
  const uint32_t* masks;  // [dim][nblk]
  const uint32_t* offs;   // [dim][nblk] (+1: total)
  const uint32_t* nc;     // [dim] postings per term
  const uint32_t* dpre;   // [dim] dense prefix spans per term
  const uint2* tinfo;     // [dim] {dense-run start, dense prefix} (bivf.cuh)
  int count_post = 1;     // 0: the postings counter comes from doc_freq . nc (screen_impl)
  const int32_t* inv;     // [k] slot -> mean
  const int32_t* order;   // [n] processing order of objects, or nullptr
  const uint8_t* slot8 = nullptr;  // sparse spans' slot bytes (ivfkm_bivf_slots), or nullptr
  const uint32_t* soff = nullptr;  // with slot8: compact span offsets [dim][nsp1] (bivf.cuh)
  int nsp1 = 0;                    // spans per term + 1
  // rows presorted by dense prefix (presort_rows_kernel), per entry {term,
  // dense prefix} and {dense-run start, fp32 value bits}; or nullptr: the CTA
  // sorts its staged row itself
  const int2* ps_t = nullptr;
  const int2* ps_v = nullptr;
  const float* pv32;  // fp32 screen values, or fp16 ones when half
  int half;
  double mu_max;
  int cta_blocks;  // 32-mean blocks held by one CTA (multiple of RR)
  int nsplit;      // CTAs per object (cluster size)
  int pass = -1;   // >= 0: slot-range pass `pass` of npass (one CTA per object)
  int npass = 0;
  float* st_best;  // pass state per object: best screen value so far,
  int32_t* st_slot;  // its slot,
  int32_t* st_cnt;   // candidates kept (kMaxC + 1: overflow) | kHasPost,
  int2* st_cand;     // [n][kMaxC] the candidates (slot, fp32 value bits)
  int rowcap;      // row entries staged in shared memory per pass
  int cc_bytes = 0;  // counting-sort scratch after the staged row (0: presorted rows)
  int32_t* label32;
  int32_t* slot_of;
  int32_t* q_obj;
  int32_t* q_cnt;
  int32_t* q_cid;
  ivfkm_stats* stats;
};

struct ScreenShared {
  float red_v[32];
  int red_c[32];
  unsigned long long red_p[32];
  float best_v;
  int best_c;
  int cnt;
  int cand[kMaxC];
  float cval[kMaxC];  // pass mode: the candidates' screen values
  unsigned long long post;
  float pv;  // pass mode: state of the earlier passes
  int pc, pn;
};

constexpr int kHasPost = 1 << 30;  // pass state: the object touches some posting
constexpr int kCntMask = kHasPost - 1;

__device__ __forceinline__ void better(float& bv, int& bc, float ov, int oc) {
  if (ov > bv || (ov == bv && oc < bc)) {
    bv = ov;
    bc = oc;
  }
}

// Masks of RR consecutive blocks of one term, loaded with vector loads (every
// lane reads the same address: one broadcast wavefront).
template <int RR>
struct MaskPack {
  uint32_t m[RR];
  __device__ __forceinline__ void load(const uint32_t* __restrict__ src) {
    if constexpr (RR % 4 == 0) {
#pragma unroll
      for (int q = 0; q < RR / 4; ++q) {
        const uint4 v = __ldg(reinterpret_cast<const uint4*>(src) + q);
        m[4 * q] = v.x;
        m[4 * q + 1] = v.y;
        m[4 * q + 2] = v.z;
        m[4 * q + 3] = v.w;
      }
    } else {
#pragma unroll
      for (int q = 0; q < RR / 2; ++q) {
        const uint2 v = __ldg(reinterpret_cast<const uint2*>(src) + q);
        m[2 * q] = v.x;
        m[2 * q + 1] = v.y;
      }
    }
  }
  __device__ __forceinline__ void zero() {
#pragma unroll
    for (int r = 0; r < RR; ++r) m[r] = 0u;
  }
};

// One object nonzero against RR blocks starting at block gb: lane-owned mean
// 32*(gb+r)+lane reads its value at o_r + popc(mask_r below the lane), with
// o_{r+1} = o_r + popc(mask_r); in a dense span (kDense on the offset) the
// lane's values sit at span_base + 128*(r/4) + 4*lane + r%4 (bivf.cuh).
template <int RR>
__device__ __forceinline__ bool gather_values(const MaskPack<RR>& mk, uint32_t o, uint32_t gb,
                                              const float* __restrict__ pv, unsigned lane,
                                              unsigned lanebit, unsigned lt, float (&u)[RR]) {
  if (o & kDense) {
    const uint32_t r0 = gb & (kSpan - 1);
    const uint32_t sbase = (o & ~kDense) - 32u * r0;
    if constexpr (RR == kSpan) {  // r0 == 0: two aligned 16-B loads
      const float4 a = __ldg(reinterpret_cast<const float4*>(pv + sbase) + lane);
      const float4 b = __ldg(reinterpret_cast<const float4*>(pv + sbase) + 32 + lane);
      u[0] = a.x; u[1] = a.y; u[2] = a.z; u[3] = a.w;
      u[4] = b.x; u[5] = b.y; u[6] = b.z; u[7] = b.w;
    } else {
#pragma unroll
      for (int r = 0; r < RR; ++r) {
        const uint32_t rr = r0 + r;
        u[r] = __ldg(pv + sbase + 128u * (rr >> 2) + 4u * lane + (rr & 3u));
      }
    }
    return true;
  }
  uint32_t any = 0;
#pragma unroll
  for (int r = 0; r < RR; ++r) any |= mk.m[r];
  if (!any) return false;  // the term populates none of these blocks
#pragma unroll
  for (int r = 0; r < RR; ++r) {
    const uint32_t mr = mk.m[r];
    u[r] = 0.f;
    if (mr & lanebit) u[r] = __ldg(pv + (o + (uint32_t)__popc(mr & lt)));
    o += (uint32_t)__popc(mr);
  }
  return true;
}

// fp16 screen values (bivf.cuh, bivf_find16_slot): a dense span holds each
// lane's 8 values contiguously, so one 16-B load serves the whole span.  The
// raw bits stay packed in registers until the FMAs: converting right after
// the load would make the warp wait for it and defeat the software pipeline.
// Returns 0 (term absent from these blocks), 1 (w[r] = one value's bits per
// block) or 2 (w[0..RR/2) = packed pairs).
template <int RR>
__device__ __forceinline__ int gather_values16(const MaskPack<RR>& mk, uint32_t o, uint32_t gb,
                                               const __half* __restrict__ pv, unsigned lane,
                                               unsigned lanebit, unsigned lt, uint32_t (&w)[RR]) {
  const unsigned short* __restrict__ p16 = reinterpret_cast<const unsigned short*>(pv);
  if (o & kDense) {
    const uint32_t r0 = gb & (kSpan - 1);
    const uint32_t sbase = (o & ~kDense) - 32u * r0;
    if constexpr (RR == kSpan) {
      const uint4 a = __ldg(reinterpret_cast<const uint4*>(pv + sbase) + lane);
      w[0] = a.x; w[1] = a.y; w[2] = a.z; w[3] = a.w;
      return 2;
    } else {
#pragma unroll
      for (int r = 0; r < RR; ++r) w[r] = __ldg(p16 + sbase + 8u * lane + r0 + r);
      return 1;
    }
  }
  uint32_t any = 0;
#pragma unroll
  for (int r = 0; r < RR; ++r) any |= mk.m[r];
  if (!any) return 0;
#pragma unroll
  for (int r = 0; r < RR; ++r) {
    const uint32_t mr = mk.m[r];
    w[r] = 0u;
    if (mr & lanebit) w[r] = __ldg(p16 + (o + (uint32_t)__popc(mr & lt)));
    o += (uint32_t)__popc(mr);
  }
  return 1;
}

// The screen's in-flight values of one (entry, span): fp32 values, or fp16 bits.
template <int RR, bool HALF, bool F2 = false>
struct SpanVals;

template <int RR>
struct SpanVals<RR, false, false> {
  float u[RR];
  bool has;
  __device__ __forceinline__ void gather(const MaskPack<RR>& mk, uint32_t o, uint32_t gb,
                                         const void* pv, unsigned lane, unsigned lanebit,
                                         unsigned lt) {
    has = gather_values<RR>(mk, o, gb, static_cast<const float*>(pv), lane, lanebit, lt, u);
  }
  // Lane's first dense value of a span in bytes from the array start, given the
  // span's first value index sbase: slot 32*(b0+r)+lane at sbase + 128*(r/4) +
  // 4*lane + r%4 for blocks r = r0 .. r0+RR-1 (bivf.cuh).
  static __device__ __forceinline__ uint32_t lane_bytes(uint32_t sbase, uint32_t r0,
                                                        unsigned lane) {
    return 4u * (sbase + 128u * (r0 >> 2) + 4u * lane + (r0 & 3u));
  }
  __device__ __forceinline__ void load_dense(const char* at) {
    has = true;
    if constexpr (RR == 8) {
      const float4 a = __ldg(reinterpret_cast<const float4*>(at));
      const float4 b = __ldg(reinterpret_cast<const float4*>(at + 512));
      u[0] = a.x; u[1] = a.y; u[2] = a.z; u[3] = a.w;
      u[4] = b.x; u[5] = b.y; u[6] = b.z; u[7] = b.w;
    } else if constexpr (RR == 4) {
      const float4 a = __ldg(reinterpret_cast<const float4*>(at));
      u[0] = a.x; u[1] = a.y; u[2] = a.z; u[3] = a.w;
    } else {
      const float2 a = __ldg(reinterpret_cast<const float2*>(at));
      u[0] = a.x; u[1] = a.y;
    }
  }
  static constexpr uint32_t kElem = 4;
  __device__ __forceinline__ void fma(float v, float (&acc)[RR]) const {
    // fma(v, 0, acc) == acc exactly: absent postings cost no rounding;
    // a span the term does not populate skips the FMAs altogether
    if (has) {
#pragma unroll
      for (int r = 0; r < RR; ++r) acc[r] = fmaf(v, u[r], acc[r]);
    }
  }
  // the entry's value is read only when the span holds postings
  __device__ __forceinline__ void fma(const int* vbits, float (&acc)[RR]) const {
    if (has) {
      const float v = __int_as_float(*vbits);
#pragma unroll
      for (int r = 0; r < RR; ++r) acc[r] = fmaf(v, u[r], acc[r]);
    }
  }
};

// F2: packed FFMA2 (faster in the 56-register small-CTA screen; the
// 64-register instantiations lose more to register pairing than they gain)
template <int RR, bool F2>
struct SpanVals<RR, true, F2> {
  uint32_t w[RR];
  int code;
  __device__ __forceinline__ void gather(const MaskPack<RR>& mk, uint32_t o, uint32_t gb,
                                         const void* pv, unsigned lane, unsigned lanebit,
                                         unsigned lt) {
    code = gather_values16<RR>(mk, o, gb, static_cast<const __half*>(pv), lane, lanebit, lt, w);
  }
  // lane's RR contiguous halves of a dense span: sbase + 8*lane + r0 (bivf.cuh)
  static __device__ __forceinline__ uint32_t lane_bytes(uint32_t sbase, uint32_t r0,
                                                        unsigned lane) {
    return 2u * (sbase + 8u * lane + r0);
  }
  __device__ __forceinline__ void load_dense(const char* at) {
    code = 2;
    if constexpr (RR == 8) {
      const uint4 a = __ldg(reinterpret_cast<const uint4*>(at));
      w[0] = a.x; w[1] = a.y; w[2] = a.z; w[3] = a.w;
    } else if constexpr (RR == 4) {
      const uint2 a = __ldg(reinterpret_cast<const uint2*>(at));
      w[0] = a.x; w[1] = a.y;
    } else {
      w[0] = __ldg(reinterpret_cast<const unsigned int*>(at));
    }
  }
  static constexpr uint32_t kElem = 2;
  __device__ __forceinline__ void fma(const int* vbits, float (&acc)[RR]) const {
    if (code != 0) fma(__int_as_float(*vbits), acc);
  }
  // packed fp32 FMA (FFMA2): two slots per instruction, each lane of the pair
  // rounded exactly as fmaf
  static __device__ __forceinline__ void fma2(float v, float a, float b, float& x, float& y) {
    unsigned long long ab, xy;
    asm("mov.b64 %0, {%1, %2};" : "=l"(ab) : "f"(a), "f"(b));
    asm("mov.b64 %0, {%1, %2};" : "=l"(xy) : "f"(x), "f"(y));
    unsigned long long vv;
    asm("mov.b64 %0, {%1, %1};" : "=l"(vv) : "f"(v));
    asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(xy) : "l"(vv), "l"(ab));
    asm("mov.b64 {%0, %1}, %2;" : "=f"(x), "=f"(y) : "l"(xy));
  }
  __device__ __forceinline__ void fma(float v, float (&acc)[RR]) const {
    if (code == 2) {
#pragma unroll
      for (int q = 0; q < RR / 2; ++q) {
        const float2 f = __half22float2(*reinterpret_cast<const __half2*>(&w[q]));
        if constexpr (F2) {
          fma2(v, f.x, f.y, acc[2 * q], acc[2 * q + 1]);
        } else {
          acc[2 * q] = fmaf(v, f.x, acc[2 * q]);
          acc[2 * q + 1] = fmaf(v, f.y, acc[2 * q + 1]);
        }
      }
    } else if (code == 1) {
      if constexpr (F2) {
#pragma unroll
        for (int q = 0; q < RR / 2; ++q)
          fma2(v, __half2float(__ushort_as_half((unsigned short)w[2 * q])),
               __half2float(__ushort_as_half((unsigned short)w[2 * q + 1])), acc[2 * q],
               acc[2 * q + 1]);
      } else {
#pragma unroll
        for (int r = 0; r < RR; ++r)
          acc[r] = fmaf(v, __half2float(__ushort_as_half((unsigned short)w[r])), acc[r]);
      }
    }
  }
};

// Half-width of the rigorous screen window of an object with n_i entries
// (DESIGN.md §3): |rho_screen - rho_f64| <= eps for every mean.
__device__ __forceinline__ double window_eps(const ScreenParams& p, int64_t obj, int64_t n_i) {
  const double xn = p.xnorm ? p.xnorm[obj] : 1.0;
  // fp16 screen values add a relative 2^-11 rounding per mean value plus an
  // absolute 2^-25 below fp16's normal range (sum over h of |x_h| <= n*|x|)
  // (n_i + 5): the sparse spans' products are summed apart and folded in
  // with one more rounding (screen_kernel)
  return p.half ? (0x1p-11 + (double)(n_i + 5) * 0x1p-24) * xn * p.mu_max * (1.0 + 0x1p-9) +
                      (double)n_i * xn * 0x1p-25 * (1.0 + 0x1p-9) + (double)(n_i + 1) * 0x1p-125
                : ((double)(n_i + 3) * 0x1p-24 + (double)n_i * 0x1p-50) * xn * p.mu_max *
                          (1.0 + 1e-6) +
                      (double)(n_i + 1) * 0x1p-125;
}

// Slot-range pass epilogue: merge this pass's slots into the object's running
// state — the best screen value so far and every slot within 2*eps of it.  A
// slot kept at pass z satisfies rho >= best_z - 2 eps >= best_final - 2 eps,
// and candidates are re-filtered against each new best, so after the last
// pass the set is exactly the one-pass window (an overflow stays one: its
// dropped values are unknown, and the overflow kernel rescores every mean).
__device__ void pass_epilogue(const ScreenParams& p, ScreenShared& sh, const float* rho,
                              int64_t obj, int z, int64_t n_i, float gv, int gc,
                              unsigned long long gpost) {
  const int cta_cids = p.cta_blocks * 32;
  const int64_t cid0 = (int64_t)z * cta_cids;
  // (sh.pv/pc/pn were loaded at the kernel's start, pass_state_prefetch)
  if (threadIdx.x == 0) {
    if (z == 0) sh.pn = gpost ? kHasPost : 0;
    sh.cnt = 0;
  }
  __syncthreads();
  float bv = sh.pv;
  int bc = sh.pc;
  better(bv, bc, gv, gc);
  const int pn = sh.pn;
  const bool has = (pn & kHasPost) != 0;
  const int prev = pn & kCntMask;
  if (has) {
    const double thr = (double)bv - 2.0 * window_eps(p, obj, n_i);
    const int2* pc = p.st_cand + obj * kMaxC;
    // after an overflow the stored candidates are incomplete: not read
    for (int j = threadIdx.x; j < (prev <= kMaxC ? prev : 0); j += blockDim.x) {
      const int2 c = pc[j];
      const float v = __int_as_float(c.y);
      if ((double)v >= thr) {
        const int s = atomicAdd(&sh.cnt, 1);
        if (s < kMaxC) {
          sh.cand[s] = c.x;
          sh.cval[s] = v;
        }
      }
    }
    for (int j = threadIdx.x; j < cta_cids; j += blockDim.x) {
      const int64_t cid = cid0 + j;
      if (cid >= p.k) break;
      const float v = rho[j];
      if ((double)v >= thr) {
        const int s = atomicAdd(&sh.cnt, 1);
        if (s < kMaxC) {
          sh.cand[s] = (int)cid;
          sh.cval[s] = v;
        }
      }
    }
  }
  __syncthreads();
  const int got = sh.cnt;
  const int stored = got < kMaxC ? got : kMaxC;  // valid entries of sh.cand
  int total = got;
  if (prev > kMaxC && total <= kMaxC) total = kMaxC + 1;  // an overflow stays one
  if (z < p.npass - 1) {
    if (threadIdx.x == 0) {
      p.st_best[obj] = bv;
      p.st_slot[obj] = bc;
      p.st_cnt[obj] = (total < kMaxC + 1 ? total : kMaxC + 1) | (has ? kHasPost : 0);
    }
    for (int j = threadIdx.x; j < stored; j += blockDim.x)
      p.st_cand[obj * kMaxC + j] = make_int2(sh.cand[j], __float_as_int(sh.cval[j]));
    return;
  }
  if (threadIdx.x == 0) {
    p.label32[obj] = has ? __ldg(p.inv + bc) : 0;
    if (total <= 1) {
      p.slot_of[obj] = -1;
    } else {
      const int slot = (int)atomicAdd(&p.stats->queue_len, 1ull);
      atomicAdd(&p.stats->near_ties, 1ull);
      if (total > kMaxC) atomicAdd(&p.stats->overflow, 1ull);
      p.slot_of[obj] = slot;
      p.q_obj[slot] = (int)obj;
      p.q_cnt[slot] = total;
      for (int j = 0; j < stored; ++j)
        p.q_cid[(int64_t)slot * kMaxC + j] = __ldg(p.inv + sh.cand[j]);
    }
  }
}

// Two adjacent words at any 4-byte alignment.
__device__ __forceinline__ uint2 ldg_u2(const uint32_t* at) {
  return make_uint2(__ldg(at), __ldg(at + 1));
}

// Byte offset of a dense run's value index: 32-bit for fp16 values (indices
// stay below 2^31, bivf.cu), 64-bit for fp32 ones (4 B x 2^30+ values pass 2^32).
template <bool HALF>
__device__ __forceinline__ size_t dense_off(int x) {
  if constexpr (HALF) return (size_t)(2u * (uint32_t)x);
  else return (size_t)4 * (uint32_t)x;
}

// CTA-local argmax (value desc, index asc) over the parked rho, merged over
// the cluster through DSMEM when k is split; then the rigorous fp32 window and
// the candidate queue for exact rescoring.  Every thread of the CTA calls it.
__device__ __forceinline__ void screen_epilogue(const ScreenParams& p, ScreenShared& sh,
                                                const float* rho, int64_t obj, int z, int64_t rb,
                                                int64_t re, unsigned long long post) {
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const int nwarps = blockDim.x >> 5;
  const int cta_cids = p.cta_blocks * 32;
  const int64_t blk0 = (int64_t)z * p.cta_blocks;
  float bv = -INFINITY;
  int bc = INT_MAX;
  const int64_t cid0 = blk0 * 32;
  for (int j = threadIdx.x; j < cta_cids; j += blockDim.x) {
    const int64_t cid = cid0 + j;
    if (cid >= p.k) break;
    const float v = rho[j];
    if (v > bv) {
      bv = v;
      bc = (int)cid;
    }
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    const float ov = __shfl_xor_sync(kFull, bv, off);
    const int oc = __shfl_xor_sync(kFull, bc, off);
    better(bv, bc, ov, oc);
    post += __shfl_xor_sync(kFull, post, off);
  }
  if (lane == 0) {
    sh.red_v[warp] = bv;
    sh.red_c[warp] = bc;
    sh.red_p[warp] = post;
  }
  __syncthreads();
  if (warp == 0) {
    float v = lane < nwarps ? sh.red_v[lane] : -INFINITY;
    int c = lane < nwarps ? sh.red_c[lane] : INT_MAX;
    unsigned long long q = lane < nwarps ? sh.red_p[lane] : 0ull;
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
      better(v, c, __shfl_xor_sync(kFull, v, off), __shfl_xor_sync(kFull, c, off));
      q += __shfl_xor_sync(kFull, q, off);
    }
    if (lane == 0) {
      sh.best_v = v;
      sh.best_c = c;
      sh.post = q;
      sh.cnt = 0;
      if (q && p.count_post) atomicAdd(&p.stats->postings, q);
    }
  }

  cg::cluster_group cluster = cg::this_cluster();
  const bool clus = p.nsplit > 1 && p.pass < 0;
  float gv;
  int gc;
  unsigned long long gpost;
  if (clus) {
    cluster.sync();
    gv = -INFINITY;
    gc = INT_MAX;
    gpost = 0;
    for (int q = 0; q < p.nsplit; ++q) {
      const ScreenShared* o = cluster.map_shared_rank(&sh, q);
      better(gv, gc, o->best_v, o->best_c);
      gpost += o->post;
    }
  } else {
    __syncthreads();
    gv = sh.best_v;
    gc = sh.best_c;
    gpost = sh.post;
  }
  if (p.pass >= 0) {
    pass_epilogue(p, sh, rho, obj, z, re - rb, gv, gc, gpost);
    return;
  }

  // ---- rigorous fp32 window and candidate collection ----
  const double thr = (double)gv - 2.0 * window_eps(p, obj, re - rb);
  if (gpost != 0) {
    for (int j = threadIdx.x; j < cta_cids; j += blockDim.x) {
      const int64_t cid = cid0 + j;
      if (cid >= p.k) break;
      if ((double)rho[j] >= thr) {
        const int s = atomicAdd(&sh.cnt, 1);
        if (s < kMaxC) sh.cand[s] = (int)cid;
      }
    }
  }
  if (clus) cluster.sync(); else __syncthreads();

  if (z == 0 && threadIdx.x == 0) {
    int total = 0;
    if (clus) {
      for (int q = 0; q < p.nsplit; ++q) total += cluster.map_shared_rank(&sh, q)->cnt;
    } else {
      total = sh.cnt;
    }
    // gpost == 0: no posting touched, every rho is exactly 0 -> label 0.
    // (slots map back to mean ids here; exact ties are always in the window)
    const int label = gpost == 0 ? 0 : __ldg(p.inv + gc);
    p.label32[obj] = label;
    if (total <= 1) {
      p.slot_of[obj] = -1;
    } else {
      const int slot = (int)atomicAdd(&p.stats->queue_len, 1ull);
      atomicAdd(&p.stats->near_ties, 1ull);
      if (total > kMaxC) atomicAdd(&p.stats->overflow, 1ull);
      p.slot_of[obj] = slot;
      p.q_obj[slot] = (int)obj;
      p.q_cnt[slot] = total;
      int w = 0;
      for (int q = 0; q < p.nsplit && w < kMaxC; ++q) {
        const ScreenShared* o = p.nsplit > 1 ? cluster.map_shared_rank(&sh, q) : &sh;
        const int cq = min(o->cnt, kMaxC);
        for (int j = 0; j < cq && w < kMaxC; ++j)
          p.q_cid[(int64_t)slot * kMaxC + w++] = __ldg(p.inv + o->cand[j]);
      }
    }
  }
  if (clus) cluster.sync();  // peers keep their shared memory alive
}

// MAXREG: 64 in general; 56 for small CTAs (<= 4 warps, k <= ~1000), where it
// lifts residency from 8 to 9 CTAs per SM (measured +2% at config 1; larger
// CTAs gain no residency and lose to the spills)
template <int RR, bool HALF, int MAXREG = 64>
__global__ void __maxnreg__(MAXREG) screen_kernel(ScreenParams p) {
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ ScreenShared sh;
  float* rho = reinterpret_cast<float*>(smem);
  const int cta_cids = p.cta_blocks * 32;
  // staged row entries {header row t*nblk, value, dense-run start, value},
  // sorted by dense prefix; then each entry's position and local prefix
  int4* s_ent = reinterpret_cast<int4*>(rho + cta_cids);
  uint16_t* s_pos = reinterpret_cast<uint16_t*>(s_ent + p.rowcap);
  uint8_t* s_lp = reinterpret_cast<uint8_t*>(s_pos + p.rowcap);
  // slot-byte sparse path: a 256-slot scratch per warp (zero between spans)
  // [chunk][bucket] counts of the in-CTA counting sort (absent when the rows
  // arrive presorted: the shared-memory footprint decides the L1 carve-out)
  uint16_t* s_cc = reinterpret_cast<uint16_t*>(s_lp + ((p.rowcap + 15) & ~15));
  float* s_scr = reinterpret_cast<float*>(reinterpret_cast<unsigned char*>(s_cc) + p.cc_bytes);

  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const int nwarps = blockDim.x >> 5;
  const int ctas = p.pass >= 0 ? 1 : p.nsplit;
  const int z = p.pass >= 0 ? p.pass : blockIdx.x % p.nsplit;
  const int64_t obj = p.order ? (int64_t)__ldg(p.order + blockIdx.x / ctas)
                              : (int64_t)(blockIdx.x / ctas);
  if (obj >= p.n_obj) return;  // whole cluster shares obj
  const int64_t rb = p.row_ptr[obj], re = p.row_ptr[obj + 1];
  const int64_t nblk = p.nblk;
  const int64_t blk0 = (int64_t)z * p.cta_blocks;
  const int nspans = p.cta_blocks / RR;
  const unsigned lanebit = 1u << lane;
  const unsigned lt = lanebit - 1u;
  // The bases go through shared memory so they stay in registers: ptxas would
  // otherwise re-load kernel parameters from the constant bank inside every
  // predicated gather (one extra LDC per posting block).
  __shared__ const void* s_base[3];
  if (HALF && RR == 8 && p.slot8) {
    for (int q = threadIdx.x; q < (int)(blockDim.x >> 5) * 256; q += blockDim.x) s_scr[q] = 0.f;
  }
  if (threadIdx.x == 0) {
    s_base[0] = p.masks;
    s_base[1] = p.offs;
    s_base[2] = p.pv32;
    if (p.pass > 0) {  // the earlier passes' state, read long before the epilogue
      sh.pv = p.st_best[obj];
      sh.pc = p.st_slot[obj];
      sh.pn = p.st_cnt[obj];
    } else {
      sh.pv = -INFINITY;
      sh.pc = INT_MAX;
      sh.pn = 0;
    }
  }
  __syncthreads();
  const bool sparse8 = HALF && RR == 8 && p.slot8 != nullptr;
  const uint32_t* __restrict__ masks = static_cast<const uint32_t*>(s_base[0]);
  const uint32_t* __restrict__ offs = static_cast<const uint32_t*>(s_base[1]);
  const void* pv = s_base[2];
  unsigned long long post = 0;  // postings of this CTA's blocks (counters.py:71-81)

  // BIVF spans this CTA touches: gs0 .. gs0+nls-1 (bivf.cuh: 8 blocks each)
  const int gs0 = (int)(blk0 >> 3);
  int nls = (int)(((blk0 + p.cta_blocks - 1) >> 3) - gs0 + 1);
  if (nls > kMaxLocalSpans) nls = kMaxLocalSpans;  // later local spans: masked path
  const int nb = nls + 1;                           // prefix buckets 0..nls
  __shared__ int s_cntd[kMaxLocalSpans + 1];  // entries whose prefix covers local span s
  __shared__ int s_next;                      // next span to process (dynamic)
  int64_t c0 = rb;
  do {
    const int64_t rem = re - c0;
    const int cn = (int)(rem < p.rowcap ? rem : p.rowcap);
    const int nch = (cn + 31) >> 5;
    if (p.ps_t) {
      // The row arrives sorted by dense prefix, descending (ivfkm_presort_rows):
      // every pass's clamped bucket order is the same order, so staging is a
      // copy, and bucket b starts where the (non-increasing) buckets drop to b.
      __syncthreads();
      if (threadIdx.x == 0) s_next = 0;
      // (the entry's dense prefix and run start were looked up once, by the
      // presort: no dependent gathers between the row's load and its spans)
      for (int j = threadIdx.x; j < cn; j += blockDim.x) {
        const int2 td = __ldg(p.ps_t + c0 + j);
        const int2 bv = __ldg(p.ps_v + c0 + j);
        int lp = (td.y & 0x7fffffff) - gs0;
        lp = lp < 0 ? 0 : (lp > nls ? nls : lp);
        // the postings counter, or (counted from doc_freq) whether any exist
        if (z == 0) post += p.count_post ? __ldg(p.nc + td.x) : ((uint32_t)td.y >> 31);
        // staged row word: the term's row of the block headers, or — when the
        // sparse spans go through slot bytes — of the span offsets table
        const uint32_t row = (uint32_t)td.x * (sparse8 ? (uint32_t)p.nsp1 : (uint32_t)nblk);
        s_ent[j] = make_int4((int)row, bv.y, lp ? bv.x : 0, bv.y);
        s_lp[j] = (uint8_t)lp;
      }
      __syncthreads();
      for (int b = threadIdx.x; b < nb; b += blockDim.x) {  // first j with lp <= b
        int lo = 0, hi = cn;
        while (lo < hi) {
          const int mid = (lo + hi) >> 1;
          if ((int)s_lp[mid] > b) lo = mid + 1; else hi = mid;
        }
        s_cntd[b] = lo;  // = entries with a longer prefix than b
      }
      __syncthreads();
    } else {
      __syncthreads();
      // Stage the row chunk sorted by the terms' dense prefix (bivf.cuh, dpre),
      // longest first, stable: for local span s the entries [0, cntd[s]) read
      // span s as one contiguous 256-value run (no masks, no offsets), the rest
      // [cntd[s], cn) go through masks + offsets.  (The screen's fp32 sum may run
      // in any order — its error bound does not depend on it — and the sort is
      // stable, so the sums are deterministic; the exact rescoring keeps the
      // reference order.)  Counting sort over 32-entry chunks: rank within the
      // chunk by __match_any_sync, per-(chunk, bucket) counts, offsets.
      for (int q = threadIdx.x; q < nch * nb; q += blockDim.x) s_cc[q] = 0;
      if (threadIdx.x == 0) s_next = 0;
      __syncthreads();
      for (int j0 = warp * 32; j0 < cn; j0 += nwarps * 32) {
        const int j = j0 + lane;
        int lp = -1;
        if (j < cn) {
          const uint32_t t = (uint32_t)p.terms[c0 + j];
          const uint32_t dy = __ldg(p.tinfo + t).y;
          lp = (int)(dy & 0x7fffffffu) - gs0;
          lp = lp < 0 ? 0 : (lp > nls ? nls : lp);
          if (z == 0) post += p.count_post ? __ldg(p.nc + t) : (dy >> 31);
        }
        const unsigned peers = __match_any_sync(kFull, lp);
        if (j < cn) {
          s_lp[j] = (uint8_t)lp;
          s_pos[j] = (uint16_t)__popc(peers & lt);  // rank among the chunk's equals
          if (lane == __ffs(peers) - 1) s_cc[(j0 >> 5) * nb + lp] = (uint16_t)__popc(peers);
        }
      }
      __syncthreads();
      for (int b = threadIdx.x; b < nb; b += blockDim.x) {  // per bucket: chunk offsets
        int run = 0;
        for (int c = 0; c < nch; ++c) {
          const int x = s_cc[c * nb + b];
          s_cc[c * nb + b] = (uint16_t)run;
          run += x;
        }
        s_cntd[b] = run;
      }
      __syncthreads();
      if (warp == 0) {  // bucket starts in descending prefix order
        int run = 0;
        for (int b0 = nls; b0 >= 0; b0 -= 32) {
          const int b = b0 - lane;
          const int c = b >= 0 ? s_cntd[b] : 0;
          int x = c;
  #pragma unroll
          for (int off = 1; off < 32; off <<= 1) {
            const int y = __shfl_up_sync(kFull, x, off);
            if (lane >= off) x += y;
          }
          if (b >= 0) s_cntd[b] = run + x - c;  // = entries with a longer prefix than b
          run += __shfl_sync(kFull, x, 31);
        }
      }
      __syncthreads();
      for (int j = threadIdx.x; j < cn; j += blockDim.x) {
        const int lp = s_lp[j];
        const uint32_t t = (uint32_t)p.terms[c0 + j];
        const uint32_t row = t * (uint32_t)nblk;
        const int v = __float_as_int(p.val32[c0 + j]);
        const uint32_t base = lp ? __ldg(p.tinfo + t).x : 0u;  // (same sector as the prefix)
        s_ent[s_cntd[lp] + s_cc[(j >> 5) * nb + lp] + s_pos[j]] =
            make_int4((int)(sparse8 ? t * (uint32_t)p.nsp1 : row), v, (int)base, v);
      }
      __syncthreads();
    }
    const bool first = (c0 == rb);
    for (;;) {  // spans handed out dynamically: dense low spans and sparse high
                // ones cost very differently
      int sp = 0;
      if (lane == 0) sp = atomicAdd(&s_next, 1);
      sp = __shfl_sync(kFull, sp, 0);
      if (sp >= nspans) break;
      const int64_t gb = blk0 + (int64_t)sp * RR;
      float acc[RR];
#pragma unroll
      for (int r = 0; r < RR; ++r) acc[r] = first ? 0.f : rho[(sp * RR + r) * 32 + lane];
      if (gb < nblk) {  // nblk is a multiple of RR: a span is all in or all out
        // 32-bit row arithmetic: dim * nblk < 2^31 is checked at build time
        const uint32_t gb32 = (uint32_t)gb;
        const int ls = (int)(gb32 >> 3) - gs0;
        const int nd = ls < nls ? s_cntd[ls] : 0;
        {
          // dense-prefix entries: span gb>>3 starts 256*(gb>>3) values into the
          // term's run; kDepth entries' values in flight, then their FMAs
          using SV = SpanVals<RR, HALF, HALF && MAXREG == 56>;
          const uint32_t r0 = gb32 & (kSpan - 1);
          const char* pl =
              static_cast<const char*>(pv) + SV::lane_bytes(32u * (gb32 - r0), r0, lane);
          const int2* dl = reinterpret_cast<const int2*>(s_ent) + 1;  // {base, value}
          constexpr int kDepth = HALF ? 8 : 2;
          int e = 0;
          for (; e + kDepth <= nd; e += kDepth) {
            SV q[kDepth];
            int2 en[kDepth];
#pragma unroll
            for (int u = 0; u < kDepth; ++u) {
              en[u] = dl[2 * (e + u)];
              q[u].load_dense(pl + dense_off<HALF>(en[u].x));
            }
#pragma unroll
            for (int u = 0; u < kDepth; ++u) q[u].fma(__int_as_float(en[u].y), acc);
          }
          for (; e < nd; ++e) {
            SV q;
            const int2 en = dl[2 * e];
            q.load_dense(pl + dense_off<HALF>(en.x));
            q.fma(__int_as_float(en.y), acc);
          }
        }
        // other terms: masks + offsets, software pipeline (unrolled by two):
        // values of entries e, e+1 and masks of e+2 in flight while e accumulates
        auto ld = [&](int e, MaskPack<RR>& mk, uint32_t& o) {
          if (e < cn) {
            const uint32_t row = (uint32_t)s_ent[e].x + gb32;
            mk.load(masks + row);
            o = __ldg(offs + row);
          } else {
            mk.zero();
            o = 0u;
          }
        };
        if constexpr (HALF && RR == 8) {
          if (p.slot8 && nd < cn) {
            // Sparse spans (< dense_fill*256 postings): the span's values are
            // contiguous at its offset and their slots are in slot8 — a lane
            // per posting, products summed into the warp's slot scratch in
            // entry order (deterministic: one entry's slots are distinct),
            // folded into the registers once per span.  Dense spans beyond
            // the prefix: one 16-B load per lane as in the dense loop.
            float* scr = s_scr + warp * 256;
            float2* stg = reinterpret_cast<float2*>(s_scr + (blockDim.x >> 5) * 256) + warp * 32;
            const unsigned short* p16 = static_cast<const unsigned short*>(pv);
            bool any = false;
            // four entries at a time, eight lanes each (a sparse span holds
            // fewer than dense_fill*256 postings — 4 by default — padded to a
            // multiple of 8 values)
            const int g = lane >> 3, gi = lane & 7;
            for (int e0 = nd; e0 < cn; e0 += 4) {
              const int e = e0 + g;
              uint32_t o0 = 0u, cnt = 0u;
              float v = 0.f;
              bool dense = false;
              if (e < cn) {
                // the span's start and end: adjacent words of the span offsets
                const uint2 oo = ldg_u2(p.soff + (uint32_t)s_ent[e].x + (gb32 >> 3));
                o0 = oo.x;
                v = __int_as_float(s_ent[e].y);
                dense = (o0 & kDense) != 0u;
                if (!dense) cnt = (oo.y & ~kDense) - o0;
              }
              // dense spans beyond the prefix (rare): whole-warp 16-B loads, in entry order
              unsigned dm = __ballot_sync(kFull, dense && gi == 0);
              while (dm) {
                const int src = __ffs(dm) - 1;
                dm &= dm - 1u;
                const uint32_t od = __shfl_sync(kFull, o0, src) & ~kDense;
                const float vd = __shfl_sync(kFull, v, src);
                SpanVals<RR, HALF, HALF && MAXREG == 56> q;
                q.load_dense(static_cast<const char*>(pv) + 2u * (od + 8u * (uint32_t)lane));
                q.fma(vd, acc);
              }
              // sparse postings: a lane each, eight per entry and round (one
              // round under the default dense_fill); equal slots of different
              // entries are added by the lowest lane, in lane order
              const uint32_t rounds = (__reduce_max_sync(kFull, dense ? 0u : cnt) + 7u) >> 3;
              for (uint32_t j = 0; j < rounds; ++j) {
                const uint32_t pi = (uint32_t)gi + 8u * j;
                int sl = 256 + lane;  // distinct sentinel: nothing to add
                float u = 0.f;
                if (!dense && pi < cnt) {
                  const unsigned short hv = __ldg(p16 + o0 + pi);
                  if (hv & 0x7fffu) {  // padding (and an fp16 underflow) is +-0
                    sl = __ldg(p.slot8 + o0 + pi);
                    u = __half2float(__ushort_as_half(hv));
                  }
                }
                any = any || __any_sync(kFull, sl < 256);
                stg[lane] = make_float2(v, u);
                const unsigned peers = __match_any_sync(kFull, sl);
                __syncwarp();
                if (sl < 256 && lane == __ffs(peers) - 1) {
                  float acc_s = scr[sl];
                  for (unsigned pm = peers; pm; pm &= pm - 1u) {
                    const float2 vu = stg[__ffs(pm) - 1];
                    acc_s = fmaf(vu.x, vu.y, acc_s);
                  }
                  scr[sl] = acc_s;
                }
                __syncwarp();
              }
            }
            if (any) {
#pragma unroll
              for (int r = 0; r < RR; ++r) {
                acc[r] += scr[32 * r + lane];
                scr[32 * r + lane] = 0.f;
              }
              __syncwarp();
            }
          }
        }
        if (nd < cn && !(HALF && RR == 8 && p.slot8)) {
          MaskPack<RR> mk;
          uint32_t o;
          ld(nd, mk, o);
          SpanVals<RR, HALF, HALF && MAXREG == 56> A, B;
          A.gather(mk, o, gb32, pv, lane, lanebit, lt);
          ld(nd + 1, mk, o);
          for (int e = nd; e < cn; e += 2) {
            B.gather(mk, o, gb32, pv, lane, lanebit, lt);  // entry e+1
            ld(e + 2, mk, o);
            A.fma(&s_ent[e].y, acc);
            A.gather(mk, o, gb32, pv, lane, lanebit, lt);  // entry e+2
            ld(e + 3, mk, o);
            B.fma(&s_ent[e + 1].y, acc);  // e+1 may be cn: read only if present
          }
        }
      }
#pragma unroll
      for (int r = 0; r < RR; ++r) rho[(sp * RR + r) * 32 + lane] = acc[r];
    }
    c0 += p.rowcap;
  } while (c0 < re);
  __syncthreads();

  screen_epilogue(p, sh, rho, obj, z, rb, re, post);
}

// ---------------------------------------------------------------------------
// exact float64 similarity of object rows to one mean, in the reference order

// headers -> the exact-value lookup view (bivf.cuh: masks, perm, off64)
BivfView exact_view(const uint32_t* headers, int64_t k, int64_t dim) {
  const int64_t nb = ivfkm_bivf_nblk(k);
  const int64_t nh = dim * nb;
  const uint32_t* nc = headers + 2 * nh + 1;
  return BivfView{nb, reinterpret_cast<const uint2*>(headers + bivf_mo_word(k, dim, nb)),
                  reinterpret_cast<const int32_t*>(nc + dim)};
}

struct ExactCtx {
  const int64_t* row_ptr;
  const int32_t* terms;
  const double* val64;
  BivfView bv;
  const double* pv64;
  // optional rank directory of the means' CSR: dir[c*nw + w] = {bits of
  // terms 32w..32w+31 in mean c, rank of the first within the mean's row}
  const uint2* dir = nullptr;
  const int64_t* m_ptr = nullptr;
  const double* m_vals = nullptr;
  int64_t nw = 0;
};

// Warp-cooperative: lanes look up kExactU*32 nonzeros at a time (every
// lookup chain of the chunk in flight: term -> mask + block offset -> value)
// and park the products in the warp's shared scratch; lane 0 then adds them
// in row order.  An absent posting parks +0.0: adding it is exact
// (x + 0.0 == x; at most the sign of an all-zero sum differs, which no
// comparison or sum can see), so the sum equals the reference's sum over
// present postings.
constexpr int kExactU = 4;

__device__ double exact_score_warp(const ExactCtx& x, int64_t rb, int64_t re, int c, int lane,
                                   double* scratch) {
  double acc = 0.0;
  if (x.dir) {  // mean-major lookups through the rank directory
    const uint2* drow = x.dir + (int64_t)c * x.nw;
    const double* mv = x.m_vals + __ldg(x.m_ptr + c);
    for (int64_t h0 = rb; h0 < re; h0 += 32 * kExactU) {
      int32_t t[kExactU];
      uint2 d[kExactU];
#pragma unroll
      for (int u = 0; u < kExactU; ++u) {
        const int64_t h = h0 + 32 * u + lane;
        t[u] = h < re ? __ldg(x.terms + h) : -1;
      }
#pragma unroll
      for (int u = 0; u < kExactU; ++u) d[u] = t[u] >= 0 ? __ldg(drow + (t[u] >> 5)) : make_uint2(0u, 0u);
#pragma unroll
      for (int u = 0; u < kExactU; ++u) {
        const int64_t h = h0 + 32 * u + lane;
        const uint32_t b = t[u] >= 0 ? 1u << (t[u] & 31) : 0u;
        scratch[32 * u + lane] =
            (d[u].x & b) ? __dmul_rn(__ldg(x.val64 + h),
                                     __ldg(mv + d[u].y + __popc(d[u].x & (b - 1u))))
                         : 0.0;
      }
      __syncwarp();
      if (lane == 0) {
        const int n = re - h0 < 32 * kExactU ? (int)(re - h0) : 32 * kExactU;
        int j = 0;
        for (; j + 4 <= n; j += 4) {
          const double2 u = reinterpret_cast<const double2*>(scratch)[j >> 1];
          const double2 v = reinterpret_cast<const double2*>(scratch)[(j >> 1) + 1];
          acc = __dadd_rn(__dadd_rn(__dadd_rn(__dadd_rn(acc, u.x), u.y), v.x), v.y);
        }
        for (; j < n; ++j) acc = __dadd_rn(acc, scratch[j]);
      }
      __syncwarp();
    }
    return __shfl_sync(kFull, acc, 0);
  }
  const int64_t slot = x.bv.perm ? (int64_t)__ldg(x.bv.perm + c) : c;
  const int64_t sb = slot >> 5;
  const uint32_t bit = 1u << (slot & 31);
  for (int64_t h0 = rb; h0 < re; h0 += 32 * kExactU) {
    int32_t t[kExactU];
    uint2 m[kExactU];
#pragma unroll
    for (int u = 0; u < kExactU; ++u) {
      const int64_t h = h0 + 32 * u + lane;
      t[u] = h < re ? __ldg(x.terms + h) : -1;
    }
#pragma unroll
    for (int u = 0; u < kExactU; ++u)
      m[u] = t[u] >= 0 ? __ldg(x.bv.mo + (int64_t)t[u] * x.bv.nblk + sb) : make_uint2(0u, 0u);
#pragma unroll
    for (int u = 0; u < kExactU; ++u) {
      const int64_t h = h0 + 32 * u + lane;
      scratch[32 * u + lane] =
          (m[u].x & bit) ? __dmul_rn(__ldg(x.val64 + h),
                                     __ldg(x.pv64 + m[u].y + __popc(m[u].x & (bit - 1u))))
                         : 0.0;
    }
    __syncwarp();
    if (lane == 0) {
      const int n = re - h0 < 32 * kExactU ? (int)(re - h0) : 32 * kExactU;
      int j = 0;
      for (; j + 4 <= n; j += 4) {
        const double2 u = reinterpret_cast<const double2*>(scratch)[j >> 1];
        const double2 v = reinterpret_cast<const double2*>(scratch)[(j >> 1) + 1];
        acc = __dadd_rn(__dadd_rn(__dadd_rn(__dadd_rn(acc, u.x), u.y), v.x), v.y);
      }
      for (; j < n; ++j) acc = __dadd_rn(acc, scratch[j]);
    }
    __syncwarp();
  }
  return __shfl_sync(kFull, acc, 0);
}

// One thread scores one mean over the whole row.
__device__ double exact_score_thread(const ExactCtx& x, int64_t rb, int64_t re, int64_t c) {
  double acc = 0.0;
  for (int64_t h = rb; h < re; ++h) {
    const int64_t pos = bivf_find(x.bv, x.terms[h], c);
    if (pos >= 0) acc = __dadd_rn(acc, __dmul_rn(x.val64[h], __ldg(x.pv64 + pos)));
  }
  return acc;
}

__global__ void winner_hist_kernel(int64_t n_obj, const int32_t* __restrict__ label32,
                                   unsigned int* __restrict__ hist) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n_obj;
       i += (int64_t)gridDim.x * blockDim.x)
    atomicAdd(&hist[label32[i]], 1u);
}

__global__ void winner_scatter_kernel(int64_t n_obj, const int32_t* __restrict__ label32,
                                      unsigned int* __restrict__ cursor,
                                      int32_t* __restrict__ order) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n_obj;
       i += (int64_t)gridDim.x * blockDim.x)
    order[atomicAdd(&cursor[label32[i]], 1u)] = (int32_t)i;
}

// rank directory of a mean-major CSR (0-based terms ascending per row):
// each warp takes a contiguous range of entries (one binary search for its
// first mean, then advancing), 32 at a time; lanes sharing a (mean, word) OR
// their bits together and the lowest of them publishes
__global__ void rankdir_bits_kernel(int64_t k, int64_t nw, const int64_t* __restrict__ ptr,
                                    const int32_t* __restrict__ terms, uint2* __restrict__ dir) {
  const int lane = threadIdx.x & 31;
  const int64_t nwarps = (int64_t)gridDim.x * (blockDim.x >> 5);
  const int64_t wid = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5);
  const int64_t nnz = ptr[k];
  const int64_t per = ((nnz + nwarps - 1) / nwarps + 31) / 32 * 32;
  const int64_t b0 = wid * per, b1 = b0 + per < nnz ? b0 + per : nnz;
  if (b0 >= b1) return;
  int64_t c;
  {
    int64_t lo = 0, hi = k;  // ptr[c] <= b0 < ptr[c+1]
    while (hi - lo > 1) {
      const int64_t mid = (lo + hi) >> 1;
      if (__ldg(ptr + mid) <= b0) lo = mid; else hi = mid;
    }
    c = lo;
  }
  for (int64_t e0 = b0; e0 < b1; e0 += 32) {
    const int64_t e = e0 + lane;
    int64_t key = -1;
    uint32_t bit = 0u;
    if (e < b1) {
      int64_t cl = c;
      while (__ldg(ptr + cl + 1) <= e) ++cl;  // rows are long: rarely more than once
      const int32_t t = terms[e];
      key = cl * nw + (t >> 5);
      bit = 1u << (t & 31);
    }
    // keys ascend across the lanes: a segmented OR towards each run's last
    // lane (shuffles), which publishes — with an atomic only where the run
    // may continue in a neighbouring chunk (first and last run)
    const int64_t kn = __shfl_down_sync(kFull, key, 1);
    uint32_t acc = bit;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const uint32_t y = __shfl_up_sync(kFull, acc, off);
      const int64_t ky = __shfl_up_sync(kFull, key, off);
      if (lane >= off && ky == key) acc |= y;
    }
    const int64_t k0 = __shfl_sync(kFull, key, 0);
    const bool tail = lane == 31 || kn < 0;  // the chunk's last valid run
    if (key >= 0 && (tail || kn != key)) {
      if (key == k0 || tail) atomicOr(&dir[key].x, acc);
      else dir[key].x = acc;  // wholly inside this chunk
    }
    // the mean of the next chunk's first entry
    const int64_t nx = e0 + 32;
    if (nx < b1)
      while (__ldg(ptr + c + 1) <= nx) ++c;
  }
}

__global__ void rankdir_scan_kernel(int64_t k, int64_t nw, uint2* __restrict__ dir) {
  const int lane = threadIdx.x & 31;
  const int64_t wpb = blockDim.x >> 5;
  for (int64_t c = blockIdx.x * wpb + (threadIdx.x >> 5); c < k; c += gridDim.x * wpb) {
    uint2* row = dir + c * nw;
    unsigned int carry = 0;
    for (int64_t w0 = 0; w0 < nw; w0 += 32) {
      const int64_t w = w0 + lane;
      const unsigned int pc = w < nw ? __popc(row[w].x) : 0u;
      unsigned int inc = pc;
#pragma unroll
      for (int off = 1; off < 32; off <<= 1) {
        const unsigned int y = __shfl_up_sync(kFull, inc, off);
        if (lane >= off) inc += y;
      }
      if (w < nw) row[w].y = carry + inc - pc;
      carry += __shfl_sync(kFull, inc, 31);
    }
  }
}

struct FinalParams {
  int64_t n_obj;
  ExactCtx x;
  const int32_t* label32;
  const int32_t* slot_of;
  const int32_t* q_cnt;
  const int32_t* q_cid;
  int32_t* labels;
  double* sims;
  int32_t* ovf_list;
  unsigned int* ovf_len;
  int rule;  // 0: IVF argmax (_kernels.pyx:17-26); 1: IVFD (_kernels.pyx:178-207)
  const int32_t* order = nullptr;  // objects grouped by screen winner, or nullptr
};

// IVFD keeps a label only when its similarity beats 0.0 (rho_max starts at
// 0.0 and label at 1, strict '>', _kernels.pyx:190-205): otherwise mean 0,
// whose exact similarity is then the objective summand.
__device__ __forceinline__ bool ivfd_falls_back(const FinalParams& p, double best, int c) {
  return p.rule == 1 && !(best > 0.0) && c != 0;
}

__global__ void __launch_bounds__(256) finalize_kernel(FinalParams p) {
  __shared__ __align__(16) double s_scr[8][32 * kExactU];
  const int lane = threadIdx.x & 31;
  double* scratch = s_scr[threadIdx.x >> 5];
  const int64_t wpb = blockDim.x >> 5;
  for (int64_t q = blockIdx.x * wpb + (threadIdx.x >> 5); q < p.n_obj; q += gridDim.x * wpb) {
    const int64_t i = p.order ? (int64_t)p.order[q] : q;
    const int64_t rb = p.x.row_ptr[i], re = p.x.row_ptr[i + 1];
    const int slot = p.slot_of[i];
    if (slot < 0) {
      int c = p.label32[i];
      double s = exact_score_warp(p.x, rb, re, c, lane, scratch);
      if (ivfd_falls_back(p, s, c)) {
        c = 0;
        s = exact_score_warp(p.x, rb, re, 0, lane, scratch);
      }
      if (lane == 0) {
        p.labels[i] = c;
        p.sims[i] = s;
      }
      continue;
    }
    const int cnt = p.q_cnt[slot];
    if (cnt > kMaxC) {
      if (lane == 0) p.ovf_list[atomicAdd(p.ovf_len, 1u)] = (int)i;
      continue;
    }
    double bv = -INFINITY;
    int bc = INT_MAX;
    for (int j = 0; j < cnt; ++j) {
      const int c = p.q_cid[(int64_t)slot * kMaxC + j];
      const double s = exact_score_warp(p.x, rb, re, c, lane, scratch);
      if (s > bv || (s == bv && c < bc)) {
        bv = s;
        bc = c;
      }
    }
    if (ivfd_falls_back(p, bv, bc)) {
      bc = 0;
      bv = exact_score_warp(p.x, rb, re, 0, lane, scratch);
    }
    if (lane == 0) {
      p.labels[i] = bc;
      p.sims[i] = bv;
    }
  }
}

__global__ void __launch_bounds__(256) score_labels_kernel(int64_t n_obj, ExactCtx x,
                                                           const int32_t* labels, double* sims) {
  __shared__ __align__(16) double s_scr[8][32 * kExactU];
  const int lane = threadIdx.x & 31;
  double* scratch = s_scr[threadIdx.x >> 5];
  const int64_t wpb = blockDim.x >> 5;
  for (int64_t i = blockIdx.x * wpb + (threadIdx.x >> 5); i < n_obj; i += gridDim.x * wpb) {
    const double s =
        exact_score_warp(x, x.row_ptr[i], x.row_ptr[i + 1], labels[i], lane, scratch);
    if (lane == 0) sims[i] = s;
  }
}

// Objects whose window held more than kMaxC means: score every mean exactly.
__global__ void __launch_bounds__(1024) overflow_kernel(FinalParams p, int64_t k) {
  __shared__ double rv[32];
  __shared__ int rc[32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const unsigned n = *p.ovf_len;
  for (unsigned q = blockIdx.x; q < n; q += gridDim.x) {
    const int64_t i = p.ovf_list[q];
    const int64_t rb = p.x.row_ptr[i], re = p.x.row_ptr[i + 1];
    double bv = -INFINITY;
    int bc = INT_MAX;
    for (int64_t c = threadIdx.x; c < k; c += blockDim.x) {
      const double s = exact_score_thread(p.x, rb, re, c);
      if (s > bv) {
        bv = s;
        bc = (int)c;
      }
    }
    for (int off = 16; off > 0; off >>= 1) {
      const double ov = __shfl_xor_sync(kFull, bv, off);
      const int oc = __shfl_xor_sync(kFull, bc, off);
      if (ov > bv || (ov == bv && oc < bc)) {
        bv = ov;
        bc = oc;
      }
    }
    __syncthreads();
    if (lane == 0) {
      rv[warp] = bv;
      rc[warp] = bc;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      for (int w = 1; w < nw; ++w)
        if (rv[w] > bv || (rv[w] == bv && rc[w] < bc)) {
          bv = rv[w];
          bc = rc[w];
        }
      if (ivfd_falls_back(p, bv, bc)) {
        bc = 0;
        bv = exact_score_thread(p.x, rb, re, 0);
      }
      p.labels[i] = bc;
      p.sims[i] = bv;
    }
  }
}

// Add s exactly into a fixed-point accumulator: X = s * 2^1074 is an integer;
// limb l holds bits [32l, 32l+32) as a signed partial sum.
__device__ __forceinline__ void add_exact(double s, long long* limbs, unsigned& flags) {
  if (s == 0.0) return;
  const unsigned long long bits = (unsigned long long)__double_as_longlong(s);
  const int ex = (int)((bits >> 52) & 0x7ff);
  if (ex == 0x7ff) {
    flags |= 1u;
    return;
  }
  unsigned long long m = bits & ((1ull << 52) - 1ull);
  int b = 0;
  if (ex != 0) {
    m |= 1ull << 52;
    b = ex - 1;
  }
  const int idx = b >> 5, sh = b & 31;
  if (idx + 2 >= kLimbs) {
    flags |= 2u;
    return;
  }
  const unsigned c0 = (unsigned)(m << sh);
  const unsigned long long t = sh ? (m >> (32 - sh)) : (m >> 32);
  const long long sg = (bits >> 63) ? -1 : 1;
  limbs[idx] += sg * (long long)c0;
  limbs[idx + 1] += sg * (long long)(unsigned)t;
  limbs[idx + 2] += sg * (long long)(unsigned)(t >> 32);
}

__global__ void __launch_bounds__(256) accumulate_kernel(int64_t n_obj, const int32_t* labels,
                                                         const double* sims,
                                                         const int32_t* prev,
                                                         unsigned long long* sizes,
                                                         ivfkm_stats* stats) {
  __shared__ long long s_limbs[kLimbs];
  __shared__ unsigned long long s_changed;
  __shared__ unsigned s_flags;
  for (int l = threadIdx.x; l < kLimbs; l += blockDim.x) s_limbs[l] = 0;
  if (threadIdx.x == 0) {
    s_changed = 0;
    s_flags = 0;
  }
  __syncthreads();
  long long limbs[kLimbs];
#pragma unroll
  for (int l = 0; l < kLimbs; ++l) limbs[l] = 0;
  unsigned flags = 0;
  unsigned long long changed = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n_obj;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int lab = labels[i];
    if (prev && prev[i] != lab) ++changed;
    if (sizes) atomicAdd(&sizes[lab], 1ull);
    add_exact(sims[i], limbs, flags);
  }
#pragma unroll
  for (int l = 0; l < kLimbs; ++l)
    if (limbs[l]) atomicAdd(reinterpret_cast<unsigned long long*>(&s_limbs[l]),
                            (unsigned long long)limbs[l]);
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) changed += __shfl_xor_sync(kFull, changed, off);
  if ((threadIdx.x & 31) == 0 && changed) atomicAdd(&s_changed, changed);
  if (flags) atomicOr(&s_flags, flags);
  __syncthreads();
  for (int l = threadIdx.x; l < kLimbs; l += blockDim.x)
    if (s_limbs[l])
      atomicAdd(reinterpret_cast<unsigned long long*>(&stats->obj_limbs[l]),
                (unsigned long long)s_limbs[l]);
  if (threadIdx.x == 0) {
    if (s_changed) atomicAdd(&stats->changed, s_changed);
    if (s_flags) atomicOr(&stats->obj_flags, (unsigned long long)s_flags);
  }
}

// ---------------------------------------------------------------------------
// IVFD, object-inverted (_kernels.pyx:178-207): means outermost, each mean's
// similarity to every object accumulated in a length-N vector over the
// objects' inverted file, then folded into the running best per object.
// The GPU shape: a *wave* of M means at once, one CTA per mean, each with its
// own length-N float64 slot (scratch in HBM); inside a CTA the mean's terms go
// in ascending order with a barrier between terms (one object may appear in
// consecutive terms' lists), the term's object postings split over the
// threads — every object's sum therefore adds u*x in ascending term order
// with __dmul_rn/__dadd_rn, bit-identical to the reference's rho; a reduce
// kernel then scans the wave's slots per object in ascending mean order
// (strict '>' from 0.0, label 1 when nothing beats it) and clears them.

__global__ void __launch_bounds__(256) ivfd_scatter_kernel(
    int64_t n_obj, int64_t j0, int64_t k, const int64_t* __restrict__ x_ptr,
    const int32_t* __restrict__ x_obj, const double* __restrict__ x_val,
    const int64_t* __restrict__ m_ptr, const int32_t* __restrict__ m_terms,
    const double* __restrict__ m_vals, double* __restrict__ slots,
    unsigned long long* __restrict__ postings) {
  const int64_t j = j0 + blockIdx.x;
  if (j >= k) return;
  double* rho = slots + (int64_t)blockIdx.x * n_obj;
  unsigned long long cnt = 0;
  for (int64_t h = m_ptr[j]; h < m_ptr[j + 1]; ++h) {
    const int32_t t = __ldg(m_terms + h);
    const double u = __ldg(m_vals + h);
    const int64_t q0 = __ldg(x_ptr + t), q1 = __ldg(x_ptr + t + 1);
    for (int64_t q = q0 + threadIdx.x; q < q1; q += blockDim.x) {
      const int32_t i = __ldg(x_obj + q);
      rho[i] = __dadd_rn(rho[i], __dmul_rn(u, __ldg(x_val + q)));
    }
    if (threadIdx.x == 0) cnt += (unsigned long long)(q1 - q0);
    __syncthreads();  // the next term may hit the same objects
  }
  if (threadIdx.x == 0 && cnt) atomicAdd(postings, cnt);
}

__global__ void __launch_bounds__(256) ivfd_reduce_kernel(
    int64_t n_obj, int64_t j0, int64_t m, double* __restrict__ slots, double* __restrict__ best,
    int32_t* __restrict__ label, double* __restrict__ sim0) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n_obj;
       i += (int64_t)gridDim.x * blockDim.x) {
    double b = j0 == 0 ? 0.0 : best[i];
    int32_t l = j0 == 0 ? 0 : label[i];
    for (int64_t c = 0; c < m; ++c) {
      double* r = slots + c * n_obj + i;
      const double v = *r;
      *r = 0.0;
      if (j0 + c == 0) sim0[i] = v;  // mean 1's similarity: the summand when nothing beats 0.0
      if (v > b) {
        b = v;
        l = (int32_t)(j0 + c);
      }
    }
    best[i] = b;
    label[i] = l;
  }
}

__global__ void ivfd_finish_kernel(int64_t n_obj, const double* __restrict__ best,
                                   const int32_t* __restrict__ label,
                                   const double* __restrict__ sim0, int32_t* __restrict__ labels,
                                   double* __restrict__ sims) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n_obj;
       i += (int64_t)gridDim.x * blockDim.x) {
    labels[i] = label[i];
    sims[i] = best[i] > 0.0 ? best[i] : sim0[i];
  }
}

// objects' inverted file: entry -> (term key, entry index), stably sorted by term
__global__ void entry_keys_kernel(int64_t n_obj, const int64_t* __restrict__ row_ptr,
                                  const int32_t* __restrict__ terms, int32_t* __restrict__ key,
                                  int32_t* __restrict__ obj, int32_t* __restrict__ idx,
                                  unsigned int* __restrict__ hist) {
  const int lane = threadIdx.x & 31;
  const int64_t wpb = blockDim.x >> 5;
  for (int64_t i = blockIdx.x * wpb + (threadIdx.x >> 5); i < n_obj; i += gridDim.x * wpb) {
    for (int64_t e = row_ptr[i] + lane; e < row_ptr[i + 1]; e += 32) {
      const int32_t t = terms[e];
      key[e] = t;
      obj[e] = (int32_t)i;
      idx[e] = (int32_t)e;
      atomicAdd(&hist[t], 1u);
    }
  }
}

__global__ void entry_gather_kernel(int64_t nnz, const int32_t* __restrict__ sidx,
                                    const int32_t* __restrict__ obj,
                                    const double* __restrict__ val64,
                                    int32_t* __restrict__ x_obj, double* __restrict__ x_val) {
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < nnz;
       q += (int64_t)gridDim.x * blockDim.x) {
    const int32_t e = sidx[q];
    x_obj[q] = obj[e];
    x_val[q] = val64[e];
  }
}

// The assign's posting volume from the objects' document frequencies.
__global__ void postings_dot_kernel(int64_t dim, const uint32_t* __restrict__ df,
                                    const uint32_t* __restrict__ nc, ivfkm_stats* stats) {
  unsigned long long s = 0;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < dim;
       t += (int64_t)gridDim.x * blockDim.x)
    s += (unsigned long long)df[t] * (unsigned long long)nc[t];
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) s += __shfl_xor_sync(kFull, s, off);
  if ((threadIdx.x & 31) == 0 && s) atomicAdd(&stats->postings, s);
}

// Each row's entries stably sorted by the terms' dense prefix, longest first
// (for the slot-range passes: every pass's clamped bucket order is this order,
// so the screen stages a pass by copying).  One warp per row: a counting sort
// over the prefix lengths 0..nsp, ranks within 32-entry chunks by
// __match_any_sync.
constexpr int kPresortBuckets = 256;
__global__ void __launch_bounds__(256) presort_rows_kernel(
    int64_t n_obj, const int64_t* __restrict__ row_ptr, const int32_t* __restrict__ terms,
    const float* __restrict__ val32, const uint32_t* __restrict__ dpre,
    const uint2* __restrict__ tinfo, int nsp, int2* __restrict__ ps_t,
    int2* __restrict__ ps_v) {
  __shared__ int s_cnt[8][kPresortBuckets];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const unsigned lt = (1u << lane) - 1u;
  int* cnt = s_cnt[w];
  const int nbk = nsp + 1;
  const int64_t wpb = blockDim.x >> 5;
  for (int64_t i = blockIdx.x * wpb + w; i < n_obj; i += gridDim.x * wpb) {
    const int64_t rb = row_ptr[i], re = row_ptr[i + 1];
    for (int b = lane; b < nbk; b += 32) cnt[b] = 0;
    __syncwarp();
    for (int64_t h0 = rb; h0 < re; h0 += 32) {
      const int64_t h = h0 + lane;
      int key = -1;
      if (h < re) {
        const int d = (int)__ldg(dpre + terms[h]);
        key = nsp - (d < nsp ? d : nsp);
      }
      const unsigned peers = __match_any_sync(kFull, key);
      if (h < re && lane == __ffs(peers) - 1) cnt[key] += __popc(peers);
      __syncwarp();
    }
    int carry = 0;  // exclusive scan of the bucket counts
    for (int b0 = 0; b0 < nbk; b0 += 32) {
      const int b = b0 + lane;
      const int c = b < nbk ? cnt[b] : 0;
      int x = c;
#pragma unroll
      for (int off = 1; off < 32; off <<= 1) {
        const int y = __shfl_up_sync(kFull, x, off);
        if (lane >= off) x += y;
      }
      if (b < nbk) cnt[b] = carry + x - c;
      carry += __shfl_sync(kFull, x, 31);
    }
    __syncwarp();
    for (int64_t h0 = rb; h0 < re; h0 += 32) {
      const int64_t h = h0 + lane;
      int key = -1;
      int32_t t = 0;
      int d = 0;
      if (h < re) {
        t = terms[h];
        d = (int)__ldg(dpre + t);
        key = nsp - (d < nsp ? d : nsp);
      }
      const unsigned peers = __match_any_sync(kFull, key);
      if (h < re) {
        const int64_t pos = rb + cnt[key] + __popc(peers & lt);
        // {the start of the term's dense run, dense prefix | has-postings bit}
        const uint2 ti = __ldg(tinfo + t);
        ps_t[pos] = make_int2(t, (int)ti.y);
        ps_v[pos] = make_int2((int)ti.x, __float_as_int(val32[h]));
      }
      __syncwarp();
      if (h < re && lane == __ffs(peers) - 1) cnt[key] += __popc(peers);
      __syncwarp();
    }
  }
}

struct AssignWs {
  int32_t* label32;
  int32_t* slot_of;
  int32_t* q_obj;
  int32_t* q_cnt;
  int32_t* q_cid;
  int32_t* ovf_list;
  unsigned int* ovf_len;
  unsigned int* cl_pos;  // k + 1: objects per screen winner, then their cursors
  int32_t* fin_order;    // n: objects grouped by screen winner
  float* st_best;        // slot-range pass state (ScreenParams)
  int32_t* st_slot;
  int32_t* st_cnt;
  int2* st_cand;
  void* cub;
  size_t cub_bytes;
};

AssignWs carve_assign(void* base, int64_t n, int64_t k, size_t* total) {
  Carver c(base);
  AssignWs w;
  w.label32 = c.take<int32_t>(n);
  w.slot_of = c.take<int32_t>(n);
  w.q_obj = c.take<int32_t>(n);
  w.q_cnt = c.take<int32_t>(n);
  w.q_cid = c.take<int32_t>((size_t)n * kMaxC);
  w.ovf_list = c.take<int32_t>(n);
  w.ovf_len = c.take<unsigned int>(4);
  w.cl_pos = c.take<unsigned int>((size_t)k + 1);
  w.fin_order = c.take<int32_t>(n);
  w.st_best = c.take<float>(n);
  w.st_slot = c.take<int32_t>(n);
  w.st_cnt = c.take<int32_t>(n);
  w.st_cand = c.take<int2>((size_t)n * kMaxC);
  w.cub_bytes = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, w.cub_bytes, (unsigned int*)nullptr,
                                (unsigned int*)nullptr, (int)(k + 1));
  w.cub = c.take_bytes(w.cub_bytes);
  if (total) *total = c.off;
  return w;
}

static int g_max_warps = 16;  // register screen: warps per CTA at most
static int g_force_warps = 0;  // register screen: exact warps per CTA (0 = planned)

struct Plan {
  int rr, nsplit, cta_blocks, warps, rowcap;
  bool passes = false;  // nsplit slot-range passes instead of a cluster of nsplit CTAs
  bool tma = false;  // (staged screens removed in round 2; the plan query reports 0)
  int mode = 0;
  size_t smem;
  size_t cc_bytes = 0;
};

static int g_passes = 0;  // slot-range passes (0/1 = off; set per launch by the engine)

int choose_warps(int spans, size_t smem) {
  const int by_smem = (228 * 1024) / (int)(smem + 1024 + 5 * 1024);
  int best_w = 1;
  long best = -1;
  for (int w = 1; w <= 16 && w <= (spans > 0 ? spans : 1); ++w) {
    int ctas = 65536 / (w * 32 * 64);
    if (ctas > by_smem) ctas = by_smem;
    if (ctas > 32) ctas = 32;
    const long score = (long)ctas * w * 64 + ctas;
    if (score > best) {
      best = score;
      best_w = w;
    }
  }
  return best_w;
}

// Counting-sort scratch of the in-CTA row sort: a uint16 per (32-entry chunk,
// dense-prefix bucket), buckets = the CTA's spans + 1 (<= kMaxLocalSpans + 1).
size_t cc_bytes_for(int rowcap, int cta_blocks) {
  int nb = cta_blocks / kSpan + 2;
  if (nb > kMaxLocalSpans + 1) nb = kMaxLocalSpans + 1;
  return ((size_t)(rowcap / 32) * nb * sizeof(uint16_t) + 15) & ~(size_t)15;
}

int plan_screen(int64_t k, int rowcap, int smem_limit, int rr, Plan* out,
                bool sparse_scratch = false, bool presorted = false) {
  const int64_t nblk = ivfkm_bivf_nblk(k);
  Plan pl;
  const bool adaptive = smem_limit <= 0;
  if (smem_limit <= 0) {
    // Adaptive budget (measured on configs 1-4): one CTA per object while rho
    // and the staged row fit in 64 KB (k <= ~13,000: every split CTA would
    // stage the whole row again); beyond, split rho over a thread-block
    // cluster at about half of it per CTA, between 24 KB and 100 KB.
    const int64_t rho = nblk * 128;
    const int64_t stg = (int64_t)rowcap * kEntryBytes;
    int64_t b = rho / 2 + (stg > 8 * 1024 ? stg : 8 * 1024);
    if (b < 24 * 1024) b = 24 * 1024;
    if (b > 100 * 1024) b = 100 * 1024;
    if (rho + stg <= 64 * 1024) b = kSmemLimit - 2048;
    smem_limit = (int)b;
  }
  pl.tma = false;
  pl.mode = 0;
  pl.rr = rr > 0 ? rr : (nblk >= 32 ? 8 : 2);
  pl.rowcap = rowcap < kMaxChunks * 32 ? rowcap : kMaxChunks * 32;  // staging counts cap
  const size_t stage = (size_t)pl.rowcap * kEntryBytes;
  pl.nsplit = 0;
  for (int s = 1; s <= kMaxSplit; ++s) {
    int64_t cb = (nblk + s - 1) / s;
    cb = (cb + pl.rr - 1) / pl.rr * pl.rr;
    const size_t smem = (size_t)cb * 128 + stage;
    if (smem <= (size_t)smem_limit) {
      pl.nsplit = s;
      pl.cta_blocks = (int)cb;
      pl.smem = smem;
      break;
    }
  }
  if (pl.nsplit == 0) return IVFKM_E_UNSUPPORTED;
  // Warps per CTA (spans are handed out dynamically, so any count works):
  // the most resident warps per SM under the register file (64 registers a
  // lane) and the shared-memory footprint, then the most resident CTAs
  // (objects in flight).  Measured at config 2: 8 warps x 4 CTAs beats
  // 14 x 2 by 14%; at config 4 (95 KB per CTA) 16 x 2 beats 8 x 2 by 40%.
  if (g_passes > 1 && adaptive && rr >= 0) {
    // slot-range passes: every launch screens all objects
    // against 1/passes of the slots, so a pass's postings share the L2 and
    // small CTAs (<= 4 warps, 56 registers) keep more objects in flight
    int64_t cb = (nblk + g_passes - 1) / g_passes;
    cb = (cb + pl.rr - 1) / pl.rr * pl.rr;
    pl.nsplit = (int)((nblk + cb - 1) / cb);
    pl.cta_blocks = (int)cb;
    pl.smem = (size_t)cb * 128 + stage;
    pl.passes = pl.nsplit > 1;
  }
  // the counting-sort scratch, unless every launch stages presorted rows
  pl.cc_bytes = (presorted && pl.passes) ? 0 : cc_bytes_for(pl.rowcap, pl.cta_blocks);
  pl.smem += pl.cc_bytes;
  const int best_w = choose_warps(pl.cta_blocks / pl.rr, pl.smem);
  pl.warps = g_max_warps < best_w ? g_max_warps : best_w;
  if (g_force_warps > 0) pl.warps = g_force_warps;  // tests: any count is valid
  // the sparse-span path's slot scratch (1 KB per warp) after the 16-B
  // aligned stage (fp16 8-block spans only)
  if (sparse_scratch && pl.rr == 8)
    pl.smem += 16 + (size_t)pl.warps * (256 * sizeof(float) + 32 * sizeof(float2));
  *out = pl;
  return IVFKM_OK;
}

// The instantiation launch_screen picks for a plan (56 registers for the
// small fp16 CTAs, 64 otherwise).
int plan_maxreg(const Plan& pl, bool half) {
  return (!pl.tma && half && pl.rr == 8 && pl.warps <= 4) ? 56 : 64;
}

template <int RR>
int launch_screen(const Plan& pl, const ScreenParams& p, cudaStream_t st) {
  auto fn = p.half ? (plan_maxreg(pl, true) == 56 ? screen_kernel<RR, true, 56>
                                                   : screen_kernel<RR, true>)
                    : screen_kernel<RR, false>;
  {
    // raise the kernel's dynamic shared-memory limit only when a launch needs
    // more than it was given (per device): the call costs host time on every
    // launch otherwise
    static std::mutex mu;
    static std::map<std::pair<const void*, int>, size_t> limit;
    std::lock_guard<std::mutex> g(mu);
    int dev = 0;
    IVFKM_TRY(cudaGetDevice(&dev));
    size_t& cur = limit[std::make_pair(reinterpret_cast<const void*>(fn), dev)];
    if (pl.smem > cur) {
      IVFKM_TRY(
          cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)pl.smem));
      cur = pl.smem;
    }
  }
  if (pl.passes) {  // slot-range passes: one launch per pass, state in between
    for (int z = 0; z < pl.nsplit; ++z) {
      ScreenParams q = p;
      q.pass = z;
      q.npass = pl.nsplit;
      fn<<<(unsigned)p.n_obj, pl.warps * 32, pl.smem, st>>>(q);
      IVFKM_CHECK_LAUNCH();
    }
    return IVFKM_OK;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(p.n_obj * pl.nsplit));
  cfg.blockDim = dim3(pl.warps * 32);
  cfg.dynamicSmemBytes = pl.smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = pl.nsplit;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pl.nsplit > 1 ? 1 : 0;
  IVFKM_TRY(cudaLaunchKernelEx(&cfg, fn, p));
  return IVFKM_OK;
}

}  // namespace

// Longest rows first: a static LPT order for the one-CTA-per-object screen,
// so the long rows do not trail at the end of the grid.
namespace {
__global__ void rowlen_keys_kernel(int64_t n, const int64_t* __restrict__ row_ptr,
                                   unsigned int* __restrict__ key, int32_t* __restrict__ id) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t len = row_ptr[i + 1] - row_ptr[i];
    key[i] = ~(unsigned)(len < 0xffffffffll ? len : 0xffffffffll);
    id[i] = (int32_t)i;
  }
}
}  // namespace

extern "C" size_t ivfkm_row_order_workspace_size(int64_t n_obj) {
  size_t sb = 0;
  cub::DoubleBuffer<unsigned int> kb(nullptr, nullptr);
  cub::DoubleBuffer<int32_t> vb(nullptr, nullptr);
  cub::DeviceRadixSort::SortPairs(nullptr, sb, kb, vb, (int)n_obj);
  Carver c(nullptr);
  c.take<unsigned int>(n_obj);
  c.take<unsigned int>(n_obj);
  c.take<int32_t>(n_obj);
  c.take_bytes(sb);
  return c.off;
}

extern "C" int ivfkm_row_order(int64_t n_obj, const int64_t* row_ptr, int32_t* order, void* ws,
                               size_t ws_bytes, ivfkm_stream_t stream_) {
  if (n_obj < 0 || n_obj > INT32_MAX || !row_ptr || !order) return IVFKM_E_ARG;
  if (ws_bytes < ivfkm_row_order_workspace_size(n_obj)) return IVFKM_E_WORKSPACE;
  if (n_obj == 0) return IVFKM_OK;
  size_t sb = 0;
  {
    cub::DoubleBuffer<unsigned int> kb(nullptr, nullptr);
    cub::DoubleBuffer<int32_t> vb(nullptr, nullptr);
    cub::DeviceRadixSort::SortPairs(nullptr, sb, kb, vb, (int)n_obj);
  }
  Carver c(ws);
  unsigned int* ka = c.take<unsigned int>(n_obj);
  unsigned int* kb2 = c.take<unsigned int>(n_obj);
  int32_t* ib = c.take<int32_t>(n_obj);
  void* tmp = c.take_bytes(sb);
  cudaStream_t st = as_stream(stream_);
  rowlen_keys_kernel<<<grid_for(n_obj, 256), 256, 0, st>>>(n_obj, row_ptr, ka, order);
  IVFKM_CHECK_LAUNCH();
  cub::DoubleBuffer<unsigned int> kbuf(ka, kb2);
  cub::DoubleBuffer<int32_t> vbuf(order, ib);
  IVFKM_TRY(cub::DeviceRadixSort::SortPairs(tmp, sb, kbuf, vbuf, (int)n_obj, 0, 32, st));
  if (vbuf.Current() != order)
    IVFKM_TRY(cudaMemcpyAsync(order, vbuf.Current(), sizeof(int32_t) * n_obj,
                              cudaMemcpyDeviceToDevice, st));
  return IVFKM_OK;
}

extern "C" size_t ivfkm_assign_workspace_size(int64_t n_obj, int64_t k) {
  size_t total = 0;
  carve_assign(nullptr, n_obj, k, &total);
  return total;
}

// Tuning knobs.  rowcap: row entries staged per pass (longer rows run in
// several passes with rho parked in shared memory between passes).
// smem_limit: shared-memory budget per CTA; a smaller budget forces the
// thread-block-cluster split at small k (used by the tests).
static int g_rowcap = 1024;
static int g_smem_limit = 0;  // 0: adaptive (see plan_screen)
static int g_rr = 0;  // 0: automatic LDG screen; 2/4/8: LDG screen span; -8: TMA screen
extern "C" void ivfkm_set_tuning(int rowcap, int smem_limit, int rr) {
  if (rowcap >= 32 && rowcap <= 8192) g_rowcap = rowcap / 32 * 32;
  if (smem_limit >= 1024 && smem_limit <= kSmemLimit - 2048) g_smem_limit = smem_limit;
  if (smem_limit == -1) g_smem_limit = 0;  // back to adaptive
  if (rr == 0 || rr == 2 || rr == 4 || rr == 8) g_rr = rr;
}

// Tests: force the register screen's warps per CTA (1..16; 0 = planned) —
// spans are handed out dynamically, so every count computes the same sums.
extern "C" void ivfkm_set_screen_warps(int warps) {
  if (warps >= 0 && warps <= 16) g_force_warps = warps;
}

extern "C" int ivfkm_set_screen_option(int which, int value) {
  switch (which) {
    case 1: g_passes = value < 0 ? 0 : (value > 4096 ? 4096 : value); return IVFKM_OK;
    default: return IVFKM_E_ARG;
  }
}

extern "C" int ivfkm_screen_plan(int64_t k, int rowcap, int screen_bits, int32_t* out) {
  if (k < 1 || !out || (screen_bits != 16 && screen_bits != 32)) return IVFKM_E_ARG;
  Plan pl;
  // as the engine launches it: slot bytes for the fp16 screen's sparse spans
  // from 16 spans up, presorted rows under slot-range passes
  const bool slots = screen_bits == 16 && ivfkm_bivf_nblk(k) / kSpan >= 16;
  const int rc = plan_screen(k, rowcap >= 32 ? rowcap / 32 * 32 : g_rowcap, g_smem_limit, g_rr,
                             &pl, slots, /*presorted=*/true);
  if (rc) return rc;
  out[0] = pl.rr;
  out[1] = pl.nsplit;
  out[2] = pl.cta_blocks;
  out[3] = pl.warps;
  out[4] = pl.rowcap;
  out[5] = pl.mode;
  out[6] = (int32_t)pl.smem;
  out[7] = plan_maxreg(pl, screen_bits == 16);
  return IVFKM_OK;
}

namespace {

struct AssignArgs {
  int64_t n_obj;
  const int64_t* row_ptr;
  const int32_t* terms;
  const float* val32;
  const double* val64;
  const double* xnorm;
  int64_t k, dim;
  const uint32_t* headers;
  const void* pval_screen;
  int screen_bits;
  const double* pval64;
  double mu_max;
  ivfkm_stats* stats;
  const int32_t* order;
  int32_t* ps_t = nullptr;  // presorted rows (pass mode), see ivfkm_assign_screen_ex
  float* ps_v = nullptr;
  const uint8_t* slot8 = nullptr;  // sparse spans' slot bytes (ivfkm_bivf_slots)
  const uint32_t* doc_freq = nullptr;  // objects per term, or nullptr: the screen counts
};

int screen_impl(const AssignArgs& a, const AssignWs& w, cudaStream_t st) {
  Plan pl;
  const bool can_presort = a.ps_t && ivfkm_bivf_nblk(a.k) / kSpan < kPresortBuckets;
  int rc = plan_screen(a.k, g_rowcap, g_smem_limit, g_rr, &pl,
                       a.slot8 != nullptr && a.screen_bits == 16, can_presort);
  if (rc) return rc;
  ScreenParams sp;
  sp.n_obj = a.n_obj;
  sp.row_ptr = a.row_ptr;
  sp.terms = a.terms;
  sp.val32 = a.val32;
  sp.xnorm = a.xnorm;
  sp.k = a.k;
  sp.nblk = ivfkm_bivf_nblk(a.k);
  sp.masks = a.headers;
  sp.offs = a.headers + a.dim * sp.nblk;
  sp.nc = a.headers + 2 * a.dim * sp.nblk + 1;
  sp.inv = reinterpret_cast<const int32_t*>(sp.nc + a.dim) + a.k;
  sp.dpre = reinterpret_cast<const uint32_t*>(sp.inv + a.k);
  sp.tinfo = reinterpret_cast<const uint2*>(a.headers + bivf_tinfo_word(a.k, a.dim, sp.nblk));
  if (a.doc_freq) {
    // V = sum_t no_t * nc_t (counters.py:71-81 regrouped by term): one pass
    // over the D terms instead of a posting-count gather per object entry
    sp.count_post = 0;
    postings_dot_kernel<<<grid_for(a.dim, 256, num_sms() * 4), 256, 0, st>>>(a.dim, a.doc_freq,
                                                                            sp.nc, a.stats);
    IVFKM_CHECK_LAUNCH();
  }
  sp.order = a.order;
  sp.pv32 = static_cast<const float*>(a.pval_screen);
  sp.half = a.screen_bits == 16;
  sp.mu_max = a.mu_max > 0 ? a.mu_max : 1.0;
  sp.cta_blocks = pl.cta_blocks;
  sp.nsplit = pl.nsplit;
  sp.rowcap = pl.rowcap;
  sp.cc_bytes = (int)pl.cc_bytes;
  sp.label32 = w.label32;
  sp.slot_of = w.slot_of;
  sp.q_obj = w.q_obj;
  sp.q_cnt = w.q_cnt;
  sp.q_cid = w.q_cid;
  sp.stats = a.stats;
  if (pl.passes && can_presort && (pl.cta_blocks / pl.rr) > 0) {
    const int nsp = (int)(ivfkm_bivf_nblk(a.k) / kSpan);
    int2* pt = reinterpret_cast<int2*>(a.ps_t);
    int2* pvv = reinterpret_cast<int2*>(a.ps_v);
    presort_rows_kernel<<<grid_for(a.n_obj, 8), 256, 0, st>>>(
        a.n_obj, a.row_ptr, a.terms, a.val32, sp.dpre, sp.tinfo, nsp, pt, pvv);
    IVFKM_CHECK_LAUNCH();
    sp.ps_t = pt;
    sp.ps_v = pvv;
  }
  if (a.screen_bits == 16 && pl.rr == 8 && a.slot8) {
    // [span offsets][slot bytes] (bivf.cuh, bivf_soff_bytes)
    sp.soff = reinterpret_cast<const uint32_t*>(a.slot8);
    sp.slot8 = a.slot8 + bivf_soff_bytes(a.dim, sp.nblk);
    sp.nsp1 = (int)(sp.nblk / kSpan + 1);
  }
  sp.st_best = w.st_best;
  sp.st_slot = w.st_slot;
  sp.st_cnt = w.st_cnt;
  sp.st_cand = w.st_cand;
  switch (pl.rr) {
    case 8: return launch_screen<8>(pl, sp, st);
    case 4: return launch_screen<4>(pl, sp, st);
    default: return launch_screen<2>(pl, sp, st);
  }
}

// Rank directory of the means' mean-major CSR (ivfkm.h, ivfkm_assign_finish_dir).
int rankdir_build(int64_t k, int64_t dim, const int64_t* m_ptr, const int32_t* m_terms, uint2* dir,
                  cudaStream_t st) {
  const int T = 256;
  const int64_t nw = (dim + 31) / 32;
  IVFKM_TRY(cudaMemsetAsync(dir, 0, sizeof(uint2) * k * nw, st));
  rankdir_bits_kernel<<<num_sms() * 8, T, 0, st>>>(k, nw, m_ptr, m_terms, dir);
  IVFKM_CHECK_LAUNCH();
  rankdir_scan_kernel<<<grid_for(k, T / 32), T, 0, st>>>(k, nw, dir);
  IVFKM_CHECK_LAUNCH();
  return IVFKM_OK;
}

int finish_impl(const AssignArgs& a, const AssignWs& w, const int32_t* prev_labels,
                int32_t* labels, double* sims, unsigned long long* sizes, int rule,
                cudaStream_t st, const int64_t* m_ptr = nullptr, const int32_t* m_terms = nullptr,
                const double* m_vals = nullptr, uint2* dir = nullptr) {
  FinalParams fp;
  const int T = 256;
  const int64_t nw = (a.dim + 31) / 32;
  if (dir) {
    // m_terms == nullptr: the caller built the directory for these means
    // already (ivfkm_rankdir_build, e.g. on another stream during the screen)
    if (m_terms) {
      if (int rc = rankdir_build(a.k, a.dim, m_ptr, m_terms, dir, st)) return rc;
    }
    IVFKM_TRY(cudaMemsetAsync(w.cl_pos, 0, sizeof(unsigned int) * (a.k + 1), st));
    winner_hist_kernel<<<grid_for(a.n_obj, T), T, 0, st>>>(a.n_obj, w.label32, w.cl_pos);
    IVFKM_CHECK_LAUNCH();
    size_t cb = w.cub_bytes;
    IVFKM_TRY(cub::DeviceScan::ExclusiveSum(w.cub, cb, w.cl_pos, w.cl_pos, (int)(a.k + 1), st));
    winner_scatter_kernel<<<grid_for(a.n_obj, T), T, 0, st>>>(a.n_obj, w.label32, w.cl_pos,
                                                             w.fin_order);
    IVFKM_CHECK_LAUNCH();
    fp.order = w.fin_order;
  }
  fp.n_obj = a.n_obj;
  fp.rule = rule;
  fp.x.row_ptr = a.row_ptr;
  fp.x.terms = a.terms;
  fp.x.val64 = a.val64;
  fp.x.bv = exact_view(a.headers, a.k, a.dim);
  fp.x.pv64 = a.pval64;
  if (dir) {
    fp.x.dir = dir;
    fp.x.m_ptr = m_ptr;
    fp.x.m_vals = m_vals;
    fp.x.nw = nw;
  }
  fp.label32 = w.label32;
  fp.slot_of = w.slot_of;
  fp.q_cnt = w.q_cnt;
  fp.q_cid = w.q_cid;
  fp.labels = labels;
  fp.sims = sims;
  fp.ovf_list = w.ovf_list;
  fp.ovf_len = w.ovf_len;
  finalize_kernel<<<grid_for(a.n_obj, 8), 256, 0, st>>>(fp);
  IVFKM_CHECK_LAUNCH();
  overflow_kernel<<<num_sms(), 1024, 0, st>>>(fp, a.k);
  IVFKM_CHECK_LAUNCH();
  accumulate_kernel<<<grid_for(a.n_obj, 256, num_sms() * 8), 256, 0, st>>>(
      a.n_obj, labels, sims, prev_labels, sizes, a.stats);
  IVFKM_CHECK_LAUNCH();
  return IVFKM_OK;
}

}  // namespace

extern "C" int ivfkm_assign_screen_ex(int64_t n_obj, const int64_t* row_ptr,
                                      const int32_t* terms, const float* val32,
                                      const double* xnorm, int64_t k, int64_t dim,
                                      const uint32_t* headers, const void* pval_screen,
                                      int screen_bits, double mu_max, ivfkm_stats* stats,
                                      const int32_t* order, int32_t* presort_terms,
                                      float* presort_vals, const uint8_t* slot8,
                                      const uint32_t* doc_freq, void* ws, size_t ws_bytes,
                                      ivfkm_stream_t stream_);

extern "C" int ivfkm_assign_screen(int64_t n_obj, const int64_t* row_ptr, const int32_t* terms,
                                   const float* val32, const double* xnorm, int64_t k,
                                   int64_t dim, const uint32_t* headers, const void* pval_screen,
                                   int screen_bits, double mu_max, ivfkm_stats* stats,
                                   const int32_t* order, void* ws, size_t ws_bytes,
                                   ivfkm_stream_t stream_) {
  return ivfkm_assign_screen_ex(n_obj, row_ptr, terms, val32, xnorm, k, dim, headers,
                                pval_screen, screen_bits, mu_max, stats, order, nullptr, nullptr,
                                nullptr, nullptr, ws, ws_bytes, stream_);
}

extern "C" int ivfkm_assign_screen_ex(int64_t n_obj, const int64_t* row_ptr,
                                      const int32_t* terms, const float* val32,
                                      const double* xnorm, int64_t k, int64_t dim,
                                      const uint32_t* headers, const void* pval_screen,
                                      int screen_bits, double mu_max, ivfkm_stats* stats,
                                      const int32_t* order, int32_t* presort_terms,
                                      float* presort_vals, const uint8_t* slot8,
                                      const uint32_t* doc_freq, void* ws, size_t ws_bytes,
                                      ivfkm_stream_t stream_) {
  if (n_obj < 0 || k < 1 || dim < 1 || !row_ptr || !stats || !headers) return IVFKM_E_ARG;
  if (screen_bits != 32 && screen_bits != 16) return IVFKM_E_ARG;
  // fp16 holds mean values up to 65504; unit-norm means are far inside
  if (screen_bits == 16 && !(mu_max <= 32768.0)) return IVFKM_E_UNSUPPORTED;
  if (n_obj > INT32_MAX || k > INT32_MAX) return IVFKM_E_UNSUPPORTED;
  size_t need = 0;
  AssignWs w = carve_assign(ws, n_obj, k, &need);
  if (ws_bytes < need) return IVFKM_E_WORKSPACE;
  cudaStream_t st = as_stream(stream_);
  IVFKM_TRY(cudaMemsetAsync(stats, 0, sizeof(ivfkm_stats), st));
  IVFKM_TRY(cudaMemsetAsync(w.ovf_len, 0, sizeof(unsigned int), st));
  if (n_obj == 0) return IVFKM_OK;
  AssignArgs a{n_obj,   row_ptr,     terms,       val32,   nullptr, xnorm, k, dim,
               headers, pval_screen, screen_bits, nullptr, mu_max,  stats, order};
  a.ps_t = presort_terms;
  a.ps_v = presort_vals;
  a.slot8 = slot8;
  a.doc_freq = doc_freq;
  return screen_impl(a, w, st);
}

// Objects per term (the document frequencies no_p of data.py:200-211) as the
// screen's posting counter reads them.
namespace {
__global__ void doc_freq_kernel(int64_t nnz, const int32_t* __restrict__ terms, int64_t dim,
                                unsigned int* __restrict__ df) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < nnz;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int32_t t = terms[e];
    if (t >= 0 && t < dim) atomicAdd(&df[t], 1u);
  }
}
}  // namespace

extern "C" int ivfkm_doc_freq(int64_t nnz, const int32_t* terms, int64_t dim, uint32_t* doc_freq,
                              ivfkm_stream_t stream_) {
  if (nnz < 0 || dim < 1 || !doc_freq || (nnz > 0 && !terms)) return IVFKM_E_ARG;
  cudaStream_t st = as_stream(stream_);
  IVFKM_TRY(cudaMemsetAsync(doc_freq, 0, sizeof(uint32_t) * dim, st));
  if (nnz == 0) return IVFKM_OK;
  doc_freq_kernel<<<grid_for(nnz, 256), 256, 0, st>>>(nnz, terms, dim, doc_freq);
  IVFKM_CHECK_LAUNCH();
  return IVFKM_OK;
}

extern "C" int ivfkm_assign_finish(int64_t n_obj, const int64_t* row_ptr, const int32_t* terms,
                                   const double* val64, int64_t k, int64_t dim,
                                   const uint32_t* headers, const double* pval64,
                                   const int32_t* prev_labels, int32_t* labels, double* sims,
                                   unsigned long long* sizes, ivfkm_stats* stats, int label_rule,
                                   void* ws, size_t ws_bytes, ivfkm_stream_t stream_) {
  if (n_obj < 0 || k < 1 || dim < 1 || !row_ptr || !labels || !sims || !stats || !headers)
    return IVFKM_E_ARG;
  if (label_rule != 0 && label_rule != 1) return IVFKM_E_ARG;
  size_t need = 0;
  AssignWs w = carve_assign(ws, n_obj, k, &need);
  if (ws_bytes < need) return IVFKM_E_WORKSPACE;
  cudaStream_t st = as_stream(stream_);
  if (sizes) IVFKM_TRY(cudaMemsetAsync(sizes, 0, sizeof(unsigned long long) * k, st));
  if (n_obj == 0) return IVFKM_OK;
  AssignArgs a{n_obj,   row_ptr, terms, nullptr, val64, nullptr, k,      dim,
               headers, nullptr, 32,    pval64,  0.0,   stats,   nullptr};
  return finish_impl(a, w, prev_labels, labels, sims, sizes, label_rule, st);
}

extern "C" int ivfkm_assign_finish_dir(int64_t n_obj, const int64_t* row_ptr,
                                       const int32_t* terms, const double* val64, int64_t k,
                                       int64_t dim, const uint32_t* headers, const double* pval64,
                                       const int64_t* m_ptr, const int32_t* m_terms,
                                       const double* m_vals, void* dir, const int32_t* prev_labels,
                                       int32_t* labels, double* sims, unsigned long long* sizes,
                                       ivfkm_stats* stats, int label_rule, void* ws,
                                       size_t ws_bytes, ivfkm_stream_t stream_) {
  if (n_obj < 0 || k < 1 || dim < 1 || !row_ptr || !labels || !sims || !stats || !headers)
    return IVFKM_E_ARG;
  if (!m_ptr || !m_vals || !dir) return IVFKM_E_ARG;  // m_terms NULL: dir is prebuilt
  if (label_rule != 0 && label_rule != 1) return IVFKM_E_ARG;
  size_t need = 0;
  AssignWs w = carve_assign(ws, n_obj, k, &need);
  if (ws_bytes < need) return IVFKM_E_WORKSPACE;
  cudaStream_t st = as_stream(stream_);
  if (sizes) IVFKM_TRY(cudaMemsetAsync(sizes, 0, sizeof(unsigned long long) * k, st));
  if (n_obj == 0) return IVFKM_OK;
  AssignArgs a{n_obj,   row_ptr, terms, nullptr, val64, nullptr, k,      dim,
               headers, nullptr, 32,    pval64,  0.0,   stats,   nullptr};
  return finish_impl(a, w, prev_labels, labels, sims, sizes, label_rule, st, m_ptr, m_terms,
                     m_vals, static_cast<uint2*>(dir));
}

extern "C" int ivfkm_rankdir_build(int64_t k, int64_t dim, const int64_t* m_ptr,
                                   const int32_t* m_terms, void* dir, ivfkm_stream_t stream_) {
  if (k < 1 || dim < 1 || !m_ptr || !m_terms || !dir) return IVFKM_E_ARG;
  return rankdir_build(k, dim, m_ptr, m_terms, static_cast<uint2*>(dir), as_stream(stream_));
}

extern "C" int ivfkm_assign(int64_t n_obj, const int64_t* row_ptr, const int32_t* terms,
                            const float* val32, const double* val64, const double* xnorm,
                            int64_t k, int64_t dim, const uint32_t* headers,
                            const void* pval_screen, int screen_bits, const double* pval64,
                            double mu_max, const int32_t* prev_labels,
                            int32_t* labels, double* sims, unsigned long long* sizes,
                            ivfkm_stats* stats, const int32_t* order, int label_rule, void* ws,
                            size_t ws_bytes, ivfkm_stream_t stream_) {
  int rc = ivfkm_assign_screen(n_obj, row_ptr, terms, val32, xnorm, k, dim, headers,
                               pval_screen, screen_bits, mu_max, stats, order, ws, ws_bytes,
                               stream_);
  if (rc) return rc;
  return ivfkm_assign_finish(n_obj, row_ptr, terms, val64, k, dim, headers, pval64, prev_labels,
                             labels, sims, sizes, stats, label_rule, ws, ws_bytes, stream_);
}

extern "C" int ivfkm_score_labels(int64_t n_obj, const int64_t* row_ptr, const int32_t* terms,
                                  const double* val64, int64_t k, int64_t dim,
                                  const uint32_t* headers, const double* pval64,
                                  const int32_t* labels, double* sims, ivfkm_stats* stats,
                                  ivfkm_stream_t stream_) {
  if (n_obj < 0 || k < 1 || dim < 1 || !row_ptr || !labels || !sims || !stats) return IVFKM_E_ARG;
  cudaStream_t st = as_stream(stream_);
  IVFKM_TRY(cudaMemsetAsync(stats, 0, sizeof(ivfkm_stats), st));
  if (n_obj == 0) return IVFKM_OK;
  ExactCtx x;
  x.row_ptr = row_ptr;
  x.terms = terms;
  x.val64 = val64;
  x.bv = exact_view(headers, k, dim);
  x.pv64 = pval64;
  score_labels_kernel<<<grid_for(n_obj, 8), 256, 0, st>>>(n_obj, x, labels, sims);
  IVFKM_CHECK_LAUNCH();
  accumulate_kernel<<<grid_for(n_obj, 256, num_sms() * 8), 256, 0, st>>>(n_obj, labels, sims, nullptr,
                                                                      nullptr, stats);
  IVFKM_CHECK_LAUNCH();
  return IVFKM_OK;
}

// ---------------------------------------------------------------------------
// IVFD, object-inverted (see ivfd_scatter_kernel).

extern "C" size_t ivfkm_objects_inverted_workspace_size(int64_t nnz, int64_t dim) {
  size_t sb = 0;
  cub::DoubleBuffer<int32_t> kb(nullptr, nullptr), vb(nullptr, nullptr);
  cub::DeviceRadixSort::SortPairs(nullptr, sb, kb, vb, (int)nnz);
  size_t sc = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, sc, (unsigned int*)nullptr, (int64_t*)nullptr,
                                (int)dim + 1);
  Carver c(nullptr);
  for (int q = 0; q < 5; ++q) c.take<int32_t>((size_t)(nnz > 0 ? nnz : 1));
  c.take<unsigned int>((size_t)dim + 1);
  c.take_bytes(sb > sc ? sb : sc);
  return c.off;
}

extern "C" int ivfkm_objects_inverted(int64_t n_obj, int64_t nnz, int64_t dim,
                                      const int64_t* row_ptr, const int32_t* terms,
                                      const double* val64, int64_t* x_ptr, int32_t* x_obj,
                                      double* x_val, void* ws, size_t ws_bytes,
                                      ivfkm_stream_t stream_) {
  if (n_obj < 0 || nnz < 0 || dim < 1 || !x_ptr) return IVFKM_E_ARG;
  if (n_obj > INT32_MAX || nnz > INT32_MAX) return IVFKM_E_UNSUPPORTED;
  if (ws_bytes < ivfkm_objects_inverted_workspace_size(nnz, dim)) return IVFKM_E_WORKSPACE;
  cudaStream_t st = as_stream(stream_);
  size_t sb = 0;
  {
    cub::DoubleBuffer<int32_t> kb(nullptr, nullptr), vb(nullptr, nullptr);
    cub::DeviceRadixSort::SortPairs(nullptr, sb, kb, vb, (int)nnz);
  }
  size_t sc = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, sc, (unsigned int*)nullptr, (int64_t*)nullptr,
                                (int)dim + 1);
  Carver c(ws);
  const size_t nz = (size_t)(nnz > 0 ? nnz : 1);
  int32_t* k0 = c.take<int32_t>(nz);
  int32_t* k1 = c.take<int32_t>(nz);
  int32_t* i0 = c.take<int32_t>(nz);
  int32_t* i1 = c.take<int32_t>(nz);
  int32_t* ob = c.take<int32_t>(nz);
  unsigned int* hist = c.take<unsigned int>((size_t)dim + 1);
  void* tmp = c.take_bytes(sb > sc ? sb : sc);
  IVFKM_TRY(cudaMemsetAsync(hist, 0, sizeof(unsigned int) * (dim + 1), st));
  if (nnz > 0) {
    entry_keys_kernel<<<grid_for(n_obj, 8), 256, 0, st>>>(n_obj, row_ptr, terms, k0, ob, i0,
                                                          hist);
    IVFKM_CHECK_LAUNCH();
    cub::DoubleBuffer<int32_t> kb(k0, k1), vb(i0, i1);
    int bits = 1;
    while (bits < 31 && (1ll << bits) < dim) ++bits;
    IVFKM_TRY(cub::DeviceRadixSort::SortPairs(tmp, sb, kb, vb, (int)nnz, 0, bits, st));
    entry_gather_kernel<<<grid_for(nnz, 256), 256, 0, st>>>(nnz, vb.Current(), ob, val64, x_obj,
                                                            x_val);
    IVFKM_CHECK_LAUNCH();
  }
  IVFKM_TRY(cub::DeviceScan::ExclusiveSum(tmp, sc, hist, x_ptr, (int)dim + 1, st));
  return IVFKM_OK;
}

extern "C" size_t ivfkm_ivfd_workspace_size(int64_t n_obj, int64_t wave) {
  Carver c(nullptr);
  const size_t n = (size_t)(n_obj > 0 ? n_obj : 1);
  c.take<double>(n * (size_t)(wave > 0 ? wave : 1));
  c.take<double>(n);
  c.take<int32_t>(n);
  c.take<double>(n);
  return c.off;
}

extern "C" int ivfkm_assign_ivfd(int64_t n_obj, int64_t dim, const int64_t* x_ptr,
                                 const int32_t* x_obj, const double* x_val, int64_t k,
                                 const int64_t* m_ptr, const int32_t* m_terms,
                                 const double* m_vals, const int32_t* prev_labels,
                                 int32_t* labels, double* sims, unsigned long long* sizes,
                                 ivfkm_stats* stats, int64_t wave, void* ws, size_t ws_bytes,
                                 ivfkm_stream_t stream_) {
  if (n_obj < 0 || dim < 1 || k < 1 || wave < 1 || !x_ptr || !m_ptr || !labels || !sims ||
      !stats)
    return IVFKM_E_ARG;
  if (n_obj > INT32_MAX || k > INT32_MAX) return IVFKM_E_UNSUPPORTED;
  if (ws_bytes < ivfkm_ivfd_workspace_size(n_obj, wave)) return IVFKM_E_WORKSPACE;
  cudaStream_t st = as_stream(stream_);
  IVFKM_TRY(cudaMemsetAsync(stats, 0, sizeof(ivfkm_stats), st));
  if (sizes) IVFKM_TRY(cudaMemsetAsync(sizes, 0, sizeof(unsigned long long) * k, st));
  if (n_obj == 0) return IVFKM_OK;
  Carver c(ws);
  const size_t n = (size_t)n_obj;
  double* slots = c.take<double>(n * (size_t)wave);
  double* best = c.take<double>(n);
  int32_t* label = c.take<int32_t>(n);
  double* sim0 = c.take<double>(n);
  IVFKM_TRY(cudaMemsetAsync(slots, 0, sizeof(double) * n * (size_t)wave, st));
  for (int64_t j0 = 0; j0 < k; j0 += wave) {
    const int64_t m = k - j0 < wave ? k - j0 : wave;
    ivfd_scatter_kernel<<<(unsigned)m, 256, 0, st>>>(n_obj, j0, k, x_ptr, x_obj, x_val, m_ptr,
                                                      m_terms, m_vals, slots, &stats->postings);
    IVFKM_CHECK_LAUNCH();
    ivfd_reduce_kernel<<<grid_for(n_obj, 256), 256, 0, st>>>(n_obj, j0, m, slots, best, label,
                                                              sim0);
    IVFKM_CHECK_LAUNCH();
  }
  ivfd_finish_kernel<<<grid_for(n_obj, 256), 256, 0, st>>>(n_obj, best, label, sim0, labels, sims);
  IVFKM_CHECK_LAUNCH();
  accumulate_kernel<<<grid_for(n_obj, 256, num_sms() * 8), 256, 0, st>>>(
      n_obj, labels, sims, prev_labels, sizes, stats);
  IVFKM_CHECK_LAUNCH();
  return IVFKM_OK;
}
