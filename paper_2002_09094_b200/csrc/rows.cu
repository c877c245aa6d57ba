// Object rows shipped to the device in a compact form: each row's sorted
// 0-based term ids as 16-bit gaps (first gap = t0 + 1, later ones
// t[h] - t[h-1] >= 1), gaps that do not fit (>= 0xFFFF) marked 0xFFFF with the
// absolute id in a short exception list.  The end-to-end path streams the
// corpus every step over PCIe, which binds it; 2 bytes per term instead of 4
// cut the step's host->device bytes by a sixth.  ivfkm_rows_decode restores
// the int32 ids bit for bit (the decode is integer work).

#include <cstdint>

#include "common.cuh"
#include "ivfkm.h"

using namespace ivfkm;

namespace {

constexpr uint16_t kEsc = 0xFFFFu;

// One warp per row: a segmented inclusive scan of the gaps in 32-entry
// chunks (an exception restarts the sum at its absolute id), carried across
// chunks.
__global__ void __launch_bounds__(256) rows_decode_kernel(
    int64_t n_obj, const int64_t* __restrict__ row_ptr, const uint16_t* __restrict__ gaps,
    int64_t n_exc, const int64_t* __restrict__ exc_idx, const int32_t* __restrict__ exc_term,
    int32_t* __restrict__ terms) {
  const int lane = threadIdx.x & 31;
  const int64_t wpb = blockDim.x >> 5;
  for (int64_t i = blockIdx.x * wpb + (threadIdx.x >> 5); i < n_obj; i += gridDim.x * wpb) {
    const int64_t rb = row_ptr[i], re = row_ptr[i + 1];
    int32_t carry = -1;  // the id before the row's first entry
    for (int64_t h0 = rb; h0 < re; h0 += 32) {
      const int64_t h = h0 + lane;
      int32_t v = 0;
      int abs_ = 0;
      if (h < re) {
        const uint16_t g = gaps[h];
        if (g == kEsc) {
          int64_t lo = 0, hi = n_exc;  // exc_idx ascending
          while (lo < hi) {
            const int64_t mid = (lo + hi) >> 1;
            if (exc_idx[mid] < h) lo = mid + 1; else hi = mid;
          }
          v = exc_term[lo];
          abs_ = 1;
        } else {
          v = (int32_t)g;
        }
      }
      // segmented inclusive scan: (v, abs) . (w, abs') = abs' ? (w, 1) : (v + w, abs)
#pragma unroll
      for (int off = 1; off < 32; off <<= 1) {
        const int32_t pv = __shfl_up_sync(kFull, v, off);
        const int pa = __shfl_up_sync(kFull, abs_, off);
        if (lane >= off && !abs_) {
          v += pv;
          abs_ = pa;
        }
      }
      const int32_t t = abs_ ? v : carry + v;
      if (h < re) terms[h] = t;
      carry = __shfl_sync(kFull, t, 31);
    }
  }
}

// One warp per row: the reference's 1-based term ids -> 0-based, the fp32
// screen copy of the values, and the row norm (used only inside the screen's
// error bound, which carries a relative margin far above the order-dependent
// last bits of this sum).
__global__ void __launch_bounds__(256) rows_prepare_kernel(
    int64_t n_obj, const int64_t* __restrict__ row_ptr, const int32_t* __restrict__ terms1,
    const double* __restrict__ val64, int32_t* __restrict__ terms0, float* __restrict__ val32,
    double* __restrict__ xnorm) {
  const int lane = threadIdx.x & 31;
  const int64_t wpb = blockDim.x >> 5;
  for (int64_t i = blockIdx.x * wpb + (threadIdx.x >> 5); i < n_obj; i += gridDim.x * wpb) {
    const int64_t rb = row_ptr[i], re = row_ptr[i + 1];
    double ss = 0.0;
    for (int64_t h = rb + lane; h < re; h += 32) {
      const double v = val64[h];
      terms0[h] = terms1[h] - 1;
      val32[h] = (float)v;
      ss = fma(v, v, ss);
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) ss += __shfl_xor_sync(kFull, ss, off);
    if (lane == 0) xnorm[i] = sqrt(ss);
  }
}

}  // namespace

extern "C" int ivfkm_rows_prepare(int64_t n_obj, const int64_t* row_ptr, const int32_t* terms1,
                                  const double* val64, int32_t* terms0, float* val32,
                                  double* xnorm, ivfkm_stream_t stream_) {
  if (n_obj < 0 || (n_obj > 0 && (!row_ptr || !terms1 || !val64 || !terms0 || !val32 || !xnorm)))
    return IVFKM_E_ARG;
  if (n_obj == 0) return IVFKM_OK;
  cudaStream_t st = as_stream(stream_);
  rows_prepare_kernel<<<grid_for(n_obj, 8), 256, 0, st>>>(n_obj, row_ptr, terms1, val64, terms0,
                                                          val32, xnorm);
  IVFKM_CHECK_LAUNCH();
  return IVFKM_OK;
}

extern "C" int ivfkm_rows_decode(int64_t n_obj, const int64_t* row_ptr, const uint16_t* gaps,
                                 int64_t n_exc, const int64_t* exc_idx, const int32_t* exc_term,
                                 int32_t* terms, ivfkm_stream_t stream_) {
  if (n_obj < 0 || n_exc < 0 || (n_obj > 0 && (!row_ptr || !terms))) return IVFKM_E_ARG;
  if (n_exc > 0 && (!exc_idx || !exc_term)) return IVFKM_E_ARG;
  if (n_obj == 0) return IVFKM_OK;
  cudaStream_t st = as_stream(stream_);
  rows_decode_kernel<<<grid_for(n_obj, 8), 256, 0, st>>>(n_obj, row_ptr, gaps, n_exc, exc_idx,
                                                         exc_term, terms);
  IVFKM_CHECK_LAUNCH();
  return IVFKM_OK;
}
