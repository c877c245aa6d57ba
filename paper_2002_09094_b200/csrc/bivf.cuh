// Bitmap-block inverted file (BIVF): layout constants and the O(1) lookup
// shared by the build, the fp32 screen and the exact fp64 rescoring.
//
// Mean ids inside the BIVF are *slots*: slot = perm[mean], means sorted by
// their number of terms (descending) so that the postings of mid-frequency
// terms crowd into the low slots and fill whole spans.  Results are mapped
// back (inv[slot] = mean) before any tie is broken, so the order is invisible
// outside (ties are always rescored exactly, see assign.cu).
//
// headers (uint32), planar:
//   masks[t*nblk + b]        bit j <=> slot 32*b+j holds term t
//   offs [t*nblk + b]        start of block b's values (+ kDense flag)
//   offs [dim*nblk]          padded total (size of the screen-value array)
//   nc   [t]                 postings of term t (= centroid_freq, means.py:144-147)
//   perm [k], inv [k]        mean -> slot, slot -> mean
//   dpre [t]                 dense prefix: t's first dpre[t] spans are all dense,
//                            so their values are one contiguous run — span s at
//                            (offs[t*nblk] & ~kDense) + 256*s — and the screen
//                            reads them without masks or offsets
//   off64[t*nblk + b]        start of block b in the compact exact-value (fp64)
//                            array: postings only, term-major, slot ascending;
//   off64[dim*nblk]          their number
//   mo   [t*nblk + b]        (uint2, at the next even word) {mask, off64}: the
//                            exact lookup's two words in one 8-byte gather
//   tinfo[t]                 (uint2) {offs[t*nblk] & ~kDense, dpre[t] | bit 31
//                            when nc[t] > 0}: the screen's per-entry staging
//                            lookup in one gather
// Screen values: blocks are grouped in spans of 8 (256 slots); every span's
// value segment is padded to a multiple of 8 values, so a span start is 16-B
// aligned in both the fp32 and the fp16 screen arrays.
// A span holding at least dense_fill*256 postings is stored *dense*: all 256
// values (0.0 for absent slots) lane-major in two halves (slot 32*(b0+r)+j at
// span_base + 128*(r/4) + 4*j + r%4), so a warp lane owning slots
// 32*(b0+r)+lane reads its 8 values with two 16-B loads, coalesced in global
// memory and conflict-free in shared memory; every block of a dense span
// carries kDense in its offset.  The zeros are exact no-ops for the FMAs.
// Other spans keep the reference order (term-major, mean ascending,
// means.py:169-179, in slot order).
// The fp16 screen array (screen_bits = 16) uses the same positions except
// inside dense spans, where each lane's 8 values are contiguous (slot
// 32*(b0+r)+j at span_base + 8*j + r: one 16-B load per lane and span).
#pragma once
#include <cstdint>

namespace ivfkm {

constexpr uint32_t kDense = 0x80000000u;
constexpr int kSpan = 8;

// Lookup view for the exact (fp64) values: the compact array holds only the
// postings, term-major and slot-ascending (the reference's order,
// means.py:169-179), so block b of term t starts at off64[t*nblk + b].
struct BivfView {
  int64_t nblk;
  const uint2* mo;      // {mask, off64} per block
  const int32_t* perm;  // mean -> slot (nullptr: identity)
};

__host__ __device__ inline int64_t bivf_nh(int64_t dim, int64_t nblk) { return dim * nblk; }

// Word offset of the mo array in the headers (8-byte aligned).
__host__ __device__ inline int64_t bivf_mo_word(int64_t k, int64_t dim, int64_t nblk) {
  const int64_t nh = bivf_nh(dim, nblk);
  const int64_t w = 2 * nh + 1 + dim + 2 * k + dim + nh + 1;
  return (w + 1) & ~(int64_t)1;
}

// Word offset of tinfo (after mo): per term {start of its dense-prefix run,
// dense prefix} — the screen's staging reads both with one 8-byte gather.
__host__ __device__ inline int64_t bivf_tinfo_word(int64_t k, int64_t dim, int64_t nblk) {
  return bivf_mo_word(k, dim, nblk) + 2 * bivf_nh(dim, nblk);
}

// The slot-byte buffer of the sparse path (ivfkm_bivf_slots) starts with the
// compact span offsets soff[t*(nsp+1) + s] = offs[t*nblk + 8*s] (s = nsp: the
// end of the term's last span): the screen's sparse path reads a span's start
// and end from two adjacent words of a table of dim*(nsp+1) words (23 MB at
// config 3, 133 MB at config 4) instead of two words 32 bytes apart in the
// (term x block) offsets (0.45 / 5.3 GB).  The slot bytes follow, 16-B aligned.
__host__ __device__ inline size_t bivf_soff_bytes(int64_t dim, int64_t nblk) {
  return ((size_t)dim * (size_t)(nblk / kSpan + 1) * 4 + 15) & ~(size_t)15;
}

// Position of slot s's exact value for term t, or -1 when the slot lacks it.
__device__ __forceinline__ int64_t bivf_find_slot(const BivfView& v, int64_t t, int64_t s) {
  const uint32_t bit = 1u << (s & 31);
  const uint2 m = __ldg(v.mo + t * v.nblk + (s >> 5));
  if (!(m.x & bit)) return -1;
  return (int64_t)m.y + __popc(m.x & (bit - 1u));
}

// Position of mean c's exact value for term t, or -1.
__device__ __forceinline__ int64_t bivf_find(const BivfView& v, int64_t t, int64_t c) {
  return bivf_find_slot(v, t, v.perm ? (int64_t)__ldg(v.perm + c) : c);
}

}  // namespace ivfkm
