/*
 * ivfkm.h — C ABI of the B200 (sm_100a) IVF spherical k-means Lloyd path.
 *
 * Drop-in boundary for the hot path of arXiv 2002.09094's reference package
 * `sparse_kmeans` (/root/reference/pkg/src/sparse_kmeans).  Plain pointers,
 * sizes and a cudaStream_t; no torch types.  Every entry point returns 0 on
 * success, a positive cudaError_t, or a negative IVFKM_E_* code
 * (ivfkm_error_string() names it).  [dev] marks device pointers, [host] host
 * pointers.  Ids on the device are 0-based; the reference's 1-based ids are
 * converted only by the host-buffer entry point ivfkm_assign_ivf_host().
 *
 * Reference interfaces replaced (file:line under /root/reference/pkg/src/sparse_kmeans):
 *   ivfkm_assign_ivf_host   <- _kernels.pyx:106-128  assign_ivf(indptr, terms, vals,
 *                              m_indptr, m_cids, m_vals, rho, labels, ctr): the
 *                              kernel-module ABI that kernels.py:23-52 dispatches to
 *   ivfkm_bivf_build        <- means.py:169-179      MeanSet.inverted (term-major postings)
 *   ivfkm_assign            <- variants.py:162-174   assign_ivf, with _kernels.pyx:17-26
 *                              (_argmax_label), clustering.py:105-119 (objective_cosine),
 *                              clustering.py:286 (convergence: changed labels),
 *                              variants.py:56-59 (Assignment sizes) and
 *                              counters.py:71-81 (mult_volume_ivf, counted in-kernel)
 *   ivfkm_update_count/fill <- variants.py:254-312   update_means / update_ivf
 *   ivfkm_fnv1a64           <- variants.py:77-83     fnv1a64 (assignment digest)
 *   ivfkm_synth_*           <- no reference counterpart: seeded stand-ins for the
 *                              BASELINE.json configs (PubMed/NYT are not offline)
 */
#ifndef IVFKM_H
#define IVFKM_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct CUstream_st* ivfkm_stream_t; /* == cudaStream_t */

#define IVFKM_OK 0
#define IVFKM_E_ARG (-1)         /* bad argument / shape                         */
#define IVFKM_E_UNSUPPORTED (-2) /* e.g. k beyond the largest cluster split      */
#define IVFKM_E_CAPACITY (-3)    /* caller output buffer too small               */
#define IVFKM_E_WORKSPACE (-4)   /* workspace smaller than *_workspace_size()    */
#define IVFKM_E_NOGPU (-5)       /* no CUDA device visible                       */
#define IVFKM_E_RANGE (-6)       /* an id outside its range (CorruptionError)    */

#define IVFKM_OBJ_LIMBS 34 /* 32-bit limbs of the exact objective accumulator  */
#define IVFKM_MAXC 32      /* near-tie candidates rescored per object in fp64   */

/* Per-iteration device-side statistics; ivfkm_assign() zeroes them. */
typedef struct ivfkm_stats {
  unsigned long long postings;  /* V = sum_i sum_h nc_{t(i,h)} (counters.py:71-81)  */
  unsigned long long changed;   /* labels != prev_labels (clustering.py:286)        */
  unsigned long long near_ties; /* objects whose fp32 window held >1 candidate      */
  unsigned long long overflow;  /* of those, more than IVFKM_MAXC candidates        */
  unsigned long long queue_len; /* internal: rescoring queue length                 */
  unsigned long long obj_flags; /* nonzero: a similarity fell outside |s| < 8       */
  long long obj_limbs[IVFKM_OBJ_LIMBS]; /* exact sum of sims; limb l weighs 2^(32l-1074) */
} ivfkm_stats;

const char* ivfkm_error_string(int code);
int ivfkm_version(void);
int ivfkm_device_count(void);

/* ---- bitmap-block inverted file (BIVF) of the means ---------------------
 * Means occupy *slots*: slot = perm[mean], means ordered by term count
 * (descending), so mid-frequency postings crowd into whole spans; results
 * are mapped back before any tie is broken.  headers is planar uint32
 * (ivfkm_bivf_headers_size() words):
 *   masks[t*nblk + b]    bit j set <=> slot 32*b+j holds term t
 *   offs[t*nblk + b]     at headers[dim*nblk + t*nblk + b]: start of the block's
 *                        values; bit 31 set = the block's 256-slot span is dense
 *   total                at headers[2*dim*nblk]: padded value count in use
 *   nc[t]                at headers[2*dim*nblk + 1 + t]: postings of term t
 *   perm[k], inv[k]      (int32) after nc: mean -> slot, slot -> mean
 *   dpre[dim], off64[nh+1], then (8-byte aligned) {mask, off64} pairs for the
 *                        exact rescoring (csrc/bivf.cuh has the full layout)
 * Values (val32 for the fp32 screen, val64 for the exact fp64 rescoring) are
 * term-major, slot ascending — the order of MeanSet.inverted
 * (means.py:169-179) — except that each 256-slot span is padded to a multiple
 * of 4 values and a span holding >= dense_fill*256 postings is stored dense
 * and lane-major (slot 32*(b0+r)+j at span_base + 128*(r/4) + 4*j + r%4,
 * exact zeros for absent slots).  The value arrays need
 * ivfkm_bivf_values_capacity() elements.                                     */
int64_t ivfkm_bivf_nblk(int64_t k); /* 32-mean blocks per term, padded */
int64_t ivfkm_bivf_headers_size(int64_t k, int64_t dim);
int64_t ivfkm_bivf_values_capacity(int64_t k, int64_t dim, int64_t nnz);
/* Build options: dense_fill in [1/256, 1] (> 1: never dense; default 1/64),
 * permute = 1 orders slots by mean term count (default), 0 keeps mean ids.
 * Out-of-range values leave the setting unchanged.                          */
void ivfkm_set_bivf_options(float dense_fill, int permute);
size_t ivfkm_bivf_workspace_size(int64_t dim, int64_t k);
/* major = 0: rows of (ptr, cols) are means (mean-major CSR, cols = terms);
 * major = 1: rows are terms (term-major IVF, cols = mean ids).  0-based ids.
 * Screen values: screen_bits = 32 stores them as fp32, 16 as fp16 (half the
 * bytes; the screen's error window widens accordingly, labels stay exact).
 *
 * The exact (fp64) values are stored compactly — postings only, term-major,
 * slot ascending — so val64 holds one value per input entry.
 * Two-step build (exact allocation): ivfkm_bivf_plan writes the headers,
 * synchronises the stream and returns totals = (screen values, exact values)
 * (raising the dense threshold itself if the 31-bit screen-value offsets
 * would overflow; IVFKM_E_RANGE on an out-of-range id); ivfkm_bivf_fill then
 * writes val_screen (totals[0]) and val64 (totals[1]).
 * One-step build: ivfkm_bivf_build = plan + fill without a host round trip,
 * into val_screen of ivfkm_bivf_values_capacity() values and val64 of one
 * value per input entry (ids not checked).                                  */
int ivfkm_bivf_plan(int64_t k, int64_t dim, int major, int64_t nrows,
                    const int64_t* ptr /*[dev] nrows+1*/, const int32_t* cols /*[dev]*/,
                    uint32_t* headers /*[dev]*/, int64_t* totals /*[host] out, 2*/, void* ws,
                    size_t ws_bytes, ivfkm_stream_t stream);
/* fill: with a workspace of ivfkm_bivf_fill_workspace_size(k, dim, nnz)
 * bytes (nnz = input entries) the postings are sorted by position first, so
 * the writes stream; ws = NULL scatters them directly.                      */
/* plan + fill in one call when val_screen / val64 / ws_fill are large enough
 * (screen_cap, val64_cap elements); otherwise IVFKM_E_WORKSPACE with the plan
 * done and totals set, and the caller runs ivfkm_bivf_fill.                 */
int ivfkm_bivf_plan_fill(int64_t k, int64_t dim, int major, int64_t nrows, const int64_t* ptr,
                         const int32_t* cols, const double* vals, uint32_t* headers,
                         int64_t* totals /*[host] out, 2*/, void* val_screen,
                         int64_t screen_cap, int screen_bits, double* val64, int64_t val64_cap,
                         void* ws_plan, size_t ws_plan_bytes, void* ws_fill,
                         size_t ws_fill_bytes, ivfkm_stream_t stream);
size_t ivfkm_bivf_fill_workspace_size(int64_t k, int64_t dim, int64_t nnz);
int ivfkm_bivf_fill(int64_t k, int64_t dim, int major, int64_t nrows,
                    const int64_t* ptr /*[dev]*/, const int32_t* cols /*[dev]*/,
                    const double* vals /*[dev]*/, const uint32_t* headers /*[dev], planned*/,
                    void* val_screen /*[dev]*/, int screen_bits, double* val64 /*[dev]*/,
                    int64_t nnz, void* ws /*or NULL*/, size_t ws_bytes, ivfkm_stream_t stream);
int ivfkm_bivf_build(int64_t k, int64_t dim, int major, int64_t nrows,
                     const int64_t* ptr /*[dev] nrows+1*/, const int32_t* cols /*[dev]*/,
                     const double* vals /*[dev]*/, uint32_t* headers /*[dev]*/,
                     void* val_screen /*[dev]*/, int screen_bits /*32 or 16*/,
                     double* val64 /*[dev]*/, void* ws, size_t ws_bytes, ivfkm_stream_t stream);

/* ---- assignment step ------------------------------------------------------
 * For every object i: rho_i[c] = sum_h x_{i,h} mu_c[t_h] screened in fp32
 * (registers, fixed order), every mean within the rigorous fp32 error window
 * of the best rescored in fp64 in the reference's summation order, label =
 * argmax with the smallest index winning ties (_kernels.pyx:17-26).  Also
 * writes the per-object similarity to the chosen mean (the objective's
 * summand), counts changed labels vs prev_labels, histograms sizes, and
 * accumulates the exact objective into stats->obj_limbs.                      */
size_t ivfkm_assign_workspace_size(int64_t n_obj, int64_t k);
/* Tuning: rowcap = row entries staged in shared memory per pass (default 1024;
 * longer rows run in several passes), smem_limit = shared-memory budget per
 * CTA in bytes (min 1 KB; -1 = adaptive default: rho is split over a
 * thread-block cluster once it passes ~24 KB; a smaller budget forces the thread-block
 * cluster split), rr = 32-mean blocks per warp span of the register screen
 * (2, 4 or 8; 0 = automatic).
 * Out-of-range values leave the setting unchanged.                          */
void ivfkm_set_tuning(int rowcap, int smem_limit, int rr);
/* Tests / tuning: force the register screen's warps per CTA (1..16; 0 = the
 * planned count).  Spans are handed out to warps dynamically, so every count
 * computes identical sums. */
void ivfkm_set_screen_warps(int warps);
/* ivfkm_assign_screen with caller buffers for slot-range passes
 * (presort_terms int32[2*nnz], presort_vals fp32[2*nnz], [dev], 8-byte
 * aligned, or NULL): when the plan runs passes, each row's entries are first
 * sorted by the terms' dense prefix, longest first, into them — per entry
 * {term, dense prefix} and {dense-run start, value} — so that every pass
 * stages its rows by copying, with no per-term lookups.  slot8 (ivfkm_bivf_slots, fp16
 * screens): the sparse spans are read through their slot bytes instead of
 * the block masks.  doc_freq (ivfkm_doc_freq of these rows, [dev] uint32[dim],
 * or NULL): the postings counter is then sum_t doc_freq[t] * nc[t] — one pass
 * over the terms — instead of a posting-count gather per object entry. */
int ivfkm_assign_screen_ex(int64_t n_obj, const int64_t* row_ptr, const int32_t* terms,
                           const float* val32, const double* xnorm, int64_t k, int64_t dim,
                           const uint32_t* headers, const void* pval_screen, int screen_bits,
                           double mu_max, ivfkm_stats* stats, const int32_t* order,
                           int32_t* presort_terms, float* presort_vals,
                           const uint8_t* slot8 /*[dev] or NULL*/,
                           const uint32_t* doc_freq /*[dev] or NULL*/, void* ws, size_t ws_bytes,
                           ivfkm_stream_t stream);
/* Objects per term of a corpus (0-based terms [dev] int32[nnz]) -> doc_freq
 * [dev] uint32[dim] (the reference's Dataset.doc_freq, data.py:200-211). */
int ivfkm_doc_freq(int64_t nnz, const int32_t* terms, int64_t dim, uint32_t* doc_freq,
                   ivfkm_stream_t stream);
/* Screen tuning: which = 1: slot-range passes for the next screens (0 or 1
 * = one pass).  With P > 1 passes the fp16 register screen runs P launches,
 * each over all objects and 1/P of the slots (one CTA per object, no
 * cluster), merging each object's best value and near-tie candidates in a
 * workspace state between launches; the candidate window — and so every
 * result — equals the one-pass screen's.  Ignored under a forced shared-
 * memory budget.  Returns IVFKM_E_ARG
 * for an unknown `which`. */
int ivfkm_set_screen_option(int which, int value);
/* The screen plan ivfkm_assign_screen would use for k means under the
 * current tuning ([host] out[8]: span blocks RR, cluster CTAs per object,
 * 32-mean blocks per CTA, warps per CTA, staged row entries, mode (0 register
 * screen — the only one since round 2), dynamic shared bytes, registers per
 * thread of the instantiation).  rowcap < 32: the current default. */
int ivfkm_screen_plan(int64_t k, int rowcap, int screen_bits, int32_t* out /*[host] 8*/);
/* Object order: ivfkm_assign/_screen take `order`, the order in which the
 * screen visits objects ([dev] permutation of 0..n_obj-1; NULL = natural
 * order).  Results do not depend on it; it only changes load balance and
 * cache locality.  The default order the engine uses: objects by row length, longest first
 * (static longest-processing-time scheduling of the one-CTA-per-object grid). */
size_t ivfkm_row_order_workspace_size(int64_t n_obj);
int ivfkm_row_order(int64_t n_obj, const int64_t* row_ptr /*[dev]*/, int32_t* order /*[dev]*/,
                    void* ws, size_t ws_bytes, ivfkm_stream_t stream);
int ivfkm_assign(int64_t n_obj, const int64_t* row_ptr /*[dev] n+1*/,
                 const int32_t* terms /*[dev]*/, const float* val32 /*[dev]*/,
                 const double* val64 /*[dev]*/, const double* xnorm /*[dev] n or NULL (=1)*/,
                 int64_t k, int64_t dim, const uint32_t* headers /*[dev]*/,
                 const void* pval_screen /*[dev]*/, int screen_bits /*as built*/,
                 const double* pval64 /*[dev]*/, double mu_max,
                 const int32_t* prev_labels /*[dev] n or NULL*/, int32_t* labels /*[dev] n*/,
                 double* sims /*[dev] n*/, unsigned long long* sizes /*[dev] k*/,
                 ivfkm_stats* stats /*[dev]*/, const int32_t* order /*[dev] n or NULL*/,
                 int label_rule, void* ws, size_t ws_bytes, ivfkm_stream_t stream);
/* label_rule 0: IVF — argmax from -inf, smallest index among maximizers
 * (_kernels.pyx:17-26); 1: IVFD — the argmax only if its similarity beats
 * 0.0, else mean 0 (_kernels.pyx:178-207, rho_max starts at 0.0).  The
 * similarities (and so the objective) are the same float64 values for both
 * variants: both add the products in ascending term order.                */

/* The two halves of ivfkm_assign, for callers that time the fp32 screen
 * (the dominant kernel) separately: screen zeroes *stats and fills the
 * workspace's candidate queue; finish rescores, writes labels/sims/sizes and
 * the objective.  Use the same workspace for both.                          */
int ivfkm_assign_screen(int64_t n_obj, const int64_t* row_ptr, const int32_t* terms,
                        const float* val32, const double* xnorm, int64_t k, int64_t dim,
                        const uint32_t* headers, const void* pval_screen, int screen_bits,
                        double mu_max,
                        ivfkm_stats* stats, const int32_t* order, void* ws, size_t ws_bytes,
                        ivfkm_stream_t stream);
int ivfkm_assign_finish(int64_t n_obj, const int64_t* row_ptr, const int32_t* terms,
                        const double* val64, int64_t k, int64_t dim, const uint32_t* headers,
                        const double* pval64, const int32_t* prev_labels, int32_t* labels,
                        double* sims, unsigned long long* sizes, ivfkm_stats* stats,
                        int label_rule, void* ws, size_t ws_bytes, ivfkm_stream_t stream);

/* finish, rescoring through the means' mean-major CSR (m_ptr[k+1], 0-based
 * m_terms, m_vals — the same means as headers/pval64) instead of the BIVF:
 * builds a rank directory in dir (k * ceil(dim/32) uint2: the mean's term
 * bits per 32-term word + the rank of the word's first term in the mean's
 * row) and rescores the objects grouped by their screen winner, so that
 * concurrently resident warps read a few means' contiguous values.  Same
 * results bit for bit.  m_terms == NULL: dir already holds these means'
 * directory (ivfkm_rankdir_build — the directory depends on the means only,
 * so it can be built on another stream while the screen runs).              */
int ivfkm_assign_finish_dir(int64_t n_obj, const int64_t* row_ptr, const int32_t* terms,
                            const double* val64, int64_t k, int64_t dim, const uint32_t* headers,
                            const double* pval64, const int64_t* m_ptr, const int32_t* m_terms,
                            const double* m_vals, void* dir /*[dev] k*ceil(dim/32)*8 B*/,
                            const int32_t* prev_labels, int32_t* labels, double* sims,
                            unsigned long long* sizes, ivfkm_stats* stats, int label_rule,
                            void* ws, size_t ws_bytes, ivfkm_stream_t stream);

/* The rank directory ivfkm_assign_finish_dir rescoring reads, alone: dir
 * (k * ceil(dim/32) * 8 bytes) from the means' CSR structure (m_ptr[k+1],
 * 0-based m_terms ascending per mean; entries past m_ptr[k] are not read).  */
int ivfkm_rankdir_build(int64_t k, int64_t dim, const int64_t* m_ptr, const int32_t* m_terms,
                        void* dir /*[dev]*/, ivfkm_stream_t stream);

/* Exact float64 similarity of every object to the mean its (0-based) label
 * names — the summand of objective_cosine (clustering.py:105-119) — written
 * to sims, with the exact sum accumulated into stats->obj_limbs (stats is
 * zeroed first).                                                            */
int ivfkm_score_labels(int64_t n_obj, const int64_t* row_ptr, const int32_t* terms,
                       const double* val64, int64_t k, int64_t dim, const uint32_t* headers,
                       const double* pval64, const int32_t* labels, double* sims,
                       ivfkm_stats* stats, ivfkm_stream_t stream);

/* ---- update step (variants.py:254-312), bit-identical to the reference ---
 * count: sort member entries by (cluster, term) keeping object order, sum
 * each (cluster, term) run in float64 in ascending object order, divide by
 * the cluster size, take numpy's pairwise sum of squares for the norm, and
 * write new_ptr[0..k] (new_ptr[k] = total nonzeros).  Empty clusters keep
 * their previous mean (retained).  fill: write the mean-major CSR.
 * The workspace must be the same buffer for the count and fill calls.       */
size_t ivfkm_update_workspace_size(int64_t n_obj, int64_t nnz, int64_t k, int64_t dim);
int ivfkm_update_count(int64_t n_obj, int64_t nnz, const int64_t* row_ptr,
                       const int32_t* terms, const double* val64, int64_t k, int64_t dim,
                       const int32_t* labels /*[dev] 0-based*/,
                       const unsigned long long* sizes /*[dev] k*/,
                       const int64_t* prev_ptr /*[dev] k+1*/, int64_t* new_ptr /*[dev] k+1*/,
                       void* ws, size_t ws_bytes, ivfkm_stream_t stream);
/* count with a label-delta sort: `state` keeps the previous iteration's
 * sorted (cluster, term, object) entries and is updated by removing the
 * objects whose label changed and merging their re-keyed entries back in
 * (one full sort when more than a quarter of the entries move).  Same
 * results as ivfkm_update_count, bit for bit.  The state belongs to ONE
 * corpus (row_ptr/terms/val64 contents): zero-fill it before first use and
 * whenever the corpus changes.  state_size returns 0 when the composite key
 * (log2 N + log2 D + log2 k bits) does not fit 64 bits.                      */
size_t ivfkm_update_state_size(int64_t n_obj, int64_t nnz, int64_t k, int64_t dim);
int ivfkm_update_count_delta(int64_t n_obj, int64_t nnz, const int64_t* row_ptr,
                             const int32_t* terms, const double* val64, int64_t k, int64_t dim,
                             const int32_t* labels, const unsigned long long* sizes,
                             const int64_t* prev_ptr, int64_t* new_ptr, void* ws,
                             size_t ws_bytes, void* state /*[dev] zero-filled first*/,
                             size_t state_bytes, ivfkm_stream_t stream);
/* Update tuning: which = 1: the label-delta sort's merge (0 = one fused
 * merge with deletions, the default; 1 = two stable CUB selects + a CUB
 * merge).  Both give the same sorted state.  IVFKM_E_ARG for an unknown
 * `which`. */
int ivfkm_set_update_option(int which, int value);
/* fill: `capacity` = entries new_terms/new_vals hold.  Size them by the
 * exact count new_ptr[k] (read after count) or by the bound
 * min(nnz + prev_ptr[k], k * dim) (runs <= nnz, plus retained means'
 * postings); writes at positions >= capacity are dropped, never performed. */
int ivfkm_update_fill(int64_t n_obj, int64_t nnz, int64_t k, int64_t dim,
                      const unsigned long long* sizes, const int64_t* prev_ptr,
                      const int32_t* prev_terms, const double* prev_vals,
                      const int64_t* new_ptr, int32_t* new_terms /*[dev]*/,
                      double* new_vals /*[dev]*/, uint8_t* retained /*[dev] k*/,
                      int64_t capacity, void* ws, size_t ws_bytes, ivfkm_stream_t stream);

/* Slot bytes of the BIVF's sparse spans ([dev] slot8, 16-byte aligned,
 * ivfkm_bivf_slots_size(k, dim, number of screen values) bytes: a table of
 * the spans' value offsets per term — dim * (spans + 1) words, so that a
 * sparse span's start and end are two adjacent words — then one byte per
 * screen value position, written only at the positions of sparse-span
 * postings: the posting's slot within its 256-slot span).  Call after the
 * fill; read by ivfkm_assign_screen_ex. */
size_t ivfkm_bivf_slots_size(int64_t k, int64_t dim, int64_t n_values);
int ivfkm_bivf_slots(int64_t k, int64_t dim, int major, int64_t nrows, const int64_t* ptr,
                     const int32_t* cols, const uint32_t* headers, uint8_t* slot8,
                     ivfkm_stream_t stream);

/* ---- IVFD, object-inverted (_kernels.pyx:178-207) ------------------------
 * The paper's comparison variant in its own loop order: means outermost, each
 * mean's similarities to all N objects accumulated over the objects' inverted
 * file.  objects_inverted builds that file from the object CSR ([dev] x_ptr
 * int64[dim+1], x_obj int32[nnz] 0-based ascending within a term, x_val fp64).
 * assign_ivfd runs waves of `wave` means, one CTA per mean with a length-N
 * float64 slot each (workspace: ivfkm_ivfd_workspace_size); every object's
 * sum adds u*x in ascending term order (mul then add, no FMA), so the
 * similarities are the reference's bit for bit; labels by strict '>' from
 * 0.0 in ascending mean order (else mean 0), sims = the label's similarity
 * (mean 0's when nothing beats 0.0), then sizes / changed / exact objective
 * as ivfkm_assign_finish.  Reference interface: replaces
 * variants.py:188-206 + _kernels.pyx:178-207. */
size_t ivfkm_objects_inverted_workspace_size(int64_t nnz, int64_t dim);
int ivfkm_objects_inverted(int64_t n_obj, int64_t nnz, int64_t dim,
                           const int64_t* row_ptr /*[dev]*/, const int32_t* terms /*[dev] 0-based*/,
                           const double* val64 /*[dev]*/, int64_t* x_ptr /*[dev] dim+1*/,
                           int32_t* x_obj /*[dev] nnz*/, double* x_val /*[dev] nnz*/, void* ws,
                           size_t ws_bytes, ivfkm_stream_t stream);
size_t ivfkm_ivfd_workspace_size(int64_t n_obj, int64_t wave);
int ivfkm_assign_ivfd(int64_t n_obj, int64_t dim, const int64_t* x_ptr, const int32_t* x_obj,
                      const double* x_val, int64_t k, const int64_t* m_ptr /*[dev] k+1*/,
                      const int32_t* m_terms /*[dev] 0-based*/, const double* m_vals,
                      const int32_t* prev_labels /*[dev] or NULL*/, int32_t* labels /*[dev]*/,
                      double* sims /*[dev]*/, unsigned long long* sizes /*[dev] k or NULL*/,
                      ivfkm_stats* stats /*[dev]*/, int64_t wave, void* ws, size_t ws_bytes,
                      ivfkm_stream_t stream);

/* ---- host-buffer drop-in for _kernels.pyx:106-128 --------------------------
 * Same arguments and meaning as the reference kernel: 1-based term / mean
 * ids, float64 values, labels written 1-based, ctr[0..2] += postings touched.
 * Copies host->device, runs the BIVF build + assign on the current device,
 * copies labels back.  Returns IVFKM_E_RANGE for an out-of-range id.          */
int ivfkm_assign_ivf_host(int64_t n, const int64_t* indptr, const int32_t* terms,
                          const double* vals, int64_t dim, const int64_t* m_indptr,
                          const int32_t* m_cids, const double* m_vals, int64_t k,
                          int32_t* labels, int64_t* ctr);
/* The IVFD entry of the same kernel-module ABI (_kernels.pyx:178-207):
 * objects as their inverted file (x_indptr[dim+1], 1-based object ids),
 * means mean-major (m_indptr[k+1], 1-based terms); labels by the IVFD rule
 * (include note at ivfkm_assign).  The reference's rho / rho_max scratch
 * arrays are not needed.                                                    */
int ivfkm_assign_ivfd_host(int64_t n, const int64_t* x_indptr, const int32_t* x_oids,
                           const double* x_vals, int64_t dim, const int64_t* m_indptr,
                           const int32_t* m_terms, const double* m_vals, int64_t k,
                           int32_t* labels, int64_t* ctr);

/* ---- compact object rows (end-to-end uploads) ------------------------------
 * terms[h] restored from 16-bit gaps: gaps[h] = t[h] - t[h-1] within a row
 * (t[-1] = -1, so the first gap is t0 + 1); a gap >= 0xFFFF is stored as
 * 0xFFFF and its absolute 0-based id is exc_term[j] where exc_idx[j] = h
 * (exc_idx ascending).  Integer work, exact.                                  */
/* Rows from the reference's arrays ([dev]): 1-based term ids -> 0-based
 * terms0, values -> fp32 val32 (the screen's copy), and each row's L2 norm
 * xnorm (the screen's error bound; any summation order — the bound carries
 * a relative margin). In-place terms0 == terms1 is allowed. */
int ivfkm_rows_prepare(int64_t n_obj, const int64_t* row_ptr /*[dev] n+1*/,
                       const int32_t* terms1 /*[dev]*/, const double* val64 /*[dev]*/,
                       int32_t* terms0 /*[dev]*/, float* val32 /*[dev]*/, double* xnorm /*[dev] n*/,
                       ivfkm_stream_t stream);
int ivfkm_rows_decode(int64_t n_obj, const int64_t* row_ptr /*[dev] n+1*/,
                      const uint16_t* gaps /*[dev] nnz*/, int64_t n_exc,
                      const int64_t* exc_idx /*[dev]*/, const int32_t* exc_term /*[dev]*/,
                      int32_t* terms /*[dev] out, nnz*/, ivfkm_stream_t stream);

/* ---- ingestion: the step before the path ---------
 *   ivfkm_uci_parse   <- io.py:72-121   parse_uci_bow (host, multi-threaded)
 *   ivfkm_bow_sort    <- io.py:120      triples.sort() + duplicate-pair check
 *   ivfkm_bow_df      <- io.py:138      df = bincount(terms)
 *   ivfkm_tfidf       <- io.py:141-174  weights, drops, L2 normalisation
 * Parse errors are returned as data (line, code, values); the Python layer
 * raises ParseError with the reference's wording.                          */
int ivfkm_uci_parse(const char* text, size_t len, int threads, int64_t* header /*[3]*/,
                    int64_t cap, int32_t* docs, int32_t* terms, int32_t* counts,
                    int64_t* lines, int64_t* n_read, int64_t* n_lines, int64_t* err_line,
                    int* err_code, int64_t* err_val /*[3]*/);
size_t ivfkm_bow_workspace_size(int64_t n);
int ivfkm_bow_sort(int64_t n, int64_t n_docs, int64_t dim, int32_t* docs /*[dev]*/,
                   int32_t* terms /*[dev]*/, int32_t* counts /*[dev]*/, int64_t* lines /*[dev]*/,
                   unsigned long long* dup_line /*[dev] 1*/, void* ws, size_t ws_bytes,
                   ivfkm_stream_t stream);
int ivfkm_bow_df(int64_t n, int64_t dim, const int32_t* terms /*[dev]*/,
                 unsigned long long* df /*[dev] dim*/, ivfkm_stream_t stream);
size_t ivfkm_tfidf_workspace_size(int64_t n, int64_t n_docs);
int ivfkm_tfidf(int64_t n, int64_t n_docs, int64_t dim, const int32_t* docs /*[dev]*/,
                const int32_t* terms /*[dev]*/, const int32_t* counts /*[dev]*/,
                const double* idf /*[dev] dim*/, int64_t* out_ptr /*[dev] n_docs+1*/,
                int32_t* out_terms /*[dev] n*/, double* out_vals /*[dev] n*/,
                int32_t* dropped /*[dev] n_docs*/, int64_t* counts_out /*[host] 2*/, void* ws,
                size_t ws_bytes, ivfkm_stream_t stream);

/* ---- host utilities -------------------------------------------------------*/
uint64_t ivfkm_fnv1a64(const void* data, size_t nbytes); /* variants.py:77-83 */

typedef struct ivfkm_synth_spec {
  int64_t n, dim;
  int32_t nnz_kind; /* 0 = Poisson(nnz_mean), 1 = lognormal(mean, sigma) */
  double nnz_mean, nnz_sigma;
  int64_t nnz_lo, nnz_hi;
  double zipf_s;
  int64_t seed;
} ivfkm_synth_spec;
int ivfkm_synth_rows(const ivfkm_synth_spec* spec, int64_t* nnz_rows /*[host] n*/);
int ivfkm_synth_fill(const ivfkm_synth_spec* spec, const int64_t* cap_ptr /*[host] n+1*/,
                     int64_t* indptr, int32_t* terms, double* vals, int64_t* n_out,
                     int64_t* nnz_out);

#ifdef __cplusplus
}
#endif
#endif
