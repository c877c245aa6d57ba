// Seeded synthetic corpus generator (host, OpenMP) for the BASELINE configs.
//
// Stand-in for PubMed / NYT, shaped by
// BASELINE.json:configs as restated in SURVEY.md §8(d):
//   nnz_i  ~ Poisson(mean) or lognormal(distribution mean, sigma), clipped;
//   terms  = first nnz_i distinct draws of a Zipf(s) sequence over 1..D
//            (successive sampling, repeats rejected), sorted;
//   value  = (1 + ln count) * ln(N / df), count ~ Geometric(1/2);
//   entries with df == N have weight 0 and are dropped (reference io.py:153-154),
//   rows left empty are dropped (io.py:156-164); rows L2-normalised in fp64.
// Every row draws from its own SplitMix64 stream keyed by (seed, row), so the
// output does not depend on the thread count.
#include <cmath>
#include <cstdint>
#include <cstring>
#include <vector>
#include <algorithm>
#include <omp.h>

#include "ivfkm.h"

namespace {

struct Stream {
  uint64_t s;
  explicit Stream(uint64_t seed, uint64_t row) {
    s = seed * 0x9E3779B97F4A7C15ull ^ (row + 0x632BE59BD9B4E019ull) * 0xD1B54A32D192ED03ull;
    next(); next();
  }
  uint64_t next() {
    s += 0x9E3779B97F4A7C15ull;
    uint64_t z = s;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
  }
  double uniform() { return (double)(next() >> 11) * 0x1.0p-53; }           // [0,1)
  double uniform_pos() { return ((double)(next() >> 11) + 0.5) * 0x1.0p-53; } // (0,1)
};

int64_t draw_nnz(Stream& st, const ivfkm_synth_spec& sp) {
  double raw;
  if (sp.nnz_kind == 0) {  // Poisson by inversion
    double u = st.uniform();
    double p = std::exp(-sp.nnz_mean), F = p;
    int64_t k = 0;
    while (u > F && k < 100000) { ++k; p *= sp.nnz_mean / (double)k; F += p; }
    raw = (double)k;
  } else {                 // lognormal, mu = ln(mean) - sigma^2/2
    double u1 = st.uniform_pos(), u2 = st.uniform();
    double z = std::sqrt(-2.0 * std::log(u1)) * std::cos(2.0 * M_PI * u2);
    double mu = std::log(sp.nnz_mean) - 0.5 * sp.nnz_sigma * sp.nnz_sigma;
    raw = std::nearbyint(std::exp(mu + sp.nnz_sigma * z));
  }
  int64_t hi = std::min<int64_t>(sp.nnz_hi, sp.dim);
  int64_t v = (int64_t)raw;
  if (v < sp.nnz_lo) v = sp.nnz_lo;
  if (v > hi) v = hi;
  return v;
}

}  // namespace

extern "C" int ivfkm_synth_rows(const ivfkm_synth_spec* sp, int64_t* nnz_rows) {
  if (!sp || !nnz_rows || sp->n <= 0 || sp->dim <= 0) return 1;
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < sp->n; ++i) {
    Stream st((uint64_t)sp->seed, (uint64_t)i);
    nnz_rows[i] = draw_nnz(st, *sp);
  }
  return 0;
}

// Fills terms (0-based, sorted per row) and counts for rows with the
// capacity layout cap_ptr (exclusive scan of nnz_rows), then computes
// tf-idf, drops df==N entries and empty rows, normalises, and compacts in
// place.  Outputs: indptr[n_out+1], terms (1-based), vals; *n_out, *nnz_out.
extern "C" int ivfkm_synth_fill(const ivfkm_synth_spec* sp, const int64_t* cap_ptr,
                                int64_t* indptr, int32_t* terms, double* vals,
                                int64_t* n_out, int64_t* nnz_out) {
  if (!sp || !cap_ptr || !indptr || !terms || !vals) return 1;
  const int64_t n = sp->n, dim = sp->dim;
  std::vector<double> cdf(dim);
  {
    double acc = 0.0;
    for (int64_t t = 0; t < dim; ++t) { acc += std::pow((double)(t + 1), -sp->zipf_s); cdf[t] = acc; }
    for (int64_t t = 0; t < dim; ++t) cdf[t] /= acc;
  }
  // pass 1: terms + geometric counts (count stored in vals for now)
#pragma omp parallel
  {
    std::vector<int64_t> mark(dim, -1);
    std::vector<int32_t> row;
#pragma omp for schedule(dynamic, 256)
    for (int64_t i = 0; i < n; ++i) {
      Stream st((uint64_t)sp->seed, (uint64_t)i);
      int64_t m = draw_nnz(st, *sp);
      row.clear();
      while ((int64_t)row.size() < m) {
        double u = st.uniform();
        int64_t t = std::upper_bound(cdf.begin(), cdf.end(), u) - cdf.begin();
        if (t >= dim) t = dim - 1;
        if (mark[t] == i) continue;
        mark[t] = i;
        row.push_back((int32_t)t);
      }
      std::sort(row.begin(), row.end());
      int64_t base = cap_ptr[i];
      for (int64_t h = 0; h < m; ++h) {
        uint64_t r = st.next();
        int c = r ? __builtin_ctzll(r) + 1 : 65;  // Geometric(1/2) on {1,2,...}
        terms[base + h] = row[h];
        vals[base + h] = (double)c;
      }
    }
  }
  const int64_t cap = cap_ptr[n];
  std::vector<int64_t> df(dim, 0);
#pragma omp parallel
  {
    std::vector<int64_t> local(dim, 0);
#pragma omp for schedule(static)
    for (int64_t e = 0; e < cap; ++e) local[terms[e]]++;
#pragma omp critical
    for (int64_t t = 0; t < dim; ++t) df[t] += local[t];
  }
  std::vector<double> idf(dim, 0.0);
  for (int64_t t = 0; t < dim; ++t)
    if (df[t] > 0) idf[t] = std::log((double)n / (double)df[t]);
  // per-row kept counts, then compaction (sequential scan; rows keep order)
  std::vector<int64_t> kept(n);
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < n; ++i) {
    int64_t c = 0;
    for (int64_t e = cap_ptr[i]; e < cap_ptr[i + 1]; ++e) c += (df[terms[e]] < n);
    kept[i] = c;
  }
  std::vector<int64_t> out_ptr(n + 1, 0), out_row(n, -1);
  int64_t rows = 0, tot = 0;
  for (int64_t i = 0; i < n; ++i) {
    if (kept[i] == 0) continue;
    out_row[i] = rows;
    out_ptr[rows] = tot;
    tot += kept[i];
    ++rows;
  }
  out_ptr[rows] = tot;
  // compaction moves entries to lower addresses only, so a sequential pass
  // over rows in order is safe in place.
  for (int64_t i = 0; i < n; ++i) {
    if (out_row[i] < 0) continue;
    int64_t w = out_ptr[out_row[i]];
    for (int64_t e = cap_ptr[i]; e < cap_ptr[i + 1]; ++e) {
      int32_t t = terms[e];
      if (df[t] >= n) continue;
      double c = vals[e];
      terms[w] = t + 1;
      vals[w] = (1.0 + std::log(c)) * idf[t];
      ++w;
    }
  }
#pragma omp parallel for schedule(static)
  for (int64_t r = 0; r < rows; ++r) {
    double sq = 0.0;
    for (int64_t e = out_ptr[r]; e < out_ptr[r + 1]; ++e) sq += vals[e] * vals[e];
    double nrm = std::sqrt(sq);
    for (int64_t e = out_ptr[r]; e < out_ptr[r + 1]; ++e) vals[e] = vals[e] / nrm;
  }
  std::memcpy(indptr, out_ptr.data(), sizeof(int64_t) * (rows + 1));
  *n_out = rows;
  *nnz_out = tot;
  return 0;
}
