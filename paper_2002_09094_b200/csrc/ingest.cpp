// UCI bag-of-words parsing (host, OpenMP), the input stage before the path.
//
// Restates reference io.py:72-121 (parse_uci_bow) over an in-memory buffer:
// three header integers (documents, vocabulary, entries), then one
// "doc term count" triple per line, ids 1-based.  The body is split into
// per-thread chunks at line boundaries and parsed in parallel; every thread
// keeps its first error, so the first error in line order is known exactly
// (the reference stops there).  Duplicate (doc, term) pairs are detected on
// the device after the sort (ivfkm_bow_sort); the caller takes the earlier
// of the two error lines, as the reference's single pass would.
//
// Integer fields follow Python's int(): optional sign, ASCII digits with
// single underscores between digits.  Error codes (messages built by the
// Python layer with the reference's exact wording, io.py:84-120):
//   1 header line not an integer    2 negative header count
//   3 not three fields              4 non-integer field
//   5 doc id out of range           6 term id out of range
//   7 count not positive
#include <algorithm>
#include <cstdint>
#include <cstring>
#include <vector>
#include <omp.h>

#include "ivfkm.h"

namespace {

inline bool is_space(char c) {
  return c == ' ' || c == '\t' || c == '\r' || c == '\n' || c == '\v' || c == '\f';
}

// Python int() of one whitespace-free token; false if not an integer.
// Values beyond int64 saturate (they are out of every valid range).
bool parse_int(const char* s, const char* e, int64_t* out) {
  if (s == e) return false;
  bool neg = false;
  if (*s == '+' || *s == '-') {
    neg = *s == '-';
    ++s;
  }
  if (s == e) return false;
  int64_t v = 0;
  bool prev_digit = false, sat = false;
  for (const char* p = s; p < e; ++p) {
    if (*p >= '0' && *p <= '9') {
      if (!sat) {
        if (v > (INT64_MAX - 9) / 10) sat = true;
        else v = v * 10 + (*p - '0');
      }
      prev_digit = true;
    } else if (*p == '_' && prev_digit && p + 1 < e && p[1] >= '0' && p[1] <= '9') {
      prev_digit = false;
    } else {
      return false;
    }
  }
  if (sat) v = INT64_MAX;
  *out = neg ? -v : v;
  return true;
}

struct Err {
  int64_t line = -1;  // global 1-based line number of the first error, -1 none
  int code = 0;
  int64_t val[3] = {0, 0, 0};
};

struct Chunk {
  const char* b;
  const char* e;
  int64_t lines = 0;        // lines in the chunk
  int64_t first_line = 0;   // global number of its first line
  std::vector<int32_t> d, t, c;
  std::vector<int64_t> ln;  // local line index of each triple
  int64_t err_local = -1;
  int err_code = 0;
  int64_t err_val[3] = {0, 0, 0};
};

void parse_body(Chunk& ck, int64_t n_docs, int64_t dim) {
  const char* p = ck.b;
  int64_t li = 0;
  while (p < ck.e) {
    const char* nl = static_cast<const char*>(memchr(p, '\n', (size_t)(ck.e - p)));
    const char* le = nl ? nl : ck.e;
    // tokens
    const char* tk[4][2];
    int nt = 0;
    const char* q = p;
    while (q < le) {
      while (q < le && is_space(*q)) ++q;
      if (q >= le) break;
      const char* s = q;
      while (q < le && !is_space(*q)) ++q;
      if (nt < 4) {
        tk[nt][0] = s;
        tk[nt][1] = q;
      }
      ++nt;
    }
    if (ck.err_local < 0 && nt > 0) {
      int64_t v[3];
      int code = 0;
      if (nt != 3) {
        code = 3;
      } else if (!parse_int(tk[0][0], tk[0][1], &v[0]) || !parse_int(tk[1][0], tk[1][1], &v[1]) ||
                 !parse_int(tk[2][0], tk[2][1], &v[2])) {
        code = 4;
      } else if (v[0] < 1 || v[0] > n_docs) {
        code = 5;
      } else if (v[1] < 1 || v[1] > dim) {
        code = 6;
      } else if (v[2] <= 0) {
        code = 7;
      }
      if (code) {
        ck.err_local = li;
        ck.err_code = code;
        if (code >= 5) {
          ck.err_val[0] = v[0];
          ck.err_val[1] = v[1];
          ck.err_val[2] = v[2];
        }
      } else {
        ck.d.push_back((int32_t)v[0]);
        ck.t.push_back((int32_t)v[1]);
        ck.c.push_back(v[2] > INT32_MAX ? INT32_MAX : (int32_t)v[2]);
        ck.ln.push_back(li);
      }
    } else if (nt > 0 && ck.err_local >= 0) {
      // after the chunk's first error only the count matters (for the
      // entry-count message, which is moot once an error is reported)
    }
    ++li;
    p = nl ? nl + 1 : ck.e;
  }
  ck.lines = li;
}

}  // namespace

// Parse a UCI bag-of-words buffer.  header[3] = (documents, vocabulary,
// declared entries).  Triples are written in line order (docs/terms/counts,
// 1-based, and their 1-based line numbers) up to `cap` entries; *n_read =
// triples parsed before the first error (all of them when there is none),
// *n_lines = lines in the buffer.  On a malformed line: *err_line (1-based),
// *err_code (see above) and err_val = (doc, term, count) where relevant;
// *err_line = -1 when every line parsed.  Returns IVFKM_OK (parse errors are
// data, not failures), IVFKM_E_CAPACITY when more than `cap` triples parsed.
extern "C" int ivfkm_uci_parse(const char* text, size_t len, int threads, int64_t* header,
                               int64_t cap, int32_t* docs, int32_t* terms, int32_t* counts,
                               int64_t* lines, int64_t* n_read, int64_t* n_lines,
                               int64_t* err_line, int* err_code, int64_t* err_val) {
  if (!header || !n_read || !n_lines || !err_line || !err_code || !err_val) return IVFKM_E_ARG;
  *err_line = -1;
  *err_code = 0;
  *n_read = 0;
  err_val[0] = err_val[1] = err_val[2] = 0;
  header[0] = header[1] = header[2] = 0;
  const char* p = text;
  const char* end = text + len;
  int64_t lineno = 0;
  // ---- header (io.py:80-96)
  for (int h = 0; h < 3 && p < end; ++h) {
    const char* nl = static_cast<const char*>(memchr(p, '\n', (size_t)(end - p)));
    const char* le = nl ? nl : end;
    ++lineno;
    const char* s = p;
    const char* e = le;
    while (s < e && is_space(*s)) ++s;
    while (e > s && is_space(e[-1])) --e;
    // text.lstrip("-").isdigit(): optional leading minus signs, then digits only
    const char* d = s;
    while (d < e && *d == '-') ++d;
    bool digits = d < e;
    for (const char* q = d; q < e; ++q) digits = digits && (*q >= '0' && *q <= '9');
    int64_t v = 0;
    if (!digits || !parse_int(s, e, &v)) {
      *err_line = lineno;
      *err_code = 1;
      *n_lines = lineno;
      return IVFKM_OK;
    }
    if (v < 0) {
      *err_line = lineno;
      *err_code = 2;
      *n_lines = lineno;
      return IVFKM_OK;
    }
    header[h] = v;
    p = nl ? nl + 1 : end;
  }
  if (lineno < 3) {  // empty input / truncated header: the caller words it
    *n_lines = lineno;
    return IVFKM_OK;
  }
  // ---- body, in parallel chunks split at line boundaries
  const int64_t body = end - p;
  int nth = threads > 0 ? threads : omp_get_max_threads();
  if (body < (int64_t)1 << 20) nth = 1;
  std::vector<Chunk> ck((size_t)nth);
  {
    const char* s = p;
    for (int i = 0; i < nth; ++i) {
      const char* e = i == nth - 1 ? end : p + body * (i + 1) / nth;
      if (e < s) e = s;
      if (i < nth - 1) {
        const char* nl = static_cast<const char*>(memchr(e, '\n', (size_t)(end - e)));
        e = nl ? nl + 1 : end;
      }
      ck[i].b = s;
      ck[i].e = e;
      s = e;
    }
  }
#pragma omp parallel for num_threads(nth) schedule(static, 1)
  for (int i = 0; i < nth; ++i) parse_body(ck[i], header[0], header[1]);
  int64_t run_line = lineno, run_n = 0;
  bool stop = false;
  for (int i = 0; i < nth; ++i) {
    ck[i].first_line = run_line + 1;
    if (!stop) {
      const size_t m = ck[i].d.size();
      for (size_t j = 0; j < m; ++j) {
        if (run_n < cap) {
          docs[run_n] = ck[i].d[j];
          terms[run_n] = ck[i].t[j];
          counts[run_n] = ck[i].c[j];
          lines[run_n] = ck[i].first_line + ck[i].ln[j];
        }
        ++run_n;
      }
      if (ck[i].err_local >= 0) {
        *err_line = ck[i].first_line + ck[i].err_local;
        *err_code = ck[i].err_code;
        err_val[0] = ck[i].err_val[0];
        err_val[1] = ck[i].err_val[1];
        err_val[2] = ck[i].err_val[2];
        stop = true;
      }
    }
    run_line += ck[i].lines;
  }
  *n_read = run_n;
  *n_lines = run_line;
  return run_n > cap ? IVFKM_E_CAPACITY : IVFKM_OK;
}
