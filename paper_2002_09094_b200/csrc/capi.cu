// C-ABI glue: error strings, the FNV-1a digest, and the host-buffer drop-in
// for the reference kernel-module entry point _kernels.pyx:106-128.
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "common.cuh"

using namespace ivfkm;

extern "C" int ivfkm_version(void) { return 1; }

extern "C" const char* ivfkm_error_string(int code) {
  switch (code) {
    case IVFKM_OK: return "ok";
    case IVFKM_E_ARG: return "invalid argument";
    case IVFKM_E_UNSUPPORTED: return "unsupported size (k or nnz beyond the supported range)";
    case IVFKM_E_CAPACITY: return "output capacity too small";
    case IVFKM_E_WORKSPACE: return "workspace too small";
    case IVFKM_E_NOGPU: return "no CUDA device";
    case IVFKM_E_RANGE: return "posting id outside its owner range";
    default: break;
  }
  if (code > 0) return cudaGetErrorString(static_cast<cudaError_t>(code));
  return "unknown error";
}

extern "C" int ivfkm_device_count(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) return 0;
  return n;
}

// 64-bit FNV-1a, the assignment digest of reference variants.py:69-83.
extern "C" uint64_t ivfkm_fnv1a64(const void* data, size_t nbytes) {
  const unsigned char* p = static_cast<const unsigned char*>(data);
  uint64_t h = 0xCBF29CE484222325ull;
  for (size_t i = 0; i < nbytes; ++i) {
    h ^= p[i];
    h *= 0x100000001B3ull;
  }
  return h;
}

namespace {

struct DevBuf {
  void* p = nullptr;
  ~DevBuf() {
    if (p) cudaFree(p);
  }
  cudaError_t alloc(size_t bytes) { return cudaMalloc(&p, bytes ? bytes : 16); }
  template <class T>
  T* as() const {
    return static_cast<T*>(p);
  }
};

}  // namespace

namespace {

// Host buffers -> device -> labels: objects as a CSR (1-based terms), means
// as term-major postings (major 1: rows = terms, cols = 1-based mean ids) or
// mean-major rows (major 0: rows = means, cols = 1-based terms).
int assign_host(int64_t n, const int64_t* indptr, const int32_t* terms, const double* vals,
                int64_t dim, int major, const int64_t* m_indptr, const int32_t* m_cids,
                const double* m_vals, int64_t k, int rule, int32_t* labels, int64_t* ctr) {
  if (n < 0 || dim < 1 || k < 1 || !indptr || !m_indptr || !labels) return IVFKM_E_ARG;
  const int64_t m_rows = major == 1 ? dim : k;
  if (ivfkm_device_count() < 1) return IVFKM_E_NOGPU;
  const int64_t nnz = indptr[n];
  const int64_t mnz = m_indptr[m_rows];
  // validation the reference performs before its kernel (data.py:148-175,
  // data.py:261-262 CorruptionError), restated on the host buffers
  std::vector<int32_t> t0((size_t)nnz), c0((size_t)mnz);
  for (int64_t e = 0; e < nnz; ++e) {
    if (terms[e] < 1 || terms[e] > dim) return IVFKM_E_RANGE;
    t0[e] = terms[e] - 1;
  }
  std::vector<double> mnorm2((size_t)k, 0.0);
  for (int64_t q = 0; q < mnz; ++q) {
    const int64_t lim = major == 1 ? k : dim;  // cols: mean ids or terms
    if (m_cids[q] < 1 || m_cids[q] > lim) return IVFKM_E_RANGE;
    c0[q] = m_cids[q] - 1;
  }
  for (int64_t r = 0; r < m_rows; ++r) {
    for (int64_t q = m_indptr[r]; q < m_indptr[r + 1]; ++q) {
      const int64_t c = major == 1 ? c0[q] : r;
      mnorm2[c] += m_vals[q] * m_vals[q];
    }
  }
  double mu_max = 0.0;
  for (double v : mnorm2) mu_max = std::fmax(mu_max, std::sqrt(v));
  std::vector<float> v32((size_t)nnz);
  std::vector<double> xn((size_t)n);
  for (int64_t i = 0; i < n; ++i) {
    double s = 0.0;
    for (int64_t e = indptr[i]; e < indptr[i + 1]; ++e) {
      v32[e] = (float)vals[e];
      s += vals[e] * vals[e];
    }
    xn[i] = std::sqrt(s);
  }
  DevBuf d_ip, d_t, d_v32, d_v64, d_xn, d_mp, d_mc, d_mv, d_hdr, d_p32, d_p64, d_bws, d_lab,
      d_sims, d_sizes, d_stats, d_aws;
  const size_t bws = ivfkm_bivf_workspace_size(dim, k);
  const size_t aws = ivfkm_assign_workspace_size(n, k);
  IVFKM_TRY(d_ip.alloc(sizeof(int64_t) * (n + 1)));
  IVFKM_TRY(d_t.alloc(sizeof(int32_t) * nnz));
  IVFKM_TRY(d_v32.alloc(sizeof(float) * nnz));
  IVFKM_TRY(d_v64.alloc(sizeof(double) * nnz));
  IVFKM_TRY(d_xn.alloc(sizeof(double) * n));
  IVFKM_TRY(d_mp.alloc(sizeof(int64_t) * (m_rows + 1)));
  IVFKM_TRY(d_mc.alloc(sizeof(int32_t) * mnz));
  IVFKM_TRY(d_mv.alloc(sizeof(double) * mnz));
  IVFKM_TRY(d_hdr.alloc(sizeof(uint32_t) * ivfkm_bivf_headers_size(k, dim)));
  IVFKM_TRY(d_bws.alloc(bws));
  IVFKM_TRY(d_lab.alloc(sizeof(int32_t) * n));
  IVFKM_TRY(d_sims.alloc(sizeof(double) * n));
  IVFKM_TRY(d_sizes.alloc(sizeof(unsigned long long) * k));
  IVFKM_TRY(d_stats.alloc(sizeof(ivfkm_stats)));
  IVFKM_TRY(d_aws.alloc(aws));
  cudaStream_t st = nullptr;
  IVFKM_TRY(cudaMemcpyAsync(d_ip.p, indptr, sizeof(int64_t) * (n + 1), cudaMemcpyHostToDevice, st));
  IVFKM_TRY(cudaMemcpyAsync(d_t.p, t0.data(), sizeof(int32_t) * nnz, cudaMemcpyHostToDevice, st));
  IVFKM_TRY(cudaMemcpyAsync(d_v32.p, v32.data(), sizeof(float) * nnz, cudaMemcpyHostToDevice, st));
  IVFKM_TRY(cudaMemcpyAsync(d_v64.p, vals, sizeof(double) * nnz, cudaMemcpyHostToDevice, st));
  IVFKM_TRY(cudaMemcpyAsync(d_xn.p, xn.data(), sizeof(double) * n, cudaMemcpyHostToDevice, st));
  IVFKM_TRY(cudaMemcpyAsync(d_mp.p, m_indptr, sizeof(int64_t) * (m_rows + 1), cudaMemcpyHostToDevice, st));
  IVFKM_TRY(cudaMemcpyAsync(d_mc.p, c0.data(), sizeof(int32_t) * mnz, cudaMemcpyHostToDevice, st));
  IVFKM_TRY(cudaMemcpyAsync(d_mv.p, m_vals, sizeof(double) * mnz, cudaMemcpyHostToDevice, st));
  // fp16 screen values (half the posting bytes) unless the means are not
  // normalised far beyond unit norm (fp16 range)
  const int bits = mu_max <= 32768.0 ? 16 : 32;
  int64_t totals[2] = {0, 0};
  int rc = ivfkm_bivf_plan(k, dim, major, m_rows, d_mp.as<int64_t>(), d_mc.as<int32_t>(),
                           d_hdr.as<uint32_t>(), totals, d_bws.p, bws, nullptr);
  if (rc) return rc;
  IVFKM_TRY(d_p32.alloc(sizeof(float) * (totals[0] + 1)));
  IVFKM_TRY(d_p64.alloc(sizeof(double) * (totals[1] + 1)));
  rc = ivfkm_bivf_fill(k, dim, major, m_rows, d_mp.as<int64_t>(), d_mc.as<int32_t>(), d_mv.as<double>(),
                       d_hdr.as<uint32_t>(), d_p32.p, bits, d_p64.as<double>(), mnz,
                       nullptr, 0, nullptr);
  if (rc) return rc;
  rc = ivfkm_assign(n, d_ip.as<int64_t>(), d_t.as<int32_t>(), d_v32.as<float>(),
                    d_v64.as<double>(), d_xn.as<double>(), k, dim, d_hdr.as<uint32_t>(),
                    d_p32.p, bits, d_p64.as<double>(), mu_max, nullptr, d_lab.as<int32_t>(),
                    d_sims.as<double>(), d_sizes.as<unsigned long long>(),
                    d_stats.as<ivfkm_stats>(), nullptr, rule, d_aws.p, aws, nullptr);
  if (rc) return rc;
  ivfkm_stats stats;
  IVFKM_TRY(cudaMemcpyAsync(labels, d_lab.p, sizeof(int32_t) * n, cudaMemcpyDeviceToHost, st));
  IVFKM_TRY(cudaMemcpyAsync(&stats, d_stats.p, sizeof(stats), cudaMemcpyDeviceToHost, st));
  IVFKM_TRY(cudaStreamSynchronize(st));
  for (int64_t i = 0; i < n; ++i) labels[i] += 1;
  if (ctr) {
    ctr[0] += (int64_t)stats.postings;
    ctr[1] += (int64_t)stats.postings;
    ctr[2] += (int64_t)stats.postings;
  }
  return IVFKM_OK;
}

}  // namespace

// Same arguments and meaning as the reference kernel (1-based ids, float64
// values, labels written 1-based, ctr[0..2] += postings).  The reference's
// rho scratch argument is not needed: rho lives in registers on the device.
extern "C" int ivfkm_assign_ivf_host(int64_t n, const int64_t* indptr, const int32_t* terms,
                                     const double* vals, int64_t dim, const int64_t* m_indptr,
                                     const int32_t* m_cids, const double* m_vals, int64_t k,
                                     int32_t* labels, int64_t* ctr) {
  return assign_host(n, indptr, terms, vals, dim, 1, m_indptr, m_cids, m_vals, k, 0, labels, ctr);
}

// IVFD (_kernels.pyx:178-207): objects arrive as their inverted file
// (x_indptr over terms, 1-based object ids ascending within a term), means
// mean-major — exactly the input of the object-inverted kernel
// (ivfkm_assign_ivfd): ids made 0-based, everything uploaded, one call.
extern "C" int ivfkm_assign_ivfd_host(int64_t n, const int64_t* x_indptr, const int32_t* x_oids,
                                      const double* x_vals, int64_t dim, const int64_t* m_indptr,
                                      const int32_t* m_terms, const double* m_vals, int64_t k,
                                      int32_t* labels, int64_t* ctr) {
  if (n < 0 || dim < 1 || k < 1 || !x_indptr || !m_indptr || !labels) return IVFKM_E_ARG;
  if (ivfkm_device_count() < 1) return IVFKM_E_NOGPU;
  const int64_t nnz = x_indptr[dim];
  const int64_t mnz = m_indptr[k];
  std::vector<int32_t> o0((size_t)nnz), t0((size_t)mnz);
  for (int64_t q = 0; q < nnz; ++q) {
    if (x_oids[q] < 1 || x_oids[q] > n) return IVFKM_E_RANGE;
    o0[q] = x_oids[q] - 1;
  }
  for (int64_t q = 0; q < mnz; ++q) {
    if (m_terms[q] < 1 || m_terms[q] > dim) return IVFKM_E_RANGE;
    t0[q] = m_terms[q] - 1;
  }
  if (n == 0) return IVFKM_OK;
  // one wave of means while their length-n slots stay within 2 GB
  int64_t wave = (int64_t)((2ull << 30) / (8ull * (uint64_t)n));
  wave = wave < 1 ? 1 : (wave > k ? k : wave);
  const size_t ws = ivfkm_ivfd_workspace_size(n, wave);
  DevBuf d_xp, d_xo, d_xv, d_mp, d_mt, d_mv, d_lab, d_sims, d_sizes, d_stats, d_ws;
  IVFKM_TRY(d_xp.alloc(sizeof(int64_t) * (dim + 1)));
  IVFKM_TRY(d_xo.alloc(sizeof(int32_t) * (nnz + 1)));
  IVFKM_TRY(d_xv.alloc(sizeof(double) * (nnz + 1)));
  IVFKM_TRY(d_mp.alloc(sizeof(int64_t) * (k + 1)));
  IVFKM_TRY(d_mt.alloc(sizeof(int32_t) * (mnz + 1)));
  IVFKM_TRY(d_mv.alloc(sizeof(double) * (mnz + 1)));
  IVFKM_TRY(d_lab.alloc(sizeof(int32_t) * n));
  IVFKM_TRY(d_sims.alloc(sizeof(double) * n));
  IVFKM_TRY(d_sizes.alloc(sizeof(unsigned long long) * k));
  IVFKM_TRY(d_stats.alloc(sizeof(ivfkm_stats)));
  IVFKM_TRY(d_ws.alloc(ws));
  cudaStream_t st = nullptr;
  IVFKM_TRY(cudaMemcpyAsync(d_xp.p, x_indptr, sizeof(int64_t) * (dim + 1), cudaMemcpyHostToDevice, st));
  IVFKM_TRY(cudaMemcpyAsync(d_xo.p, o0.data(), sizeof(int32_t) * nnz, cudaMemcpyHostToDevice, st));
  IVFKM_TRY(cudaMemcpyAsync(d_xv.p, x_vals, sizeof(double) * nnz, cudaMemcpyHostToDevice, st));
  IVFKM_TRY(cudaMemcpyAsync(d_mp.p, m_indptr, sizeof(int64_t) * (k + 1), cudaMemcpyHostToDevice, st));
  IVFKM_TRY(cudaMemcpyAsync(d_mt.p, t0.data(), sizeof(int32_t) * mnz, cudaMemcpyHostToDevice, st));
  IVFKM_TRY(cudaMemcpyAsync(d_mv.p, m_vals, sizeof(double) * mnz, cudaMemcpyHostToDevice, st));
  int rc = ivfkm_assign_ivfd(n, dim, d_xp.as<int64_t>(), d_xo.as<int32_t>(), d_xv.as<double>(), k,
                             d_mp.as<int64_t>(), d_mt.as<int32_t>(), d_mv.as<double>(), nullptr,
                             d_lab.as<int32_t>(), d_sims.as<double>(),
                             d_sizes.as<unsigned long long>(), d_stats.as<ivfkm_stats>(), wave,
                             d_ws.p, ws, st);
  if (rc) return rc;
  ivfkm_stats stats;
  IVFKM_TRY(cudaMemcpyAsync(labels, d_lab.p, sizeof(int32_t) * n, cudaMemcpyDeviceToHost, st));
  IVFKM_TRY(cudaMemcpyAsync(&stats, d_stats.p, sizeof(stats), cudaMemcpyDeviceToHost, st));
  IVFKM_TRY(cudaStreamSynchronize(st));
  for (int64_t i = 0; i < n; ++i) labels[i] += 1;
  if (ctr) {
    ctr[0] += (int64_t)stats.postings;
    ctr[1] += (int64_t)stats.postings;
    ctr[2] += (int64_t)stats.postings;
  }
  return IVFKM_OK;
}
