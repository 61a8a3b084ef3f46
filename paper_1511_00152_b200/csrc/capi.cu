// extern "C" entry points of include/sketchcu.h: argument validation (the reference's
// DimensionError / ParameterError cases) and dispatch to the kernels.
#include <stdio.h>

#include <atomic>
#include <mutex>
#include <string>
#include <vector>

#include "common.cuh"

namespace skc {

static thread_local std::string g_err;
static std::atomic<uint64_t> g_launches{0};
void set_error(const std::string& msg) { g_err = msg; }
int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}
void note_launches(int64_t delta) { g_launches.fetch_add((uint64_t)delta, std::memory_order_relaxed); }
int check_launch(const char* what) {
  g_launches.fetch_add(1, std::memory_order_relaxed);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(SKC_ECUDA, std::string(what) + ": " + cudaGetErrorString(e));
  return SKC_OK;
}
int sm_count() {
  static std::mutex mu;
  static std::vector<int> cache;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(mu);
  if ((int)cache.size() <= dev) cache.resize(dev + 1, 0);
  if (cache[dev] == 0) {
    int c = 0;
    cudaDeviceGetAttribute(&c, cudaDevAttrMultiProcessorCount, dev);
    cache[dev] = c > 0 ? c : 148;
  }
  return cache[dev];
}

// kernels (sketch.cu, moments.cu, kmeans.cu, formats.cu)
int philox_indices_launch(uint64_t, int64_t, int64_t, int32_t, int32_t, int32_t*, cudaStream_t);
int sketch_given_launch(const void*, int32_t, int64_t, int64_t, int32_t, int32_t, int32_t, uint64_t, int32_t, int32_t,
                        const int32_t*, void*, int32_t, cudaStream_t);
int reseed_at_launch(const int32_t*, const void*, int, int32_t, const long long*, const int32_t*, int32_t, int32_t,
                     double*, cudaStream_t);
int pack_records_launch(const int32_t*, const void*, int, int64_t, int32_t, uint32_t*, cudaStream_t);
int unpack_records_launch(const uint32_t*, int64_t, int32_t, int32_t*, double*, cudaStream_t);
size_t dense_sums_ws(int64_t, int32_t, int32_t);
size_t dense_assign_ws(int32_t, int32_t);
int dense_assign_launch(const void*, int, int64_t, int64_t, int32_t, const double*, int32_t, double*, int32_t*,
                        double*, cudaStream_t);
int dense_sums_launch(const void*, int, int64_t, int64_t, int32_t, const int32_t*, int32_t, double*, long long*, void*,
                      cudaStream_t);
int sketch_launch(const void*, int32_t, int64_t, int64_t, int32_t, int32_t, int32_t, uint64_t, uint64_t, int64_t,
                  int32_t, int32_t, int32_t*, void*, int32_t, double*, cudaStream_t);
int sketch_identity(const void*, int32_t, int64_t, int64_t, int32_t, int32_t, uint64_t, int64_t, int32_t, int32_t*,
                    void*, int32_t, double*, cudaStream_t);
size_t moments_ws(int64_t, int32_t);
int moments_launch(const int32_t*, const void*, int, int64_t, int32_t, int32_t, double*, double*, void*,
                   cudaStream_t);
int cov_check(int32_t, int32_t);
size_t cov_ws(int64_t, int32_t, int32_t);
int cov_launch(const int32_t*, const void*, int, int64_t, int32_t, int32_t, const double*, double*, void*,
               cudaStream_t);
int cov_finalize_launch(const double*, int32_t, int32_t, int64_t, double*, cudaStream_t);
int adjoint_launch(const double*, int64_t, int32_t, int32_t, uint64_t, int32_t, double, double, double*,
                   cudaStream_t);
int signs_launch(uint64_t, int32_t, int32_t, double*, cudaStream_t);
size_t assign_ws(int64_t, int32_t, int32_t);
int assign_launch(const int32_t*, const void*, int, int64_t, int32_t, const double*, int32_t, int32_t, const int32_t*,
                  int32_t*, double*, int64_t*, double*, void*, cudaStream_t);
int pairwise_launch(const double*, int64_t, double*, void*, cudaStream_t);
size_t pairwise_ws();
size_t partials_ws(int64_t, int32_t, int32_t, int32_t);
size_t csc_ws(int64_t, int32_t, int32_t, int);
size_t seg_ws(int64_t, int32_t, int32_t, int32_t, int);
int csc_build_launch(const int32_t*, const void*, int, int64_t, int32_t, int32_t, void*, cudaStream_t);
int csc_partials_launch(const void*, int, int64_t, int32_t, int32_t, const int32_t*, int32_t, double*, int64_t*,
                        int64_t*, void*, cudaStream_t);
int partials_check(int32_t, int32_t);
int partials_launch(const int32_t*, const void*, int, int64_t, int32_t, const int32_t*, int32_t, int32_t, double*,
                    int64_t*, int64_t*, void*, cudaStream_t);
int centers_launch(const double*, const int64_t*, const int64_t*, const double*, int32_t, int32_t, double*, int32_t*,
                   cudaStream_t);
int reseed_launch(const int32_t*, const void*, int, int32_t, const int32_t*, int32_t, int32_t, double*,
                  cudaStream_t);
int init_launch(const int32_t*, const void*, int, int32_t, const int64_t*, int32_t, int32_t, double*, cudaStream_t);
int row_sqnorms_launch(const void*, int, int64_t, int32_t, double*, cudaStream_t);
bool kmtc_supported(int32_t, int32_t, int32_t);
size_t kmtc_prep_ws(int64_t, int32_t, int32_t);
int kmtc_prepare_launch(const int32_t*, const void*, int, int64_t, int32_t, int32_t, void*, cudaStream_t);
size_t kmtc_assign_ws(int64_t, int32_t, int32_t);
int kmtc_assign_launch(const int32_t*, const void*, int, int64_t, int32_t, const double*, int32_t, int32_t,
                       const int32_t*, int32_t*, double*, int64_t*, double*, const void*, void*, cudaStream_t);
int d2_dense_launch(const int32_t*, const void*, int, int64_t, int32_t, int32_t, const double*, const double*,
                    const double*, double*, cudaStream_t);
int d2_point_launch(const int32_t*, const void*, int, int64_t, int32_t, int32_t, int64_t, const double*, double*,
                    double*, cudaStream_t);

}  // namespace skc

using namespace skc;

static inline cudaStream_t S(void* s) { return reinterpret_cast<cudaStream_t>(s); }
static inline bool pow2(int64_t x) { return x > 0 && (x & (x - 1)) == 0; }
constexpr int32_t kMaxPad = 4096;

static int check_spec(int32_t kind, int32_t p, int32_t p_pad) {
  // PreconditionSpec.__post_init__, transform.py:44-54
  if (kind == SKC_KIND_DCT) return fail(SKC_EPARAM, "dct preconditioner is not on the GPU hot path");
  if (kind != SKC_KIND_HADAMARD && kind != SKC_KIND_NONE) return fail(SKC_EPARAM, "unknown transform kind");
  if (p < 1) return fail(SKC_EDIM, "dimension must be positive");
  if (p_pad < p) return fail(SKC_EDIM, "padded dimension smaller than original");
  if (kind == SKC_KIND_HADAMARD && !pow2(p_pad)) return fail(SKC_EDIM, "hadamard padded dimension must be a power of two");
  if (kind == SKC_KIND_NONE && p_pad != p) return fail(SKC_EDIM, "none transform does not pad");
  if (p_pad > kMaxPad) return fail(SKC_EPARAM, "p_pad > 4096 is not instantiated on the GPU path");
  return SKC_OK;
}
static int check_m(int32_t m, int32_t p_pad) {
  // SamplingPlan.__post_init__, sketch.py:36-38
  if (m < 1 || m > p_pad) {
    char b[96];
    snprintf(b, sizeof b, "need 1 <= m <= p, got m=%d, p=%d", m, p_pad);
    return fail(SKC_EPARAM, b);
  }
  return SKC_OK;
}
static int check_dtype(int32_t d) {
  return (d == SKC_F32 || d == SKC_F64) ? SKC_OK : fail(SKC_EPARAM, "dtype must be SKC_F32 or SKC_F64");
}

extern "C" {

const char* skc_last_error(void) { return g_err.c_str(); }
int skc_abi_version(void) { return 1; }
int32_t skc_max_p_pad(void) { return kMaxPad; }
uint64_t skc_launch_count(void) { return g_launches.load(std::memory_order_relaxed); }
void skc_count_launches(uint64_t kernels) { note_launches((int64_t)kernels); }

int skc_signs(uint64_t sign_seed, int32_t p_pad, int32_t kind, double* out, void* stream) {
  int rc = check_spec(kind, p_pad, p_pad);
  if (rc) return rc;
  return signs_launch(sign_seed, p_pad, kind, out, S(stream));
}

int skc_precondition(const void* X, int32_t x_dtype, int64_t ld, int64_t n, int32_t p, int32_t p_pad, int32_t kind,
                     uint64_t sign_seed, double* Y, void* stream) {
  int rc;
  if ((rc = check_spec(kind, p, p_pad)) || (rc = check_dtype(x_dtype))) return rc;
  if (n < 0 || ld < p) return fail(SKC_EDIM, "expected a (n, p) row block with ld >= p");
  if (n == 0) return SKC_OK;
  if (kind == SKC_KIND_NONE)
    return sketch_identity(X, x_dtype, ld, n, p, p_pad, 0, 0, 1, nullptr, nullptr, SKC_F64, Y, S(stream));
  return sketch_launch(X, x_dtype, ld, n, p, p_pad, kind, sign_seed, 0, 0, 1, SKC_F64, nullptr, nullptr, SKC_F64, Y,
                       S(stream));
}

int skc_unprecondition(const double* Y, int64_t n, int32_t p_pad, int32_t kind, uint64_t sign_seed, int32_t p_out,
                       double* X, void* stream) {
  int rc = check_spec(kind, p_pad, p_pad);
  if (rc) return rc;
  if (p_out < 1 || p_out > p_pad) return fail(SKC_EDIM, "p_out must be in [1, p_pad]");
  return adjoint_launch(Y, n, p_pad, kind, sign_seed, p_out, 0.0, 1.0, X, S(stream));
}

int skc_fwht(const double* Y, int64_t n, int32_t p_pad, double* X, void* stream) {
  if (!pow2(p_pad)) return fail(SKC_EDIM, "length is not a power of two");
  if (p_pad > kMaxPad) return fail(SKC_EPARAM, "p_pad > 4096 is not instantiated on the GPU path");
  return adjoint_launch(Y, n, p_pad, -1, 0, p_pad, 0.0, 1.0, X, S(stream));
}

int skc_indices(uint64_t master_seed, int64_t col0, int64_t n, int32_t p_pad, int32_t m, int32_t* idx_out,
                void* stream) {
  int rc;
  if ((rc = check_m(m, p_pad))) return rc;
  if (p_pad < 1 || p_pad > kMaxPad) return fail(SKC_EPARAM, "p_pad out of range for the GPU sampler");
  if (n <= 0) return SKC_OK;
  return sketch_launch(nullptr, SKC_F32, 0, n, p_pad, p_pad, SKC_KIND_HADAMARD, 0, master_seed, col0, m, SKC_F32,
                       idx_out, nullptr, SKC_F32, nullptr, S(stream));
}

int skc_indices_philox(uint64_t master_seed, int64_t col0, int64_t n, int32_t p_pad, int32_t m, int32_t* idx_out,
                       void* stream) {
  int rc;
  if ((rc = check_m(m, p_pad))) return rc;
  if (p_pad < 1 || p_pad > kMaxPad) return fail(SKC_EPARAM, "p_pad out of range for the GPU sampler");
  if (n <= 0) return SKC_OK;
  return philox_indices_launch(master_seed, col0, n, p_pad, m, idx_out, S(stream));
}

int skc_sketch_given(const void* X, int32_t x_dtype, int64_t ld, int64_t n, int32_t p, int32_t p_pad, int32_t kind,
                     uint64_t sign_seed, int32_t m, int32_t compute_dtype, const int32_t* idx_in, void* val_out,
                     int32_t val_dtype, void* stream) {
  int rc;
  if ((rc = check_spec(kind, p, p_pad)) || (rc = check_m(m, p_pad)) || (rc = check_dtype(x_dtype)) ||
      (rc = check_dtype(compute_dtype)) || (rc = check_dtype(val_dtype)))
    return rc;
  if (n < 0 || ld < p) return fail(SKC_EDIM, "expected a (n, p) row block with ld >= p");
  return sketch_given_launch(X, x_dtype, ld, n, p, p_pad, kind, sign_seed, m, compute_dtype, idx_in, val_out,
                             val_dtype, S(stream));
}

int skc_sketch(const void* X, int32_t x_dtype, int64_t ld, int64_t n, int32_t p, int32_t p_pad, int32_t kind,
               uint64_t sign_seed, uint64_t master_seed, int64_t col0, int32_t m, int32_t compute_dtype,
               int32_t* idx_out, void* val_out, int32_t val_dtype, void* stream) {
  int rc;
  if ((rc = check_spec(kind, p, p_pad)) || (rc = check_m(m, p_pad)) || (rc = check_dtype(x_dtype)) ||
      (rc = check_dtype(compute_dtype)) || (rc = check_dtype(val_dtype)))
    return rc;
  if (n < 0 || ld < p) return fail(SKC_EDIM, "expected a (n, p) row block with ld >= p");
  if (n == 0) return SKC_OK;
  if (kind == SKC_KIND_NONE) {
    return sketch_identity(X, x_dtype, ld, n, p, p_pad, master_seed, col0, m, idx_out, val_out, val_dtype, nullptr,
                           S(stream));
  }
  return sketch_launch(X, x_dtype, ld, n, p, p_pad, kind, sign_seed, master_seed, col0, m, compute_dtype, idx_out,
                       val_out, val_dtype, nullptr, S(stream));
}

size_t skc_moments_workspace(int64_t n, int32_t m, int32_t p_pad) {
  (void)m;
  return moments_ws(n, p_pad);
}

int skc_moments(const int32_t* idx, const void* val, int32_t val_dtype, int64_t n, int32_t m, int32_t p_pad,
                double* acc, double* stats, void* workspace, size_t ws_bytes, void* stream) {
  int rc;
  if ((rc = check_dtype(val_dtype))) return rc;
  if (p_pad < 1 || p_pad > kMaxPad || m < 1 || m > p_pad) return fail(SKC_EDIM, "bad (m, p_pad)");
  if (ws_bytes < moments_ws(n, p_pad)) return fail(SKC_EPARAM, "workspace too small");
  return moments_launch(idx, val, val_dtype == SKC_F64, n, m, p_pad, acc, stats, workspace, S(stream));
}

int skc_mean_finalize(const double* acc, int32_t p, int32_t p_pad, int32_t m, int64_t n_total, int32_t kind,
                      uint64_t sign_seed, double* mean, void* stream) {
  int rc;
  if ((rc = check_spec(kind, p, p_pad))) return rc;
  if (n_total < 1) return fail(SKC_EPARAM, "empty sketch");
  // (p / m) * acc / n, estimators.py:44
  return adjoint_launch(acc, 1, p_pad, kind, sign_seed, p, (double)p_pad / (double)m, (double)n_total, mean,
                        S(stream));
}

size_t skc_cov_workspace(int64_t n, int32_t m, int32_t p_pad) { return cov_ws(n, m, p_pad); }

int skc_cov_accumulate(const int32_t* idx, const void* val, int32_t val_dtype, int64_t n, int32_t m, int32_t p_pad,
                       const double* stats, double* tri, void* workspace, size_t ws_bytes, void* stream) {
  int rc;
  if ((rc = check_dtype(val_dtype))) return rc;
  if (m < 2) return fail(SKC_EPARAM, "covariance estimation needs m >= 2");
  if (p_pad < 1 || p_pad > kMaxPad || m > p_pad) return fail(SKC_EDIM, "bad (m, p_pad)");
  if ((rc = cov_check(p_pad, m))) return rc;
  if (ws_bytes < cov_ws(n, m, p_pad)) return fail(SKC_EPARAM, "workspace too small");
  return cov_launch(idx, val, val_dtype == SKC_F64, n, m, p_pad, stats, tri, workspace, S(stream));
}

int skc_cov_finalize(const double* tri, int32_t p_pad, int32_t m, int64_t n_total, double* C, void* stream) {
  if (m < 2) return fail(SKC_EPARAM, "covariance estimation needs m >= 2");
  if (n_total < 1) return fail(SKC_EPARAM, "empty sketch");
  return cov_finalize_launch(tri, p_pad, m, n_total, C, S(stream));
}

int skc_kmeans_init(const int32_t* idx, const void* val, int32_t val_dtype, int64_t n, int32_t m,
                    const int64_t* chosen, int32_t K, int32_t p_pad, double* mu, void* stream) {
  int rc;
  if ((rc = check_dtype(val_dtype))) return rc;
  if (K < 1) return fail(SKC_EPARAM, "K must be >= 1");
  if (K > n) return fail(SKC_EPARAM, "K exceeds number of points n");
  return init_launch(idx, val, val_dtype == SKC_F64, m, chosen, K, p_pad, mu, S(stream));
}

size_t skc_kmeans_assign_workspace(int64_t n, int32_t p_pad, int32_t K) { return assign_ws(n, p_pad, K); }

int skc_kmeans_assign(const int32_t* idx, const void* val, int32_t val_dtype, int64_t n, int32_t m, const double* mu,
                      int32_t p_pad, int32_t K, const int32_t* prev_labels, int32_t* labels, double* d2min,
                      int64_t* out, double* d2max, void* workspace, size_t ws_bytes, void* stream) {
  int rc;
  if ((rc = check_dtype(val_dtype))) return rc;
  if (K < 1) return fail(SKC_EPARAM, "K must be >= 1");
  if (m < 1 || m > p_pad) return fail(SKC_EDIM, "bad (m, p_pad)");
  if ((size_t)8 * m * 20 > 227 * 1024) return fail(SKC_EPARAM, "m too large for the assignment kernel");
  if (ws_bytes < assign_ws(n, p_pad, K)) return fail(SKC_EPARAM, "workspace too small");
  return assign_launch(idx, val, val_dtype == SKC_F64, n, m, mu, p_pad, K, prev_labels, labels, d2min, out, d2max,
                       workspace, S(stream));
}

int skc_kmeans_tc_supported(int32_t p_pad, int32_t K, int32_t m) { return kmtc_supported(p_pad, K, m) ? 1 : 0; }

size_t skc_kmeans_tc_prepare_workspace(int64_t n, int32_t m, int32_t p_pad) { return kmtc_prep_ws(n, m, p_pad); }

int skc_kmeans_tc_prepare(const int32_t* idx, const void* val, int32_t val_dtype, int64_t n, int32_t m, int32_t p_pad,
                          void* prep, size_t prep_bytes, void* stream) {
  int rc;
  if ((rc = check_dtype(val_dtype))) return rc;
  if (m < 1 || m > p_pad) return fail(SKC_EDIM, "bad (m, p_pad)");
  if (!kmtc_supported(p_pad, 1, m)) return fail(SKC_EPARAM, "tensor-core assignment needs p_pad % 32 == 0");
  if ((size_t)8 * m * 8 > 200 * 1024) return fail(SKC_EPARAM, "m too large for the row-norm kernel");
  if (prep_bytes < kmtc_prep_ws(n, m, p_pad)) return fail(SKC_EPARAM, "workspace too small");
  return kmtc_prepare_launch(idx, val, val_dtype == SKC_F64, n, m, p_pad, prep, S(stream));
}

size_t skc_kmeans_assign_tc_workspace(int64_t n, int32_t p_pad, int32_t K) { return kmtc_assign_ws(n, p_pad, K); }

int skc_kmeans_assign_tc(const int32_t* idx, const void* val, int32_t val_dtype, int64_t n, int32_t m,
                         const double* mu, int32_t p_pad, int32_t K, const int32_t* prev_labels, int32_t* labels,
                         double* d2min, int64_t* out, double* d2max, const void* prep, void* workspace,
                         size_t ws_bytes, void* stream) {
  int rc;
  if ((rc = check_dtype(val_dtype))) return rc;
  if (m < 1 || m > p_pad) return fail(SKC_EDIM, "bad (m, p_pad)");
  if (!kmtc_supported(p_pad, K, m)) return fail(SKC_EPARAM, "tensor-core assignment needs p_pad % 32 == 0, K <= 128");
  if ((size_t)8 * m * 20 > 227 * 1024) return fail(SKC_EPARAM, "m too large for the assignment kernel");
  if (ws_bytes < kmtc_assign_ws(n, p_pad, K)) return fail(SKC_EPARAM, "workspace too small");
  return kmtc_assign_launch(idx, val, val_dtype == SKC_F64, n, m, mu, p_pad, K, prev_labels, labels, d2min, out, d2max,
                            prep, workspace, S(stream));
}

size_t skc_pairwise_sum_workspace(int64_t n) {
  (void)n;
  return pairwise_ws();
}

int skc_pairwise_sum(const double* x, int64_t n, double* out, void* workspace, size_t ws_bytes, void* stream) {
  if (n < 0) return fail(SKC_EDIM, "negative length");
  if (ws_bytes < pairwise_ws()) return fail(SKC_EPARAM, "workspace too small");
  return pairwise_launch(x, n, out, workspace, S(stream));
}

size_t skc_kmeans_partials_workspace(int64_t n, int32_t m, int32_t p_pad, int32_t K) {
  (void)m;
  return partials_ws(n, m, p_pad, K);
}

int skc_kmeans_partials(const int32_t* idx, const void* val, int32_t val_dtype, int64_t n, int32_t m,
                        const int32_t* labels, int32_t p_pad, int32_t K, double* sums, int64_t* counts,
                        int64_t* sizes, void* workspace, size_t ws_bytes, void* stream) {
  int rc;
  if ((rc = check_dtype(val_dtype))) return rc;
  if (K < 1) return fail(SKC_EPARAM, "K must be >= 1");
  if ((rc = partials_check(p_pad, K))) return rc;
  if (ws_bytes < partials_ws(n, m, p_pad, K)) return fail(SKC_EPARAM, "workspace too small");
  return partials_launch(idx, val, val_dtype == SKC_F64, n, m, labels, p_pad, K, sums, counts, sizes, workspace,
                         S(stream));
}

int skc_kmeans_centers(const double* sums, const int64_t* counts, const int64_t* sizes, const double* mu_prev,
                       int32_t p_pad, int32_t K, double* mu_out, int32_t* empty, void* stream) {
  if (K < 1) return fail(SKC_EPARAM, "K must be >= 1");
  return centers_launch(sums, counts, sizes, mu_prev, p_pad, K, mu_out, empty, S(stream));
}

int skc_kmeans_reseed(const int32_t* idx_c, const void* val_c, int32_t val_dtype, int32_t m, const int32_t* empty,
                      int32_t p_pad, int32_t K, double* mu, void* stream) {
  int rc;
  if ((rc = check_dtype(val_dtype))) return rc;
  return reseed_launch(idx_c, val_c, val_dtype == SKC_F64, m, empty, p_pad, K, mu, S(stream));
}

int skc_kmeans_reseed_at(const int32_t* idx, const void* val, int32_t val_dtype, int64_t n, int32_t m,
                         const int64_t* row, const int32_t* empty, int32_t p_pad, int32_t K, double* mu, void* stream) {
  int rc;
  if ((rc = check_dtype(val_dtype))) return rc;
  if (n < 1) return fail(SKC_EDIM, "empty sketch");
  return reseed_at_launch(idx, val, val_dtype == SKC_F64, m, reinterpret_cast<const long long*>(row), empty, p_pad, K,
                          mu, S(stream));
}

size_t skc_kmeans_csc_workspace(int64_t n, int32_t m, int32_t p_pad, int32_t val_dtype) {
  return csc_ws(n, m, p_pad, val_dtype == SKC_F64);
}

int skc_kmeans_build_csc(const int32_t* idx, const void* val, int32_t val_dtype, int64_t n, int32_t m, int32_t p_pad,
                         void* csc, size_t csc_bytes, void* stream) {
  int rc;
  if ((rc = check_dtype(val_dtype))) return rc;
  if ((rc = partials_check(p_pad, 1))) return rc;
  if (csc_bytes < csc_ws(n, m, p_pad, val_dtype == SKC_F64)) return fail(SKC_EPARAM, "workspace too small");
  return csc_build_launch(idx, val, val_dtype == SKC_F64, n, m, p_pad, csc, S(stream));
}

size_t skc_kmeans_seg_workspace(int64_t n, int32_t m, int32_t p_pad, int32_t K, int32_t val_dtype) {
  return seg_ws(n, m, p_pad, K, val_dtype == SKC_F64);
}

int skc_kmeans_partials_csc(const void* csc, int32_t val_dtype, int64_t n, int32_t m, int32_t p_pad,
                            const int32_t* labels, int32_t K, double* sums, int64_t* counts, int64_t* sizes, void* seg,
                            size_t seg_bytes, void* stream) {
  int rc;
  if ((rc = check_dtype(val_dtype))) return rc;
  if ((rc = partials_check(p_pad, K))) return rc;
  if (seg_bytes < seg_ws(n, m, p_pad, K, val_dtype == SKC_F64)) return fail(SKC_EPARAM, "workspace too small");
  return csc_partials_launch(csc, val_dtype == SKC_F64, n, m, p_pad, labels, K, sums, counts, sizes, seg, S(stream));
}

int skc_row_sqnorms(const void* val, int32_t val_dtype, int64_t n, int32_t m, double* out, void* stream) {
  int rc;
  if ((rc = check_dtype(val_dtype))) return rc;
  return row_sqnorms_launch(val, val_dtype == SKC_F64, n, m, out, S(stream));
}

int skc_kmeans_d2_to_point(const int32_t* idx, const void* val, int32_t val_dtype, int64_t n, int32_t m,
                           int32_t p_pad, int64_t c, const double* colsq, double* dense, double* out, void* stream) {
  int rc;
  if ((rc = check_dtype(val_dtype))) return rc;
  if (c < 0 || c >= n) return fail(SKC_EPARAM, "point index out of range");
  return d2_point_launch(idx, val, val_dtype == SKC_F64, n, m, p_pad, c, colsq, dense, out, S(stream));
}

int skc_kmeans_d2_to_dense(const int32_t* idx, const void* val, int32_t val_dtype, int64_t n, int32_t m,
                           int32_t p_pad, const double* dense, const double* dense_sq, const double* colsq, double* out,
                           void* stream) {
  int rc;
  if ((rc = check_dtype(val_dtype))) return rc;
  if (n < 0 || m < 1 || p_pad < 1) return fail(SKC_EDIM, "need n >= 0, m >= 1 and p_pad >= 1");
  return d2_dense_launch(idx, val, val_dtype == SKC_F64, n, m, p_pad, dense, dense_sq, colsq, out, S(stream));
}

int skc_sketch_pack_records(const int32_t* idx, const void* val, int32_t val_dtype, int64_t n, int32_t m,
                            uint32_t* out_words, void* stream) {
  int rc;
  if ((rc = check_dtype(val_dtype))) return rc;
  if (n < 0 || m < 1) return fail(SKC_EDIM, "need n >= 0 and m >= 1");
  return pack_records_launch(idx, val, val_dtype == SKC_F64, n, m, out_words, S(stream));
}

int skc_sketch_unpack_records(const uint32_t* words, int64_t n, int32_t m, int32_t* idx_out, double* val_out,
                              void* stream) {
  if (n < 0 || m < 1) return fail(SKC_EDIM, "need n >= 0 and m >= 1");
  return unpack_records_launch(words, n, m, idx_out, val_out, S(stream));
}

static int check_dense(int32_t x_dtype, int64_t ld, int64_t n, int32_t p, int32_t K) {
  int rc;
  if ((rc = check_dtype(x_dtype))) return rc;
  if (n < 0 || p < 1 || ld < p) return fail(SKC_EDIM, "need n >= 0, p >= 1 and ld >= p");
  if (K < 1) return fail(SKC_EPARAM, "need K >= 1");
  return SKC_OK;
}

size_t skc_dense_assign_workspace(int32_t p, int32_t K) { return dense_assign_ws(p, K); }

int skc_dense_assign(const void* X, int32_t x_dtype, int64_t ld, int64_t n, int32_t p, const double* mu, int32_t K,
                     void* ws, int32_t* labels, double* d2min, void* stream) {
  int rc;
  if ((rc = check_dense(x_dtype, ld, n, p, K))) return rc;
  return dense_assign_launch(X, x_dtype == SKC_F64, ld, n, p, mu, K, reinterpret_cast<double*>(ws), labels, d2min,
                             S(stream));
}

size_t skc_dense_sums_workspace(int64_t n, int32_t p, int32_t K) { return dense_sums_ws(n, p, K); }

int skc_dense_sums(const void* X, int32_t x_dtype, int64_t ld, int64_t n, int32_t p, const int32_t* labels, int32_t K,
                   double* sums, int64_t* counts, void* ws, void* stream) {
  int rc;
  if ((rc = check_dense(x_dtype, ld, n, p, K))) return rc;
  return dense_sums_launch(X, x_dtype == SKC_F64, ld, n, p, labels, K, sums, reinterpret_cast<long long*>(counts), ws,
                           S(stream));
}

// ---- native streaming runtime (stream_moments' loop in C++) ------------------------
struct StreamLayout {
  size_t off_buf[2], off_idx, off_val, off_mws, off_cws, total;
};

static StreamLayout stream_layout(int64_t chunk, int32_t p, int32_t p_pad, int32_t m, int x_f64, int v_f64, int cov) {
  StreamLayout L{};
  size_t o = 0;
  auto take = [&](size_t bytes) {
    const size_t r = o;
    o += (bytes + 255) & ~(size_t)255;
    return r;
  };
  const size_t rows_bytes = (size_t)chunk * p * (x_f64 ? 8 : 4);
  L.off_buf[0] = take(rows_bytes);
  L.off_buf[1] = take(rows_bytes);
  L.off_idx = take((size_t)chunk * m * 4);
  L.off_val = take((size_t)chunk * m * (v_f64 ? 8 : 4));
  L.off_mws = take(moments_ws(chunk, p_pad));
  L.off_cws = take(cov ? cov_ws(chunk, m, p_pad) : 1);
  L.total = o;
  return L;
}

size_t skc_stream_workspace(int64_t chunk_rows, int32_t p, int32_t p_pad, int32_t m, int32_t x_dtype,
                            int32_t compute_dtype, int32_t covariance) {
  if (chunk_rows < 1 || p < 1 || p_pad < p || m < 1) return 0;
  return stream_layout(chunk_rows, p, p_pad, m, x_dtype == SKC_F64, compute_dtype == SKC_F64, covariance).total;
}

int skc_stream_moments(const void* host_X, int32_t x_dtype, int64_t ld, int64_t n, int32_t p, int32_t p_pad,
                       int32_t kind, uint64_t sign_seed, uint64_t master_seed, int64_t col0, int32_t m,
                       int32_t compute_dtype, int32_t sampler, int64_t chunk_rows, double* acc, double* stats,
                       double* tri, void* ws, size_t ws_bytes, void* stream) {
  int rc;
  if ((rc = check_spec(kind, p, p_pad)) || (rc = check_m(m, p_pad)) || (rc = check_dtype(x_dtype)) ||
      (rc = check_dtype(compute_dtype)))
    return rc;
  if (n < 0 || ld < p) return fail(SKC_EDIM, "expected a (n, p) row block with ld >= p");
  if (chunk_rows < 1) return fail(SKC_EPARAM, "chunk_rows must be >= 1");
  if (sampler != 0 && sampler != 1) return fail(SKC_EPARAM, "sampler must be 0 (oracle) or 1 (philox)");
  if (tri != nullptr && (m < 2 || (rc = cov_check(p_pad, m)))) return m < 2 ? fail(SKC_EPARAM, "covariance needs m >= 2") : rc;
  const int x_f64 = x_dtype == SKC_F64, v_f64 = compute_dtype == SKC_F64;
  const StreamLayout L = stream_layout(chunk_rows, p, p_pad, m, x_f64, v_f64, tri != nullptr);
  if (ws_bytes < L.total) return fail(SKC_EPARAM, "workspace too small");
  if (n == 0) return SKC_OK;
  char* w = static_cast<char*>(ws);
  const size_t es = x_f64 ? 8 : 4;
  cudaStream_t cs = S(stream), cp;
  if (cudaStreamCreateWithFlags(&cp, cudaStreamNonBlocking) != cudaSuccess) return check_launch("copy stream");
  cudaEvent_t copied[2], freed[2];
  for (int b = 0; b < 2; ++b) {
    cudaEventCreateWithFlags(&copied[b], cudaEventDisableTiming);
    cudaEventCreateWithFlags(&freed[b], cudaEventDisableTiming);
  }
  int32_t* idx = reinterpret_cast<int32_t*>(w + L.off_idx);
  void* val = w + L.off_val;
  rc = SKC_OK;
  int64_t k = 0;
  for (int64_t c0 = 0; c0 < n && rc == SKC_OK; c0 += chunk_rows, ++k) {
    const int64_t rows = n - c0 < chunk_rows ? n - c0 : chunk_rows;
    const int b = (int)(k & 1);
    void* buf = w + L.off_buf[b];
    if (k >= 2) cudaStreamWaitEvent(cp, freed[b], 0);  // K1 of chunk k-2 has read this buffer
    if (cudaMemcpy2DAsync(buf, (size_t)p * es, static_cast<const char*>(host_X) + (size_t)c0 * ld * es, (size_t)ld * es,
                          (size_t)p * es, (size_t)rows, cudaMemcpyHostToDevice, cp) != cudaSuccess) {
      rc = check_launch("chunk copy");
      break;
    }
    cudaEventRecord(copied[b], cp);
    cudaStreamWaitEvent(cs, copied[b], 0);
    if (kind == SKC_KIND_NONE) {
      if (sampler == 1) {
        rc = philox_indices_launch(master_seed, col0 + c0, rows, p_pad, m, idx, cs);
        if (!rc) rc = sketch_given_launch(buf, x_dtype, p, rows, p, p_pad, kind, sign_seed, m, compute_dtype, idx, val,
                                          compute_dtype, cs);
      } else {
        rc = sketch_identity(buf, x_dtype, p, rows, p, p_pad, master_seed, col0 + c0, m, idx, val, compute_dtype,
                             nullptr, cs);
      }
    } else if (sampler == 1) {
      rc = philox_indices_launch(master_seed, col0 + c0, rows, p_pad, m, idx, cs);
      if (!rc) rc = sketch_given_launch(buf, x_dtype, p, rows, p, p_pad, kind, sign_seed, m, compute_dtype, idx, val,
                                        compute_dtype, cs);
    } else {
      rc = sketch_launch(buf, x_dtype, p, rows, p, p_pad, kind, sign_seed, master_seed, col0 + c0, m, compute_dtype, idx,
                         val, compute_dtype, nullptr, cs);
    }
    cudaEventRecord(freed[b], cs);
    if (!rc) rc = moments_launch(idx, val, v_f64, rows, m, p_pad, acc, stats, w + L.off_mws, cs);
    if (!rc && tri != nullptr) rc = cov_launch(idx, val, v_f64, rows, m, p_pad, stats, tri, w + L.off_cws, cs);
  }
  for (int b = 0; b < 2; ++b) {
    cudaEventDestroy(copied[b]);
    cudaEventDestroy(freed[b]);
  }
  cudaStreamDestroy(cp);  // released once its queued copies finish
  return rc;
}

}  // extern "C"
