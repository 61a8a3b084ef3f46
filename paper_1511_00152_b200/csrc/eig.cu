// Top-k eigenvectors of the resident covariance on the device: the
// solver="device" alternative to top_eigenvectors' host LAPACK eigh (estimators.py:69-81).
// cuSOLVER syevdx with an index range computes only the k largest eigenpairs of
// 0.5 * (C + C^T) (tridiagonal reduction, bisection on the k wanted eigenvalues, inverse
// iteration and back-transformation of k vectors) instead of the full spectrum of syevd.
// The columns come out in descending eigenvalue order, as the reference's V[:, ::-1][:, :k].
#include <cusolverDn.h>

#include <mutex>
#include <string>

#include "common.cuh"

namespace skc {
namespace {

__global__ void symmetrize_kernel(const double* __restrict__ C, int p, double* __restrict__ A) {
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= (int64_t)p * p) return;
  const int a = (int)(e / p), b = (int)(e % p);
  A[e] = dmul(0.5, dadd(C[e], C[(int64_t)b * p + a]));  // np: 0.5 * (C + C.T)
}

// A (column-major, p x p) holds the k eigenvectors in ascending eigenvalue order in its first
// k columns; V (p, k) row-major gets them in descending order: V[i, c] = A[i, k-1-c].
__global__ void take_topk_kernel(const double* __restrict__ A, const double* __restrict__ W, int p, int k,
                                 double* __restrict__ V, double* __restrict__ w) {
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e < (int64_t)p * k) {
    const int i = (int)(e / k), c = (int)(e % k);
    V[e] = A[(int64_t)(k - 1 - c) * p + i];
  }
  if (w != nullptr && e < k) w[e] = W[k - 1 - e];
}

struct Solver {
  cusolverDnHandle_t h = nullptr;
};
Solver& solver_for_thread() {
  thread_local Solver S;
  if (S.h == nullptr) cusolverDnCreate(&S.h);
  return S;
}

size_t align256(size_t x) { return (x + 255) & ~(size_t)255; }

int eig_fail(cusolverStatus_t s, const char* what) {
  return fail(SKC_ECUDA, std::string(what) + ": cusolver status " + std::to_string((int)s));
}

}  // namespace
}  // namespace skc

using namespace skc;

extern "C" {

size_t skc_top_eigenvectors_workspace(int32_t p, int32_t k) {
  if (p < 1 || k < 1 || k > p) return 0;
  Solver& S = solver_for_thread();
  int lwork = 0;
  double vl = 0.0, vu = 0.0;
  int meig = 0;
  if (cusolverDnDsyevdx_bufferSize(S.h, CUSOLVER_EIG_MODE_VECTOR, CUSOLVER_EIG_RANGE_I, CUBLAS_FILL_MODE_LOWER, p,
                                   nullptr, p, vl, vu, p - k + 1, p, &meig, nullptr, &lwork) != CUSOLVER_STATUS_SUCCESS)
    return 0;
  return align256((size_t)p * p * 8) + align256((size_t)p * 8) + align256((size_t)lwork * 8) + 256;
}

int skc_top_eigenvectors(const double* C, int32_t p, int32_t k, double* V, double* w, void* ws, size_t ws_bytes,
                         void* stream) {
  if (p < 1 || k < 1 || k > p) return fail(SKC_EPARAM, "need 1 <= k <= p");
  const size_t need = skc_top_eigenvectors_workspace(p, k);
  if (need == 0) return fail(SKC_ECUDA, "cusolverDnDsyevdx_bufferSize failed");
  if (ws_bytes < need) return fail(SKC_EPARAM, "workspace too small");
  Solver& S = solver_for_thread();
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  cusolverDnSetStream(S.h, st);
  char* base = static_cast<char*>(ws);
  double* A = reinterpret_cast<double*>(base);
  double* W = reinterpret_cast<double*>(base + align256((size_t)p * p * 8));
  double* work = reinterpret_cast<double*>(base + align256((size_t)p * p * 8) + align256((size_t)p * 8));
  int* info = reinterpret_cast<int*>(base + need - 256);
  const int lwork = (int)((need - 256 - align256((size_t)p * p * 8) - align256((size_t)p * 8)) / 8);
  const int64_t total = (int64_t)p * p;
  symmetrize_kernel<<<(unsigned)((total + 255) / 256), 256, 0, st>>>(C, p, A);
  int rc = check_launch("symmetrize_kernel");
  if (rc) return rc;
  int meig = 0;
  const cusolverStatus_t s =
      cusolverDnDsyevdx(S.h, CUSOLVER_EIG_MODE_VECTOR, CUSOLVER_EIG_RANGE_I, CUBLAS_FILL_MODE_LOWER, p, A, p, 0.0, 0.0,
                        p - k + 1, p, &meig, W, work, lwork, info);
  if (s != CUSOLVER_STATUS_SUCCESS) return eig_fail(s, "cusolverDnDsyevdx");
  const int64_t outn = (int64_t)p * k;
  take_topk_kernel<<<(unsigned)((outn + 255) / 256), 256, 0, st>>>(A, W, p, k, V, w);
  return check_launch("take_topk_kernel");
}

}  // extern "C"
