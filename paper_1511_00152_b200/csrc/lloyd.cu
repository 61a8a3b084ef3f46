// Device-resident Lloyd loop: the _lloyd_iterate loop body (cluster.py:230-241) from given
// centres, as ONE CUDA graph with a conditional WHILE node, so the iterations run with no host
// round trip (the convergence test of cluster.py:235-236 is evaluated on the device).
//
// Graph (built once per buffer set, cached, relaunched per call):
//   copy mu0 -> mu, state = 0
//   iteration 1 (prologue):   assign (K5/K5f, no previous labels) -> objective (numpy pairwise
//                             order) -> check -> partials -> centres -> reseed -> commit
//   WHILE (cond):             assign (K5t filter when prepared, else K5; changed count against
//                             the previous labels) -> objective -> check -> partials -> centres
//                             -> reseed -> commit
//   copy state.it -> iters
// check (one thread): traj[it] = objective; converged = (it > 1 && changed == 0);
//   cond = !converged && it < max_iter (cudaGraphSetConditional).
// The update after the check is speculative; commit keeps it (mu = mu_next, previous labels =
// current labels) only when the iteration did not converge, which is exactly the reference's
// "break before update" order. Every kernel is the same one the host-driven loop launches, so
// labels, centres and the objective trajectory are bit-identical to it.
#include <map>
#include <mutex>
#include <tuple>
#include <vector>

#include "common.cuh"

namespace skc {

size_t assign_ws(int64_t, int32_t, int32_t);
size_t kmtc_assign_ws(int64_t, int32_t, int32_t);
size_t pairwise_ws();
int pairwise_leaves_launch(const double* x, int64_t n, void* ws, int* D_out, cudaStream_t st);
size_t seg_ws(int64_t, int32_t, int32_t, int32_t, int);
void note_launches(int64_t delta);

namespace {

__global__ void lloyd_check_kernel(const int64_t* __restrict__ out, const double* __restrict__ obj,
                                   double* __restrict__ traj, int32_t* __restrict__ state, int max_iter, int first,
                                   cudaGraphConditionalHandle cond) {
  const int it = state[0] + 1;  // iterations executed, this assignment included
  traj[it - 1] = *obj;
  const int conv = (!first && out[0] == 0) ? 1 : 0;
  state[0] = it;
  state[1] = conv;
  cudaGraphSetConditional(cond, (!conv && it < max_iter) ? 1u : 0u);
}

__global__ void lloyd_commit_kernel(const int32_t* __restrict__ state, const double* __restrict__ mu_next,
                                    double* __restrict__ mu, int64_t pk, const int32_t* __restrict__ cur,
                                    int32_t* __restrict__ prev, int64_t n) {
  if (state[1]) return;  // converged: the centres of the final assignment stay
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < pk; i += stride) mu[i] = mu_next[i];
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += stride) prev[i] = cur[i];
}

// Fused tail of an iteration (SKC_LLOYD_FUSED=0 keeps the kernel-per-step sequence above).
// objcheck: the objective's subtree sums combined level by level (pairwise_combine_kernel's
// order), then the convergence check. One block.
constexpr int kPwDeepL = 14;  // = kPwDeep of the pairwise sum
__global__ void __launch_bounds__(1024) lloyd_objcheck_kernel(const double* __restrict__ gres,
                                                              const uint8_t* __restrict__ gld, int D,
                                                              const int64_t* __restrict__ out,
                                                              double* __restrict__ obj, double* __restrict__ traj,
                                                              int32_t* __restrict__ state, int max_iter, int first,
                                                              cudaGraphConditionalHandle cond) {
  extern __shared__ double lres[];
  uint8_t* ld = reinterpret_cast<uint8_t*>(lres + (1 << D));
  for (int t = threadIdx.x; t < (1 << D); t += blockDim.x) lres[t] = gres[t], ld[t] = gld[t];
  __syncthreads();
  for (int d = D - 1; d >= 0; --d) {
    const int sh = D - d;
    for (int t = threadIdx.x; t < (1 << d); t += blockDim.x)
      if (ld[t << sh] > d) lres[t << sh] = dadd(lres[(2 * t) << (sh - 1)], lres[(2 * t + 1) << (sh - 1)]);
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    const int it = state[0] + 1;  // iterations executed, this assignment included
    obj[0] = lres[0];
    traj[it - 1] = lres[0];
    const int conv = (!first && out[0] == 0) ? 1 : 0;
    state[0] = it;
    state[1] = conv;
    cudaGraphSetConditional(cond, (!conv && it < max_iter) ? 1u : 0u);
  }
}

// finish: centres, reseed and commit in one kernel (cluster.py:207-215, :238-241). Block (k, s)
// takes column k's coordinates [p s / S, p (s + 1) / S). The cluster's size is sum_j counts[j][k] / m
// (every point holds m coordinates), so only "empty or not" is needed: the sum is
// zero. A non-empty cluster's centre is sums / counts where counts > 0, else the previous value
// (left in place); an empty cluster takes the farthest point's column (zero elsewhere), the
// same point for every empty cluster. Nothing is written once the iteration converged (the
// update is speculative, the reference breaks before it); the labels become the previous labels.
template <typename V>
__global__ void __launch_bounds__(256) lloyd_finish_kernel(const int32_t* __restrict__ state,
                                                           const double* __restrict__ sums,
                                                           const int64_t* __restrict__ counts, int m, int p_pad, int K,
                                                           int S, const int32_t* __restrict__ idx,
                                                           const V* __restrict__ val, const int64_t* __restrict__ row,
                                                           double* __restrict__ mu, const int32_t* __restrict__ cur,
                                                           int32_t* __restrict__ prev, int64_t n) {
  if (state[1]) return;
  const int k = blockIdx.x % K, s = blockIdx.x / K;
  __shared__ long long red[8];
  long long c = 0;
  for (int j = threadIdx.x; j < p_pad; j += blockDim.x) c += counts[(int64_t)j * K + k];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xFFFFFFFFu, c, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = c;
  __syncthreads();
  long long tot = 0;
  for (int w = 0; w < (int)(blockDim.x >> 5); ++w) tot += red[w];
  const int j0 = (int)((int64_t)p_pad * s / S), j1 = (int)((int64_t)p_pad * (s + 1) / S);
  if (tot != 0) {
    for (int j = j0 + threadIdx.x; j < j1; j += blockDim.x) {
      const int64_t e = (int64_t)j * K + k;
      const int64_t cn = counts[e];
      if (cn != 0) mu[e] = __ddiv_rn(sums[e], (double)cn);
    }
  } else {
    const int64_t r = *row > 0 ? *row : 0;
    const int32_t* ir = idx + r * m;
    const V* vr = val + r * m;
    for (int j = j0 + threadIdx.x; j < j1; j += blockDim.x) {
      double v = 0.0;
      for (int t = 0; t < m; ++t)
        if (__ldg(ir + t) == j) v = (double)__ldg(vr + t);
      mu[(int64_t)j * K + k] = v;
    }
  }
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += stride) prev[i] = cur[i];
}

struct Carve {
  size_t off = 0;
  template <typename T>
  T* take(char* base, size_t count) {
    T* p = base ? reinterpret_cast<T*>(base + off) : nullptr;
    off += (count * sizeof(T) + 255) & ~(size_t)255;
    return p;
  }
};

struct Bufs {
  int32_t* prev;
  double* d2min;
  int64_t* out;
  double* d2max;
  double* obj;
  int32_t* state;
  double* mu_next;
  double* sums;
  int64_t* counts;
  int64_t* sizes;
  int32_t* empty;
  void* aws;
  size_t aws_bytes;
  void* pws;
  size_t pws_bytes;
  void* sws;
  size_t sws_bytes;
};

Bufs carve(char* base, int64_t n, int32_t m, int32_t p_pad, int32_t K, int32_t vdt, bool tc, size_t* total) {
  Carve c;
  Bufs b;
  const size_t pk = (size_t)p_pad * K;
  b.prev = c.take<int32_t>(base, n);
  b.d2min = c.take<double>(base, n);
  b.out = c.take<int64_t>(base, 2);
  b.d2max = c.take<double>(base, 1);
  b.obj = c.take<double>(base, 1);
  b.state = c.take<int32_t>(base, 2);
  b.mu_next = c.take<double>(base, pk);
  b.sums = c.take<double>(base, pk);
  b.counts = c.take<int64_t>(base, pk);
  b.sizes = c.take<int64_t>(base, K);
  b.empty = c.take<int32_t>(base, K);
  size_t a = assign_ws(n, p_pad, K);
  if (tc) {
    const size_t t = kmtc_assign_ws(n, p_pad, K);
    a = t > a ? t : a;
  }
  b.aws_bytes = a;
  b.aws = c.take<char>(base, a);
  b.pws_bytes = pairwise_ws();
  b.pws = c.take<char>(base, b.pws_bytes);
  b.sws_bytes = seg_ws(n, m, p_pad, K, vdt);
  b.sws = c.take<char>(base, b.sws_bytes);
  if (total) *total = c.off;
  return b;
}

struct Entry {
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t exec = nullptr;
  int prologue_kernels = 0, body_kernels = 0;
  uint64_t stamp = 0;
};
using Key = std::tuple<const void*, const void*, int64_t, int32_t, int32_t, int32_t, int32_t, const void*, int32_t,
                       const void*, const void*, const void*, size_t, const void*, const void*, const void*,
                       const void*, int>;
std::mutex g_mu;
std::map<Key, Entry> g_cache;
uint64_t g_stamp = 0;
thread_local int g_last_prologue = 0, g_last_body = 0;

struct Args {
  const int32_t* idx;
  const void* val;
  int32_t vdt;
  int64_t n;
  int32_t m, p_pad, K;
  const double* mu0;
  int32_t max_iter;
  const void* csc;
  const void* prep;
  int32_t* labels;
  double* mu;
  double* traj;
  int32_t* iters;
};

// side stream and fork / join events of one captured iteration (the fused tail runs the
// objective branch beside the partial sums)
struct Side {
  cudaStream_t st = nullptr;
  cudaEvent_t fork = nullptr, join = nullptr;
  bool make() {
    return cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking) == cudaSuccess &&
           cudaEventCreateWithFlags(&fork, cudaEventDisableTiming) == cudaSuccess &&
           cudaEventCreateWithFlags(&join, cudaEventDisableTiming) == cudaSuccess;
  }
  ~Side() {
    if (fork) cudaEventDestroy(fork);
    if (join) cudaEventDestroy(join);
    if (st) cudaStreamDestroy(st);
  }
};

static bool fused_on() {
  const char* e = getenv("SKC_LLOYD_FUSED");
  return !(e && e[0] == '0');
}

// one iteration's launches on stream s; returns SKC_OK or the first error
int iteration(const Args& A, const Bufs& B, bool first, cudaGraphConditionalHandle cond, cudaStream_t s, Side& sd) {
  int rc;
  const int32_t* prev = first ? nullptr : B.prev;
  if (!first && A.prep != nullptr)
    rc = skc_kmeans_assign_tc(A.idx, A.val, A.vdt, A.n, A.m, A.mu, A.p_pad, A.K, prev, A.labels, B.d2min, B.out,
                              B.d2max, A.prep, B.aws, B.aws_bytes, s);
  else
    rc = skc_kmeans_assign(A.idx, A.val, A.vdt, A.n, A.m, A.mu, A.p_pad, A.K, prev, A.labels, B.d2min, B.out,
                           B.d2max, B.aws, B.aws_bytes, s);
  if (rc) return rc;
  if (fused_on()) {
    // assign -> { objective leaves -> combine + check } || { partial sums } -> finish
    if (cudaEventRecord(sd.fork, s) != cudaSuccess || cudaStreamWaitEvent(sd.st, sd.fork, 0) != cudaSuccess)
      return check_launch("lloyd fork");
    if ((rc = skc_kmeans_partials_csc(A.csc, A.vdt, A.n, A.m, A.p_pad, A.labels, A.K, B.sums, B.counts, nullptr,
                                      B.sws, B.sws_bytes, sd.st)))
      return rc;
    int D = 0;
    if ((rc = pairwise_leaves_launch(B.d2min, A.n, B.pws, &D, s))) return rc;
    const size_t osm = ((size_t)1 << D) * 9 + 16;
    cudaFuncSetAttribute(lloyd_objcheck_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)osm);
    lloyd_objcheck_kernel<<<1, 1024, osm, s>>>(reinterpret_cast<const double*>(B.pws),
                                               reinterpret_cast<const uint8_t*>(B.pws) + ((size_t)8 << kPwDeepL), D,
                                               B.out, B.obj, A.traj, B.state, A.max_iter, first ? 1 : 0, cond);
    if ((rc = check_launch("lloyd_objcheck_kernel"))) return rc;
    if (cudaEventRecord(sd.join, sd.st) != cudaSuccess || cudaStreamWaitEvent(s, sd.join, 0) != cudaSuccess)
      return check_launch("lloyd join");
    int S = (2 * sm_count() + A.K - 1) / A.K;
    if (S < 1) S = 1;
    if (S > A.p_pad) S = A.p_pad;
    if (A.vdt == SKC_F64)
      lloyd_finish_kernel<double><<<(unsigned)(A.K * S), 256, 0, s>>>(
          B.state, B.sums, B.counts, A.m, A.p_pad, A.K, S, A.idx, static_cast<const double*>(A.val), B.out + 1, A.mu,
          A.labels, B.prev, A.n);
    else
      lloyd_finish_kernel<float><<<(unsigned)(A.K * S), 256, 0, s>>>(
          B.state, B.sums, B.counts, A.m, A.p_pad, A.K, S, A.idx, static_cast<const float*>(A.val), B.out + 1, A.mu,
          A.labels, B.prev, A.n);
    return check_launch("lloyd_finish_kernel");
  }
  if ((rc = skc_pairwise_sum(B.d2min, A.n, B.obj, B.pws, B.pws_bytes, s))) return rc;
  lloyd_check_kernel<<<1, 1, 0, s>>>(B.out, B.obj, A.traj, B.state, A.max_iter, first ? 1 : 0, cond);
  if ((rc = check_launch("lloyd_check_kernel"))) return rc;
  if ((rc = skc_kmeans_partials_csc(A.csc, A.vdt, A.n, A.m, A.p_pad, A.labels, A.K, B.sums, B.counts, B.sizes, B.sws,
                                    B.sws_bytes, s)))
    return rc;
  if ((rc = skc_kmeans_centers(B.sums, B.counts, B.sizes, A.mu, A.p_pad, A.K, B.mu_next, B.empty, s))) return rc;
  if ((rc = skc_kmeans_reseed_at(A.idx, A.val, A.vdt, A.n, A.m, B.out + 1, B.empty, A.p_pad, A.K, B.mu_next, s)))
    return rc;
  const int64_t pk = (int64_t)A.p_pad * A.K;
  const int64_t work = A.n > pk ? A.n : pk;
  int64_t blocks = (work + 255) / 256;
  if (blocks > 4 * (int64_t)sm_count()) blocks = 4 * (int64_t)sm_count();
  lloyd_commit_kernel<<<(unsigned)(blocks < 1 ? 1 : blocks), 256, 0, s>>>(B.state, B.mu_next, A.mu, pk, A.labels,
                                                                          B.prev, A.n);
  return check_launch("lloyd_commit_kernel");
}

int build(const Args& A, const Bufs& B, Entry& E) {
  cudaGraph_t g = nullptr;
  if (cudaGraphCreate(&g, 0) != cudaSuccess) return check_launch("cudaGraphCreate");
  cudaGraphConditionalHandle cond;
  if (cudaGraphConditionalHandleCreate(&cond, g, 0, cudaGraphCondAssignDefault) != cudaSuccess) {
    cudaGraphDestroy(g);
    return check_launch("cudaGraphConditionalHandleCreate");
  }
  cudaStream_t s1 = nullptr, s2 = nullptr;
  cudaStreamCreateWithFlags(&s1, cudaStreamNonBlocking);
  cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking);
  int rc = SKC_OK;
  Side sd1, sd2;  // prologue / body
  auto done = [&](int code) {
    cudaStreamDestroy(s1);
    cudaStreamDestroy(s2);
    if (code != SKC_OK) cudaGraphDestroy(g);
    return code;
  };
  if (!sd1.make() || !sd2.make()) return done(check_launch("lloyd side streams"));
  if (cudaStreamBeginCaptureToGraph(s1, g, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed) != cudaSuccess)
    return done(check_launch("begin capture"));
  cudaMemcpyAsync(A.mu, A.mu0, sizeof(double) * A.p_pad * A.K, cudaMemcpyDeviceToDevice, s1);
  cudaMemsetAsync(B.state, 0, 2 * sizeof(int32_t), s1);
  const uint64_t l0 = skc_launch_count();
  rc = iteration(A, B, true, cond, s1, sd1);
  const uint64_t l1 = skc_launch_count();
  cudaStreamCaptureStatus status;
  const cudaGraphNode_t* deps = nullptr;
  size_t ndeps = 0;
  cudaGraph_t cg = nullptr;
  if (rc == SKC_OK && cudaStreamGetCaptureInfo(s1, &status, nullptr, &cg, &deps, &ndeps) != cudaSuccess)
    rc = check_launch("capture info");
  cudaGraphNode_t cnode = nullptr;
  cudaGraph_t body = nullptr;
  if (rc == SKC_OK) {
    cudaGraphNodeParams cp = {};
    cp.type = cudaGraphNodeTypeConditional;
    cp.conditional.handle = cond;
    cp.conditional.type = cudaGraphCondTypeWhile;
    cp.conditional.size = 1;
    if (cudaGraphAddNode(&cnode, cg, deps, ndeps, &cp) != cudaSuccess) rc = check_launch("add conditional node");
    else body = cp.conditional.phGraph_out[0];
  }
  if (rc == SKC_OK && cudaStreamUpdateCaptureDependencies(s1, &cnode, 1, cudaStreamSetCaptureDependencies) !=
                          cudaSuccess)
    rc = check_launch("update capture dependencies");
  uint64_t l2 = l1, l3 = l1;
  if (rc == SKC_OK) {
    if (cudaStreamBeginCaptureToGraph(s2, body, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed) != cudaSuccess) {
      rc = check_launch("begin body capture");
    } else {
      l2 = skc_launch_count();
      rc = iteration(A, B, false, cond, s2, sd2);
      l3 = skc_launch_count();
      cudaGraph_t bo = nullptr;
      if (cudaStreamEndCapture(s2, &bo) != cudaSuccess && rc == SKC_OK) rc = check_launch("end body capture");
    }
  }
  if (rc == SKC_OK) cudaMemcpyAsync(A.iters, B.state, sizeof(int32_t), cudaMemcpyDeviceToDevice, s1);
  cudaGraph_t go = nullptr;
  if (cudaStreamEndCapture(s1, &go) != cudaSuccess && rc == SKC_OK) rc = check_launch("end capture");
  note_launches(-(int64_t)(skc_launch_count() - l0));  // captured, not executed
  if (rc != SKC_OK) return done(rc);
  if (cudaGraphInstantiate(&E.exec, g, 0) != cudaSuccess) return done(check_launch("graph instantiate"));
  E.graph = g;
  E.prologue_kernels = (int)(l1 - l0);
  E.body_kernels = (int)(l3 - l2);
  return done(SKC_OK);
}

// sparsified_assign (cluster.py:306-311) for one column in the reference's own arithmetic:
// diff = val[:, None] - mu[idx, :]; (diff * diff).sum(axis=0) is a sequential sum over the m
// sampled coordinates (numpy reduces a strided axis row by row), then the first argmin.
// This differs from the CSR x dense order of the Lloyd assignment (cluster.py:181-187), so
// near-ties resolve exactly as the reference's single-column call does.
// np.argmin order: a NaN is the minimum (its first occurrence wins), else the smallest value,
// ties to the lowest index
__device__ __forceinline__ bool argmin_better(double a, int ka, double b, int kb) {
  const bool an = a != a, bn = b != b;
  if (an || bn) return an && bn ? ka < kb : an;
  return a < b || (a == b && ka < kb);
}

template <typename V>
__global__ void assign_one_kernel(const int32_t* __restrict__ idx, const V* __restrict__ val, int m,
                                  const double* __restrict__ mu, int K, int32_t* __restrict__ label,
                                  double* __restrict__ d2) {
  __shared__ double bv[32];
  __shared__ int bk[32];
  double best = INFINITY;
  int bestk = 0x7FFFFFFF;
  for (int k = threadIdx.x; k < K; k += blockDim.x) {
    double acc = 0.0;
    for (int t = 0; t < m; ++t) {
      const double d = dsub((double)val[t], mu[(int64_t)idx[t] * K + k]);
      acc = t == 0 ? dmul(d, d) : dadd(acc, dmul(d, d));
    }
    if (argmin_better(acc, k, best, bestk)) best = acc, bestk = k;
  }
  for (int o = 16; o > 0; o >>= 1) {
    const double ov = __shfl_down_sync(0xFFFFFFFFu, best, o);
    const int ok = __shfl_down_sync(0xFFFFFFFFu, bestk, o);
    if (argmin_better(ov, ok, best, bestk)) best = ov, bestk = ok;
  }
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) bv[warp] = best, bk[warp] = bestk;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < (int)((blockDim.x + 31) / 32); ++w)
      if (argmin_better(bv[w], bk[w], best, bestk)) best = bv[w], bestk = bk[w];
    *label = bestk;
    if (d2) *d2 = best;
  }
}

}  // namespace
}  // namespace skc

using namespace skc;

extern "C" {

size_t skc_kmeans_lloyd_workspace(int64_t n, int32_t m, int32_t p_pad, int32_t K, int32_t val_dtype, int32_t use_tc) {
  size_t total = 0;
  carve(nullptr, n, m, p_pad, K, val_dtype, use_tc != 0, &total);
  return total;
}

int skc_kmeans_lloyd(const int32_t* idx, const void* val, int32_t val_dtype, int64_t n, int32_t m, int32_t p_pad,
                     int32_t K, const double* mu0, int32_t max_iter, const void* csc, const void* tc_prep, void* ws,
                     size_t ws_bytes, int32_t* labels, double* mu, double* traj, int32_t* iters, void* stream) {
  if (val_dtype != SKC_F32 && val_dtype != SKC_F64) return fail(SKC_EPARAM, "values must be fp32 or fp64");
  if (n < 1 || m < 1 || m > p_pad || K < 1) return fail(SKC_EDIM, "bad (n, m, p_pad, K)");
  if (max_iter < 1) return fail(SKC_EPARAM, "max_iter must be >= 1");
  if (csc == nullptr) return fail(SKC_EPARAM, "csc (skc_kmeans_build_csc) is required");
  size_t need = 0;
  const Bufs B = carve(static_cast<char*>(ws), n, m, p_pad, K, val_dtype, tc_prep != nullptr, &need);
  if (ws_bytes < need) return fail(SKC_EPARAM, "workspace too small");
  Args A{idx, val, val_dtype, n, m, p_pad, K, mu0, max_iter, csc, tc_prep, labels, mu, traj, iters};
  const Key key{idx, val, n, m, p_pad, K, val_dtype, mu0, max_iter, csc, tc_prep, ws, ws_bytes, labels, mu, traj, iters,
                [] {
                  int d = 0;
                  cudaGetDevice(&d);
                  return 2 * d + (fused_on() ? 1 : 0);  // SKC_LLOYD_FUSED is read per call (tests compare both)
                }()};
  std::lock_guard<std::mutex> lk(g_mu);
  auto it = g_cache.find(key);
  if (it == g_cache.end()) {
    if (g_cache.size() >= 8) {  // evict the least recently used graph
      auto old = g_cache.begin();
      for (auto j = g_cache.begin(); j != g_cache.end(); ++j)
        if (j->second.stamp < old->second.stamp) old = j;
      cudaGraphExecDestroy(old->second.exec);
      cudaGraphDestroy(old->second.graph);
      g_cache.erase(old);
    }
    Entry E;
    const int rc = build(A, B, E);
    if (rc) return rc;
    it = g_cache.emplace(key, E).first;
  }
  it->second.stamp = ++g_stamp;
  g_last_prologue = it->second.prologue_kernels;
  g_last_body = it->second.body_kernels;
  if (cudaGraphLaunch(it->second.exec, static_cast<cudaStream_t>(stream)) != cudaSuccess)
    return check_launch("graph launch");
  return SKC_OK;
}

int skc_kmeans_assign_one(const int32_t* idx_row, const void* val_row, int32_t val_dtype, int32_t m, const double* mu,
                          int32_t p_pad, int32_t K, int32_t* label_out, double* d2_out, void* stream) {
  if (val_dtype != SKC_F32 && val_dtype != SKC_F64) return fail(SKC_EPARAM, "values must be fp32 or fp64");
  if (m < 1 || m > p_pad || K < 1) return fail(SKC_EDIM, "bad (m, p_pad, K)");
  const int threads = K >= 256 ? 256 : ((K + 31) / 32) * 32;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (val_dtype == SKC_F64)
    assign_one_kernel<double><<<1, threads, 0, s>>>(idx_row, static_cast<const double*>(val_row), m, mu, K, label_out,
                                                    d2_out);
  else
    assign_one_kernel<float><<<1, threads, 0, s>>>(idx_row, static_cast<const float*>(val_row), m, mu, K, label_out,
                                                   d2_out);
  return check_launch("assign_one_kernel");
}

// kernels of the last skc_kmeans_lloyd graph on this thread: the prologue (first iteration) and
// one WHILE-body iteration, for launch accounting (a run launches prologue + (iters-1) * body)
void skc_kmeans_lloyd_graph_kernels(int32_t* prologue, int32_t* body) {
  if (prologue) *prologue = g_last_prologue;
  if (body) *body = g_last_body;
}

}  // extern "C"
