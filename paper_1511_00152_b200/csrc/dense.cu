// Second pass of two-pass sparsified K-means (cluster.py:407-456): one HBM-bound read of
// the raw rows per kernel, fp64 arithmetic, fixed reduction orders (deterministic).
//   K8 dense_assign  d2[i,k] = (|x_i|^2 - 2 <x_i, mu_k>) + |mu_k|^2 (cluster.py:438),
//                    labels2 = first argmin, d2min = max(d2, 0) (cluster.py:439-440)
//   K9 dense_sums    per-cluster sums of the rows under the first-pass labels
//                    (sums += chunk @ onehot, cluster.py:436) and the label counts
#include "common.cuh"

namespace skc {

constexpr uint32_t kAll = 0xFFFFFFFFu;
constexpr int kSumCols = 128;       // K9 column block (threads per CTA)
constexpr int kSumMaxK = 64;        // K9 clusters per launch (smem 64 KB)

__global__ void center_sqnorm_kernel(const double* __restrict__ mu, int32_t K, int32_t p, double* __restrict__ musq) {
  const int k = blockIdx.x;
  double s = 0.0;
  for (int j = threadIdx.x; j < p; j += 32) s = fma(mu[(int64_t)k * p + j], mu[(int64_t)k * p + j], s);
#pragma unroll
  for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(kAll, s, o);
  if (threadIdx.x == 0) musq[k] = s;
}

// K8: a skinny fp64 GEMM (rows x centres) fused with the argmin. CTA = 128 threads, tile
// of 256 rows; thread t owns rows t and t + 128 and KC centres per pass (2 KC fp64
// accumulators). Slabs of JS columns (32 fp32 / 16 fp64 = 128 B per row) stream through
// two shared-memory buffers with cp.async, so the next slab loads while this one is used.
// Rows are stored 144 B apart, so a thread's 16-byte read of its own row is bank-conflict
// free. The centres come from a transposed copy muT[j][Kpad] (prep kernel) as 16-byte
// copies; a thread reads them as broadcast LDS.128. |x|^2 accumulates in the first pass.
constexpr int kAsgThreads = 128;
constexpr int kAsgRows = 2 * kAsgThreads;
constexpr int kAsgRowBytes = 144;  // 128 B of data + 16 B pad
constexpr int kAsgMaxKC = 16;

__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src, bool ok) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "r"(ok ? 16 : 0) : "memory");
}
template <int B>
__device__ __forceinline__ void cp_async_small(uint32_t dst, const void* src, bool ok) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], %2, %3;" ::"r"(dst), "l"(src), "n"(B), "r"(ok ? B : 0)
               : "memory");
}

// muT[j][kp] = mu[k][j] for k < K, zero for K <= k < Kpad and p <= j < p_pad32
__global__ void center_transpose_kernel(const double* __restrict__ mu, int32_t K, int32_t p, int32_t Kpad,
                                        int32_t prows, double* __restrict__ muT) {
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= (int64_t)prows * Kpad) return;
  const int j = (int)(e / Kpad), k = (int)(e % Kpad);
  muT[e] = (k < K && j < p) ? mu[(int64_t)k * p + j] : 0.0;
}

template <typename V, int KC>
__global__ void __launch_bounds__(kAsgThreads) dense_assign_kernel(const V* __restrict__ X, int64_t ld, int64_t n,
                                                                   int32_t p, const double* __restrict__ muT,
                                                                   int32_t Kpad, const double* __restrict__ musq,
                                                                   int32_t K, int vec, int32_t* __restrict__ labels,
                                                                   double* __restrict__ d2min) {
  constexpr int JS = 128 / sizeof(V);        // columns per slab
  constexpr int XB = kAsgRows * kAsgRowBytes;  // bytes per X buffer
  constexpr int MB = JS * KC * 8;              // bytes per centre buffer
  extern __shared__ __align__(16) unsigned char dsm[];
  const uint32_t sbase = (uint32_t)__cvta_generic_to_shared(dsm);
  const int t = threadIdx.x;
  const int64_t tiles = (n + kAsgRows - 1) / kAsgRows;
  const int slabs = (p + JS - 1) / JS;
  for (int64_t tile = blockIdx.x; tile < tiles; tile += gridDim.x) {
    const int64_t row0 = tile * kAsgRows;
    double xsq0 = 0.0, xsq1 = 0.0, best0 = 0.0, best1 = 0.0;
    int bk0 = 0, bk1 = 0;
    for (int k0 = 0; k0 < K; k0 += KC) {
      const int nk = min(KC, K - k0);
      auto issue = [&](int sl, int buf) {
        const int j0 = sl * JS;
        const uint32_t xd = sbase + buf * XB, md = sbase + 2 * XB + buf * MB;
        if (vec) {  // 16-byte copies: 8 per row-slab, 2048 per tile
#pragma unroll 4
          for (int i = 0; i < kAsgRows * 8 / kAsgThreads; ++i) {
            const int e = t + kAsgThreads * i;
            const int r = e >> 3, q = e & 7;
            const int64_t row = row0 + r;
            const bool ok = row < n && j0 + q * (16 / (int)sizeof(V)) < p;
            cp_async16(xd + r * kAsgRowBytes + q * 16, ok ? (const void*)(X + row * ld + j0 + q * (16 / sizeof(V))) : X,
                       ok);
          }
        } else {
#pragma unroll 4
          for (int i = 0; i < kAsgRows * JS / kAsgThreads; ++i) {
            const int e = t + kAsgThreads * i;
            const int r = e / JS, c = e % JS;
            const int64_t row = row0 + r;
            const bool ok = row < n && j0 + c < p;
            cp_async_small<sizeof(V)>(xd + r * kAsgRowBytes + c * sizeof(V), ok ? (const void*)(X + row * ld + j0 + c) : X,
                                      ok);
          }
        }
        // centres: JS rows of KC doubles from muT[j0 + j][k0 .. k0 + KC)
        for (int e = t; e < JS * KC / 2; e += kAsgThreads) {
          const int j = e / (KC / 2), q = e % (KC / 2);
          cp_async16(md + (j * KC + 2 * q) * 8, muT + (int64_t)(j0 + j) * Kpad + k0 + 2 * q, true);
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
      };
      double a0[KC], a1[KC];
#pragma unroll
      for (int c = 0; c < KC; ++c) a0[c] = a1[c] = 0.0;
      issue(0, 0);
      for (int sl = 0; sl < slabs; ++sl) {
        if (sl + 1 < slabs) {
          issue(sl + 1, (sl + 1) & 1);
          asm volatile("cp.async.wait_group 1;" ::: "memory");
        } else {
          asm volatile("cp.async.wait_group 0;" ::: "memory");
        }
        __syncthreads();
        const unsigned char* xb = dsm + (sl & 1) * XB;
        const double* mb = reinterpret_cast<const double*>(dsm + 2 * XB + (sl & 1) * MB);
#pragma unroll
        for (int q = 0; q < JS * (int)sizeof(V) / 16; ++q) {  // 16 bytes of each of the two rows
          V v0[16 / sizeof(V)], v1[16 / sizeof(V)];
          *reinterpret_cast<uint4*>(v0) = *reinterpret_cast<const uint4*>(xb + t * kAsgRowBytes + q * 16);
          *reinterpret_cast<uint4*>(v1) = *reinterpret_cast<const uint4*>(xb + (t + kAsgThreads) * kAsgRowBytes + q * 16);
#pragma unroll
          for (int u = 0; u < 16 / (int)sizeof(V); ++u) {
            const int j = q * (16 / sizeof(V)) + u;
            const double x0 = (double)v0[u], x1 = (double)v1[u];
            if (k0 == 0) {
              xsq0 = fma(x0, x0, xsq0);
              xsq1 = fma(x1, x1, xsq1);
            }
            const double2* mj = reinterpret_cast<const double2*>(mb + j * KC);
#pragma unroll
            for (int c2 = 0; c2 < KC / 2; ++c2) {
              const double2 mm = mj[c2];
              a0[2 * c2] = fma(x0, mm.x, a0[2 * c2]);
              a0[2 * c2 + 1] = fma(x0, mm.y, a0[2 * c2 + 1]);
              a1[2 * c2] = fma(x1, mm.x, a1[2 * c2]);
              a1[2 * c2 + 1] = fma(x1, mm.y, a1[2 * c2 + 1]);
            }
          }
        }
        __syncthreads();  // buffer (sl & 1) is refilled by the issue two slabs on
      }
#pragma unroll
      for (int c = 0; c < KC; ++c) {
        if (c < nk) {
          const double mq = musq[k0 + c];
          const double d0 = dadd(dsub(xsq0, dmul(2.0, a0[c])), mq);
          const double d1 = dadd(dsub(xsq1, dmul(2.0, a1[c])), mq);
          if (k0 + c == 0 || d0 < best0) best0 = d0, bk0 = k0 + c;  // first minimum, as np.argmin
          if (k0 + c == 0 || d1 < best1) best1 = d1, bk1 = k0 + c;
        }
      }
    }
    const int64_t r0 = row0 + t, r1 = row0 + t + kAsgThreads;
    if (r0 < n) {
      labels[r0] = bk0;
      d2min[r0] = best0 > 0.0 ? best0 : 0.0;  // np.clip(d2, 0, None)
    }
    if (r1 < n) {
      labels[r1] = bk1;
      d2min[r1] = best1 > 0.0 ? best1 : 0.0;
    }
  }
}

// CTA (column block cb, row block rb): thread t owns column cb*128 + t; partial sums of
// clusters [kb, kb + nk) in shared memory; rows in ascending order within the block
template <typename V>
__global__ void __launch_bounds__(kSumCols) dense_sums_kernel(const V* __restrict__ X, int64_t ld, int64_t n,
                                                               int32_t p, const int32_t* __restrict__ lab, int32_t kb,
                                                               int32_t nk, int32_t nrb, double* __restrict__ part,
                                                               long long* __restrict__ counts) {
  extern __shared__ double ps[];  // [nk][kSumCols]
  const int cb = blockIdx.x % ((p + kSumCols - 1) / kSumCols), rb = blockIdx.x / ((p + kSumCols - 1) / kSumCols);
  const int c = cb * kSumCols + threadIdx.x;
  for (int k = 0; k < nk; ++k) ps[k * kSumCols + threadIdx.x] = 0.0;
  const int64_t r0 = n * rb / nrb, r1 = n * (rb + 1) / nrb;
  if (c < p) {
    int64_t r = r0;
    for (; r + 4 <= r1; r += 4) {  // four independent row loads in flight
      int k4[4];
      double v4[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        k4[u] = __ldg(lab + r + u) - kb;
        v4[u] = (double)__ldg(X + (r + u) * ld + c);
      }
#pragma unroll
      for (int u = 0; u < 4; ++u)
        if ((unsigned)k4[u] < (unsigned)nk) ps[k4[u] * kSumCols + threadIdx.x] += v4[u];
    }
    for (; r < r1; ++r) {
      const int k = __ldg(lab + r) - kb;
      if ((unsigned)k < (unsigned)nk) ps[k * kSumCols + threadIdx.x] += (double)__ldg(X + r * ld + c);
    }
    for (int k = 0; k < nk; ++k) part[((int64_t)rb * nk + k) * p + c] = ps[k * kSumCols + threadIdx.x];
  }
  if (cb == 0) {  // label counts of this row block (integers: exact in any order)
    __shared__ int cnt[kSumMaxK];
    __syncthreads();
    for (int k = threadIdx.x; k < nk; k += blockDim.x) cnt[k] = 0;
    __syncthreads();
    for (int64_t r = r0 + threadIdx.x; r < r1; r += blockDim.x) {
      const int k = __ldg(lab + r) - kb;
      if ((unsigned)k < (unsigned)nk) atomicAdd(&cnt[k], 1);
    }
    __syncthreads();
    for (int k = threadIdx.x; k < nk; k += blockDim.x)
      if (cnt[k]) atomicAdd(reinterpret_cast<unsigned long long*>(counts) + kb + k, (unsigned long long)cnt[k]);
  }
}

// sums[k][c] += sum over row blocks, in block order
__global__ void dense_sums_combine_kernel(const double* __restrict__ part, int32_t nrb, int32_t nk, int32_t p,
                                          int32_t kb, double* __restrict__ sums) {
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= (int64_t)nk * p) return;
  const int k = (int)(e / p), c = (int)(e % p);
  double s = 0.0;
  for (int b = 0; b < nrb; ++b) s += part[((int64_t)b * nk + k) * p + c];
  sums[(int64_t)(kb + k) * p + c] += s;
}

static int dense_row_blocks(int64_t n, int32_t p) {
  const int cbs = (p + kSumCols - 1) / kSumCols;
  int64_t want = (8LL * sm_count() + cbs - 1) / cbs;  // ~8 CTAs per SM
  const int64_t maxrb = (n + 255) / 256;
  if (want > maxrb) want = maxrb;
  return (int)(want < 1 ? 1 : want);
}

size_t dense_sums_ws(int64_t n, int32_t p, int32_t K) {
  const int nk = K < kSumMaxK ? K : kSumMaxK;
  return (size_t)dense_row_blocks(n, p) * nk * p * sizeof(double);
}

template <typename V, int KC>
static int assign_launch_t(const V* X, int64_t ld, int64_t n, int32_t p, const double* muT, int32_t Kpad,
                           const double* musq, int32_t K, int vec, int32_t* labels, double* d2min, cudaStream_t st) {
  constexpr int JS = 128 / sizeof(V);
  const size_t smem = 2 * (size_t)kAsgRows * kAsgRowBytes + 2 * (size_t)JS * KC * 8;
  auto kern = dense_assign_kernel<V, KC>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int occ = 1;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, kAsgThreads, smem);
  int64_t blocks = (n + kAsgRows - 1) / kAsgRows;
  const int64_t cap = (int64_t)sm_count() * (occ < 1 ? 1 : occ);
  if (blocks > cap) blocks = cap;
  kern<<<(unsigned)blocks, kAsgThreads, smem, st>>>(X, ld, n, p, muT, Kpad, musq, K, vec, labels, d2min);
  return check_launch("dense_assign_kernel");
}

template <typename V>
static int assign_dispatch(int kc, const V* X, int64_t ld, int64_t n, int32_t p, const double* muT, int32_t Kpad,
                           const double* musq, int32_t K, int vec, int32_t* labels, double* d2min, cudaStream_t st) {
  switch (kc) {
    case 2: return assign_launch_t<V, 2>(X, ld, n, p, muT, Kpad, musq, K, vec, labels, d2min, st);
    case 4: return assign_launch_t<V, 4>(X, ld, n, p, muT, Kpad, musq, K, vec, labels, d2min, st);
    case 6: return assign_launch_t<V, 6>(X, ld, n, p, muT, Kpad, musq, K, vec, labels, d2min, st);
    case 8: return assign_launch_t<V, 8>(X, ld, n, p, muT, Kpad, musq, K, vec, labels, d2min, st);
    case 10: return assign_launch_t<V, 10>(X, ld, n, p, muT, Kpad, musq, K, vec, labels, d2min, st);
    case 12: return assign_launch_t<V, 12>(X, ld, n, p, muT, Kpad, musq, K, vec, labels, d2min, st);
    case 14: return assign_launch_t<V, 14>(X, ld, n, p, muT, Kpad, musq, K, vec, labels, d2min, st);
    default: return assign_launch_t<V, 16>(X, ld, n, p, muT, Kpad, musq, K, vec, labels, d2min, st);
  }
}

// centre chunk: K <= 16 in one pass of the next even size; larger K in passes of 16
static int assign_kc(int32_t K) { return K > kAsgMaxKC ? kAsgMaxKC : ((K + 1) & ~1); }

size_t dense_assign_ws(int32_t p, int32_t K) {
  const int kc = assign_kc(K);
  const int Kpad = (K + kc - 1) / kc * kc;
  const int prows = (p + 31) / 32 * 32;
  return ((size_t)K + (size_t)prows * Kpad) * sizeof(double);
}

int dense_assign_launch(const void* X, int x_f64, int64_t ld, int64_t n, int32_t p, const double* mu, int32_t K,
                        double* ws, int32_t* labels, double* d2min, cudaStream_t st) {
  if (n == 0) return SKC_OK;
  const int kc = assign_kc(K);
  const int Kpad = (K + kc - 1) / kc * kc;
  const int prows = (p + 31) / 32 * 32;
  double* musq = ws;
  double* muT = ws + ((K + 1) & ~1);  // 16-byte aligned
  center_sqnorm_kernel<<<K, 32, 0, st>>>(mu, K, p, musq);
  int rc = check_launch("center_sqnorm_kernel");
  if (rc) return rc;
  const int64_t tot = (int64_t)prows * Kpad;
  center_transpose_kernel<<<(unsigned)((tot + 255) / 256), 256, 0, st>>>(mu, K, p, Kpad, prows, muT);
  if ((rc = check_launch("center_transpose_kernel"))) return rc;
  const size_t es = x_f64 ? 8 : 4;
  const int vec = (reinterpret_cast<uintptr_t>(X) % 16 == 0) && ((ld * es) % 16 == 0) && ((p * es) % 16 == 0);
  if (x_f64) return assign_dispatch<double>(kc, (const double*)X, ld, n, p, muT, Kpad, musq, K, vec, labels, d2min, st);
  return assign_dispatch<float>(kc, (const float*)X, ld, n, p, muT, Kpad, musq, K, vec, labels, d2min, st);
}

int dense_sums_launch(const void* X, int x_f64, int64_t ld, int64_t n, int32_t p, const int32_t* lab, int32_t K,
                      double* sums, long long* counts, void* ws, cudaStream_t st) {
  if (n == 0) return SKC_OK;
  const int nrb = dense_row_blocks(n, p);
  const int cbs = (p + kSumCols - 1) / kSumCols;
  double* part = reinterpret_cast<double*>(ws);
  for (int kb = 0; kb < K; kb += kSumMaxK) {
    const int nk = K - kb < kSumMaxK ? K - kb : kSumMaxK;
    const size_t smem = (size_t)nk * kSumCols * sizeof(double);
    if (x_f64) {
      cudaFuncSetAttribute(dense_sums_kernel<double>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      dense_sums_kernel<double><<<(unsigned)(cbs * nrb), kSumCols, smem, st>>>((const double*)X, ld, n, p, lab, kb, nk,
                                                                                nrb, part, counts);
    } else {
      cudaFuncSetAttribute(dense_sums_kernel<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      dense_sums_kernel<float><<<(unsigned)(cbs * nrb), kSumCols, smem, st>>>((const float*)X, ld, n, p, lab, kb, nk,
                                                                              nrb, part, counts);
    }
    int rc = check_launch("dense_sums_kernel");
    if (rc) return rc;
    const int64_t tot = (int64_t)nk * p;
    dense_sums_combine_kernel<<<(unsigned)((tot + 255) / 256), 256, 0, st>>>(part, nrb, nk, p, kb, sums);
    rc = check_launch("dense_sums_combine_kernel");
    if (rc) return rc;
  }
  return SKC_OK;
}

}  // namespace skc
