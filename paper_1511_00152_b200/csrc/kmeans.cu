// K5/K6: sparsified K-means on the sketch (cluster.py:133-243).
//  assign   exact fp64 emulation of [values | ones] @ [-2 mu ; mu*mu] + colsq
//           (cluster.py:181-187), so labels and d2min are bit-exact
//  pairwise numpy pairwise summation of d2min (the objective, cluster.py:233)
//  partials bit-exact np.bincount sums (cluster.py:189-208): the sketch transposed once
//           into per-coordinate lists; per iteration a segmented stable sort by label
//           and one sequential add per (coordinate, cluster) chain
//  centers  divide / keep-previous / empty flags (cluster.py:196-210)
//  reseed   cluster.py:212-215;  init  cluster.py:175-179
#include <cub/device/device_scan.cuh>

#include "common.cuh"

namespace skc {

constexpr uint32_t kFM = 0xFFFFFFFFu;

template <typename V>
__device__ __forceinline__ double ldd(const void* p, int64_t i) {
  return (double)__ldg(reinterpret_cast<const V*>(p) + i);
}

// ---------------------------------------------------------------------------------
// numpy pairwise sum (8 accumulators up to 128 elements, halving split rounded down to
// a multiple of 8 above that).
__device__ double pw_leaf(const double* a, int64_t n) {
  if (n < 8) {
    double r = 0.0;
    for (int64_t i = 0; i < n; ++i) r = dadd(r, a[i]);
    return r;
  }
  double r[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) r[k] = a[k];
  int64_t i = 8;
  for (; i < n - (n % 8); i += 8) {
#pragma unroll
    for (int k = 0; k < 8; ++k) r[k] = dadd(r[k], a[i + k]);
  }
  double res = dadd(dadd(dadd(r[0], r[1]), dadd(r[2], r[3])), dadd(dadd(r[4], r[5]), dadd(r[6], r[7])));
  for (; i < n; ++i) res = dadd(res, a[i]);
  return res;
}

__device__ double pw_rec(const double* a, int64_t n) {
  if (n <= 128) return pw_leaf(a, n);
  int64_t n2 = n / 2;
  n2 -= n2 % 8;
  return dadd(pw_rec(a, n2), pw_rec(a + n2, n - n2));
}

constexpr int kPwDeep = 14;  // deepest split level handled by the combine (2^14 subtrees)

// numpy's tree is cut at depth D (runtime, <= kPwDeep, about log2(n / 128)) into 2^D paths.
// res[t]: the sum of path t's subtree; ld[t]: the depth at which path t reaches a leaf (<= 128
// elements), D if it does not. Node t of depth d (stored at t << (D - d)) is an internal node of
// numpy's tree exactly when ld[t << (D - d)] > d. Eight lanes share a path: a leaf's eight
// accumulators r[k] = a[k] + a[k+8] + ... run one per lane (coalesced 64-byte steps), then
// ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)) by shuffles and the tail by lane 0 -- pw_leaf's order.
__global__ void __launch_bounds__(256) pairwise_leaves_kernel(const double* __restrict__ x, int64_t n, int D,
                                                              double* __restrict__ res, uint8_t* __restrict__ ld) {
  const int gt = blockIdx.x * blockDim.x + threadIdx.x;
  const int t = gt >> 3, k = gt & 7;  // path, lane within the path's group
  if (t >= (1 << D)) return;           // whole groups exit together (8 | 256)
  int64_t off = 0, len = n;
  bool active = true;
  int leafd = D;
  for (int d = 0; d < D; ++d) {
    const int bit = (t >> (D - 1 - d)) & 1;
    if (len <= 128) {  // leaf above the split depth: owned by the all-zero suffix path
      if (leafd == D) leafd = d;
      if (bit) active = false;
      continue;
    }
    int64_t n2 = len / 2;
    n2 -= n2 % 8;
    if (bit) {
      off += n2;
      len -= n2;
    } else {
      len = n2;
    }
  }
  double r = 0.0;
  const double* a = x + off;
  const unsigned gmask = 0xFFu << (threadIdx.x & 24);
  if (active && len <= 128 && len >= 8) {
    r = a[k];
    const int64_t body = len - (len % 8);
    for (int64_t i = 8 + k; i < body; i += 8) r = dadd(r, a[i]);
    const double r1 = __shfl_down_sync(gmask, r, 1, 8);
    const double s01 = dadd(r, r1);
    const double s23 = __shfl_down_sync(gmask, s01, 2, 8);
    const double q = dadd(s01, s23);
    const double q2 = __shfl_down_sync(gmask, q, 4, 8);
    if (k == 0) {
      r = dadd(q, q2);
      for (int64_t i = body; i < len; ++i) r = dadd(r, a[i]);
    }
  } else if (k == 0 && active) {
    r = len <= 128 ? pw_leaf(a, len) : pw_rec(a, len);
  }
  if (k == 0) {
    res[t] = active ? r : 0.0;
    ld[t] = (uint8_t)leafd;
  }
}

// The 2^D subtree sums are combined in shared memory, level by level; whether a node is internal
// comes from ld (one lookup instead of re-walking its path).
__global__ void __launch_bounds__(1024) pairwise_combine_kernel(const double* __restrict__ gres,
                                                                const uint8_t* __restrict__ gld, int D,
                                                                double* __restrict__ out) {
  extern __shared__ double res[];
  uint8_t* ld = reinterpret_cast<uint8_t*>(res + (1 << kPwDeep));
  for (int t = threadIdx.x; t < (1 << D); t += blockDim.x) res[t] = gres[t], ld[t] = gld[t];
  __syncthreads();
  for (int d = D - 1; d >= 0; --d) {
    const int sh = D - d;
    for (int t = threadIdx.x; t < (1 << d); t += blockDim.x)
      if (ld[t << sh] > d) res[t << sh] = dadd(res[(2 * t) << (sh - 1)], res[(2 * t + 1) << (sh - 1)]);
    __syncthreads();
  }
  if (threadIdx.x == 0) out[0] = res[0];
}

size_t pairwise_ws() { return ((size_t)1 << kPwDeep) * (sizeof(double) + 1); }

// the leaves alone (the Lloyd graph combines them in its objective-and-check kernel): subtree
// sums in ws as [2^kPwDeep] doubles then [2^kPwDeep] depth bytes, *D_out the split depth
int pairwise_leaves_launch(const double* x, int64_t n, void* ws, int* D_out, cudaStream_t st) {
  double* res = reinterpret_cast<double*>(ws);
  uint8_t* ld = reinterpret_cast<uint8_t*>(res + (1 << kPwDeep));
  int D = 0;
  while (D < kPwDeep && ((int64_t)128 << D) < n) ++D;
  const int threads = 8 << D;
  pairwise_leaves_kernel<<<(threads + 255) / 256, 256, 0, st>>>(x, n, D, res, ld);
  *D_out = D;
  return check_launch("pairwise_leaves_kernel");
}

int pairwise_launch(const double* x, int64_t n, double* out, void* ws, cudaStream_t st) {
  double* res = reinterpret_cast<double*>(ws);
  uint8_t* ld = reinterpret_cast<uint8_t*>(res + (1 << kPwDeep));
  int D = 0;
  while (D < kPwDeep && ((int64_t)128 << D) < n) ++D;  // leaves of <= ~128 elements at depth <= D
  const int threads = 8 << D;
  pairwise_leaves_kernel<<<(threads + 255) / 256, 256, 0, st>>>(x, n, D, res, ld);
  int rc = check_launch("pairwise_leaves_kernel");
  if (rc) return rc;
  const size_t smem = ((size_t)1 << kPwDeep) * (sizeof(double) + 1);
  cudaFuncSetAttribute(pairwise_combine_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  pairwise_combine_kernel<<<1, 1024, smem, st>>>(res, ld, D, out);
  return check_launch("pairwise_combine_kernel");
}

// ---------------------------------------------------------------------------------
// assign
constexpr int kAsgWarps = 8;

// packed per-(j,k) table: {-2 mu, mu*mu} (np.vstack([-2.0 * mu, mu * mu]), cluster.py:182)
// as two planes, tx = -2 mu and ty = mu * mu, each [p][K]: a group's K lanes then read K
// contiguous doubles per coordinate (half the L1 wavefronts of an interleaved {x, y} table)
__global__ void km_tables2_kernel(const double* __restrict__ mu, int64_t total, double* __restrict__ tx,
                                  double* __restrict__ ty) {
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= total) return;
  const double v = mu[e];
  tx[e] = dmul(-2.0, v);
  ty[e] = dmul(v, v);
}

// A warp holds G = 32/KP points; lane = g*KP + k. For K > KP the lane loops over k += KP.
// colsq: numpy pairwise order on 8 lanes of the group (m <= 128), else pw_rec on one lane.
// d2[k] = sum_t v_t*(-2 mu[j_t,k]) then + sum_t mu[j_t,k]^2 (csr_matvecs axpy order) + colsq.
// SMEM_TAB: the packed (p, K) table is staged in shared memory (small p*K, e.g. C2).
template <typename V, int KP, bool SMEM_TAB>
__global__ void __launch_bounds__(kAsgWarps * 32, 4)
    km_assign_kernel(const int32_t* __restrict__ idx, const void* __restrict__ val, int64_t n, int m,
                     const double* __restrict__ gtx, const double* __restrict__ gty, int K, int p_pad,
                     const int32_t* __restrict__ prev,
                     int32_t* __restrict__ labels, double* __restrict__ d2min, int64_t* __restrict__ blk_changed,
                     double* __restrict__ blk_max, int64_t* __restrict__ blk_arg) {
  constexpr int G = 32 / KP;
  extern __shared__ __align__(16) unsigned char sm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane / KP, k0 = lane % KP;
  // layout: [table (SMEM_TAB)] [per warp: sidx G*m int | sval G*m double | msq 32*m double]
  size_t off = 0;
  const double* tabx = gtx;
  const double* taby = gty;
  if constexpr (SMEM_TAB) {
    double* st = reinterpret_cast<double*>(sm);
    for (int e = threadIdx.x; e < p_pad * K; e += blockDim.x) st[e] = gtx[e], st[p_pad * K + e] = gty[e];
    tabx = st;
    taby = st + p_pad * K;
    off = (size_t)p_pad * K * 16;
    __syncthreads();
  }
  const size_t per_warp = ((size_t)G * m * 4 + 15) / 16 * 16 + (size_t)G * m * 8;
  unsigned char* wb = sm + off + per_warp * warp;
  int* sidx = reinterpret_cast<int*>(wb);  // row offsets j*K
  double* sval = reinterpret_cast<double*>(wb + ((size_t)G * m * 4 + 15) / 16 * 16);
  int64_t changed = 0;
  double bmax = -1.0;
  int64_t barg = -1;
  const int nwarps = blockDim.x >> 5;
  const int64_t gw = (int64_t)blockIdx.x * nwarps + warp, nw = (int64_t)gridDim.x * nwarps;
  for (int64_t i0 = gw * G; i0 < n; i0 += nw * G) {
    __syncwarp();
#pragma unroll
    for (int gg = 0; gg < G; ++gg) {
      const int64_t i = i0 + gg;
      if (i < n)
        for (int t = lane; t < m; t += 32) {
          sidx[gg * m + t] = __ldg(idx + i * m + t) * K;
          sval[gg * m + t] = ldd<V>(val, i * m + t);
        }
    }
    __syncwarp();
    const int64_t i = i0 + g;
    const int* si = sidx + g * m;
    const double* sv = sval + g * m;
    // colsq = (v*v).sum() in numpy's pairwise order
    double colsq = 0.0;
    if (m < 8) {
      if (k0 == 0)
        for (int t = 0; t < m; ++t) colsq = dadd(colsq, dmul(sv[t], sv[t]));
    } else if (m <= 128) {
      double r = 0.0;
      if (k0 < 8) {
        r = dmul(sv[k0], sv[k0]);
        for (int t = 8 + k0; t < m - (m % 8); t += 8) r = dadd(r, dmul(sv[t], sv[t]));
      }
      // ((r0+r1)+(r2+r3)) + ((r4+r5)+(r6+r7)) across lanes k0 = 0..7 of the group
      const double r1 = __shfl_down_sync(kFM, r, 1, KP);
      const double s01 = dadd(r, r1);
      const double s23 = __shfl_down_sync(kFM, s01, 2, KP);
      const double q = dadd(s01, s23);
      const double q2 = __shfl_down_sync(kFM, q, 4, KP);
      if (k0 == 0) {
        colsq = dadd(q, q2);
        for (int t = m - (m % 8); t < m; ++t) colsq = dadd(colsq, dmul(sv[t], sv[t]));
      }
    } else if (k0 == 0) {
      double* tmp = const_cast<double*>(sv);  // square in place, restore after
      for (int t = 0; t < m; ++t) tmp[t] = dmul(sv[t], sv[t]);
      colsq = pw_rec(tmp, m);
      for (int t = 0; t < m; ++t) tmp[t] = ldd<V>(val, i * m + t);
    }
    __syncwarp();
    colsq = __shfl_sync(kFM, colsq, g * KP, 32);
    double best = 0.0;
    int bk = -1;
    for (int kb = 0; kb < K; kb += KP) {
      const int k = kb + k0;
      double v = __longlong_as_double(0x7FF0000000000000LL);
      int kk = 0x7FFFFFFF;
      if (k < K && i < n) {
        double acc = 0.0;
        int t = 0;
        const double* tkx = tabx + k;
        const double* tky = taby + k;
        for (; t + 4 <= m; t += 4) {
          const double a0 = tkx[si[t]], a1 = tkx[si[t + 1]], a2 = tkx[si[t + 2]], a3 = tkx[si[t + 3]];
          acc = dadd(acc, dmul(sv[t], a0));
          acc = dadd(acc, dmul(sv[t + 1], a1));
          acc = dadd(acc, dmul(sv[t + 2], a2));
          acc = dadd(acc, dmul(sv[t + 3], a3));
        }
        for (; t < m; ++t) acc = dadd(acc, dmul(sv[t], tkx[si[t]]));
        for (t = 0; t + 4 <= m; t += 4) {
          const double b0 = tky[si[t]], b1 = tky[si[t + 1]], b2 = tky[si[t + 2]], b3 = tky[si[t + 3]];
          acc = dadd(acc, b0);
          acc = dadd(acc, b1);
          acc = dadd(acc, b2);
          acc = dadd(acc, b3);
        }
        for (; t < m; ++t) acc = dadd(acc, tky[si[t]]);
        v = dadd(acc, colsq);
        kk = k;
      }
      // first minimum over the group (np.argmin: lower k wins ties)
#pragma unroll
      for (int o = KP / 2; o > 0; o >>= 1) {
        const double ov = __shfl_xor_sync(kFM, v, o);
        const int ok = __shfl_xor_sync(kFM, kk, o);
        if (ov < v || (ov == v && ok < kk)) {
          v = ov;
          kk = ok;
        }
      }
      if (bk < 0 || v < best) {
        best = v;
        bk = kk;
      }
    }
    if (k0 == 0 && i < n) {
      const double dm = best > 0.0 ? best : 0.0;  // np.clip(.., 0, None)
      labels[i] = bk;
      d2min[i] = dm;
      if (prev != nullptr) changed += prev[i] != bk;
      if (dm > bmax) {  // each lane sees its points in ascending order: keeps the first max
        bmax = dm;
        barg = i;
      }
    }
  }
  // block reduction over all lanes: changed sum, (max, first index)
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const int64_t oc = __shfl_xor_sync(kFM, changed, o), oa = __shfl_xor_sync(kFM, barg, o);
    const double om = __shfl_xor_sync(kFM, bmax, o);
    changed += oc;
    if (oa >= 0 && (om > bmax || (om == bmax && (barg < 0 || oa < barg)))) {
      bmax = om;
      barg = oa;
    }
  }
  __shared__ int64_t s_ch[kAsgWarps], s_arg[kAsgWarps];
  __shared__ double s_mx[kAsgWarps];
  if (lane == 0) {
    s_ch[warp] = changed;
    s_mx[warp] = bmax;
    s_arg[warp] = barg;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    int64_t c = 0, a = -1;
    double mx = -1.0;
    for (int w = 0; w < nwarps; ++w) {
      c += s_ch[w];
      if (s_arg[w] >= 0 && (s_mx[w] > mx || (s_mx[w] == mx && (a < 0 || s_arg[w] < a)))) {
        mx = s_mx[w];
        a = s_arg[w];
      }
    }
    blk_changed[blockIdx.x] = c;
    blk_max[blockIdx.x] = mx;
    blk_arg[blockIdx.x] = a;
  }
}

// K5s: the exact assignment for small K (K <= 16, e.g. C2), one point per thread. The thread
// keeps K accumulators in registers (K independent fp64 chains hide the add latency) and reads
// the point's table rows as 16-byte vectors from L1: d2[k] = (sum_t v_t * (-2 mu[j_t,k]) then
// + sum_t mu[j_t,k]^2, t ascending: csr_matvecs' axpy order, cluster.py:181-187) + colsq (numpy
// pairwise order), first minimum over k, clipped at 0: the same arithmetic as km_assign_kernel,
// so labels and d2min are bit-identical. Tables: [p][KC] planes, KC = K rounded up to even.
__global__ void km_tables_pad_kernel(const double* __restrict__ mu, int p, int K, int KC, double* __restrict__ tx,
                                     double* __restrict__ ty) {
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= (int64_t)p * KC) return;
  const int j = (int)(e / KC), k = (int)(e % KC);
  const double v = k < K ? mu[(int64_t)j * K + k] : 0.0;
  tx[e] = dmul(-2.0, v);
  ty[e] = dmul(v, v);
}

__device__ __forceinline__ double colsq_pairwise(const int32_t* __restrict__ ir, const void* val, int64_t base, int m,
                                                 bool f64) {
  (void)ir;
  auto ld = [&](int t) -> double {
    return f64 ? __ldg(reinterpret_cast<const double*>(val) + base + t)
               : (double)__ldg(reinterpret_cast<const float*>(val) + base + t);
  };
  if (m < 8) {
    double c = 0.0;
    for (int t = 0; t < m; ++t) c = dadd(c, dmul(ld(t), ld(t)));
    return c;
  }
  if (m <= 128) {
    double r[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) r[k] = dmul(ld(k), ld(k));
    int t = 8;
    for (; t < m - (m % 8); t += 8)
#pragma unroll
      for (int k = 0; k < 8; ++k) r[k] = dadd(r[k], dmul(ld(t + k), ld(t + k)));
    double c = dadd(dadd(dadd(r[0], r[1]), dadd(r[2], r[3])), dadd(dadd(r[4], r[5]), dadd(r[6], r[7])));
    for (; t < m; ++t) c = dadd(c, dmul(ld(t), ld(t)));
    return c;
  }
  return -1.0;  // m > 128: the caller takes km_assign_kernel
}

constexpr int kSmallThreads = 256;
template <typename V, int KC>
__global__ void __launch_bounds__(kSmallThreads, 2) km_assign_small_kernel(
    const int32_t* __restrict__ idx, const void* __restrict__ val, int64_t n, int m, const double* __restrict__ tx,
    const double* __restrict__ ty, int K, const int32_t* __restrict__ prev, int32_t* __restrict__ labels,
    double* __restrict__ d2min, int64_t* __restrict__ blk_changed, double* __restrict__ blk_max,
    int64_t* __restrict__ blk_arg) {
  constexpr bool F64 = sizeof(V) == 8;
  int64_t changed = 0;
  double bmax = -1.0;
  int64_t barg = -1;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += stride) {
    const int32_t* ir = idx + i * m;
    const V* vr = reinterpret_cast<const V*>(val) + i * m;
    double acc[KC];
#pragma unroll
    for (int k = 0; k < KC; ++k) acc[k] = 0.0;
    for (int t = 0; t < m; ++t) {
      const double v = (double)__ldg(vr + t);
      const double2* row = reinterpret_cast<const double2*>(tx + (size_t)__ldg(ir + t) * KC);
#pragma unroll
      for (int c = 0; c < KC / 2; ++c) {
        const double2 a = __ldg(row + c);
        acc[2 * c] = dadd(acc[2 * c], dmul(v, a.x));
        acc[2 * c + 1] = dadd(acc[2 * c + 1], dmul(v, a.y));
      }
    }
    for (int t = 0; t < m; ++t) {
      const double2* row = reinterpret_cast<const double2*>(ty + (size_t)__ldg(ir + t) * KC);
#pragma unroll
      for (int c = 0; c < KC / 2; ++c) {
        const double2 b = __ldg(row + c);
        acc[2 * c] = dadd(acc[2 * c], b.x);
        acc[2 * c + 1] = dadd(acc[2 * c + 1], b.y);
      }
    }
    const double colsq = colsq_pairwise(ir, val, i * m, m, F64);
    double best = dadd(acc[0], colsq);
    int bk = 0;
#pragma unroll
    for (int k = 1; k < KC; ++k) {
      const double d = dadd(acc[k], colsq);
      if (k < K && d < best) best = d, bk = k;
    }
    const double dm = best > 0.0 ? best : 0.0;  // np.clip(.., 0, None)
    labels[i] = bk;
    d2min[i] = dm;
    if (prev != nullptr) changed += prev[i] != bk;
    if (dm > bmax) bmax = dm, barg = i;  // ascending i per thread: keeps the first max
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const int64_t oc = __shfl_xor_sync(kFM, changed, o), oa = __shfl_xor_sync(kFM, barg, o);
    const double om = __shfl_xor_sync(kFM, bmax, o);
    changed += oc;
    if (oa >= 0 && (om > bmax || (om == bmax && (barg < 0 || oa < barg)))) bmax = om, barg = oa;
  }
  __shared__ int64_t s_ch[kSmallThreads / 32], s_arg[kSmallThreads / 32];
  __shared__ double s_mx[kSmallThreads / 32];
  const int warp = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0) s_ch[warp] = changed, s_mx[warp] = bmax, s_arg[warp] = barg;
  __syncthreads();
  if (threadIdx.x == 0) {
    int64_t c = 0, a = -1;
    double mx = -1.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) {
      c += s_ch[w];
      if (s_arg[w] >= 0 && (s_mx[w] > mx || (s_mx[w] == mx && (a < 0 || s_arg[w] < a)))) mx = s_mx[w], a = s_arg[w];
    }
    blk_changed[blockIdx.x] = c;
    blk_max[blockIdx.x] = mx;
    blk_arg[blockIdx.x] = a;
  }
}

// K5c: small K with the padded tables in shared memory. H = KC/2 lanes cooperate on a point,
// lane h owning centres 2h and 2h+1 (one 16-byte table read per coordinate), G = 32/H points per
// warp step, the step's rows staged in shared memory with coalesced loads. Every (point, centre)
// sum runs in the reference's order (cluster.py:183: values then ones, ascending t), so labels
// and d2min equal K5s / K5 bit for bit; the argmin is the sequential lowest-index scan.
constexpr int kCoopWarps = 8;
__device__ __forceinline__ double colsq_pairwise_row(const double* __restrict__ rv, int m) {
  // numpy's pairwise-8 sum of squares, the order colsq_pairwise uses
  if (m < 8) {
    double c = 0.0;
    for (int t = 0; t < m; ++t) c = dadd(c, dmul(rv[t], rv[t]));
    return c;
  }
  double r[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) r[k] = dmul(rv[k], rv[k]);
  int t = 8;
  for (; t < m - (m % 8); t += 8)
#pragma unroll
    for (int k = 0; k < 8; ++k) r[k] = dadd(r[k], dmul(rv[t + k], rv[t + k]));
  double c = dadd(dadd(dadd(r[0], r[1]), dadd(r[2], r[3])), dadd(dadd(r[4], r[5]), dadd(r[6], r[7])));
  for (; t < m; ++t) c = dadd(c, dmul(rv[t], rv[t]));
  return c;
}

template <typename V, int H>
__global__ void __launch_bounds__(kCoopWarps * 32, 2) km_assign_coop_kernel(
    const int32_t* __restrict__ idx, const void* __restrict__ val, int64_t n, int m, const double* __restrict__ tx2,
    const double* __restrict__ ty2, int K, int p_pad, const int32_t* __restrict__ prev, int32_t* __restrict__ labels,
    double* __restrict__ d2min, int64_t* __restrict__ blk_changed, double* __restrict__ blk_max,
    int64_t* __restrict__ blk_arg) {
  constexpr int G = 32 / H;  // points per warp step
  extern __shared__ __align__(16) unsigned char csm[];
  double2* tabx = reinterpret_cast<double2*>(csm);  // [p_pad][H]: (-2 mu) pairs
  double2* taby = tabx + (size_t)p_pad * H;          // [p_pad][H]: mu^2 pairs
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double* sval = reinterpret_cast<double*>(taby + (size_t)p_pad * H) + (size_t)warp * G * m;
  int* sidx = reinterpret_cast<int*>(reinterpret_cast<double*>(taby + (size_t)p_pad * H) + (size_t)kCoopWarps * G * m) +
              (size_t)warp * G * m;
  {
    const double2* gx = reinterpret_cast<const double2*>(tx2);
    const double2* gy = reinterpret_cast<const double2*>(ty2);
    for (int e = threadIdx.x; e < p_pad * H; e += blockDim.x) tabx[e] = __ldg(gx + e), taby[e] = __ldg(gy + e);
  }
  __syncthreads();
  const int g = lane / H, h = lane - g * H;
  int64_t changed = 0;
  double bmax = -1.0;
  int64_t barg = -1;
  const int64_t step = (int64_t)gridDim.x * kCoopWarps * G;
  for (int64_t b0 = ((int64_t)blockIdx.x * kCoopWarps + warp) * G; b0 < n; b0 += step) {
    const int np = (int)min((int64_t)G, n - b0);
    const int ne = np * m;
    const int32_t* gi = idx + b0 * m;
    const V* gv = reinterpret_cast<const V*>(val) + b0 * m;
    for (int e = lane; e < ne; e += 32) sidx[e] = __ldg(gi + e), sval[e] = (double)__ldg(gv + e);
    __syncwarp();
    const bool valid = lane < G * H && g < np;
    const int* ri = sidx + (valid ? g : 0) * m;
    const double* rv = sval + (valid ? g : 0) * m;
    double a0 = 0.0, a1 = 0.0;
    for (int t = 0; t < m; ++t) {
      const double v = rv[t];
      const double2 a = tabx[ri[t] * H + h];
      a0 = dadd(a0, dmul(v, a.x));
      a1 = dadd(a1, dmul(v, a.y));
    }
    for (int t = 0; t < m; ++t) {
      const double2 b = taby[ri[t] * H + h];
      a0 = dadd(a0, b.x);
      a1 = dadd(a1, b.y);
    }
    const double cs = colsq_pairwise_row(rv, m);
    const double d0 = dadd(a0, cs), d1 = dadd(a1, cs);
    double best = 0.0;
    int bk = 0;
#pragma unroll
    for (int q = 0; q < H; ++q) {
      const int src = (g * H + q) & 31;
      const double x = __shfl_sync(kFM, d0, src), y = __shfl_sync(kFM, d1, src);
      if (q == 0) best = x;
      else if (2 * q < K && x < best) best = x, bk = 2 * q;
      if (2 * q + 1 < K && y < best) best = y, bk = 2 * q + 1;
    }
    if (valid && h == 0) {
      const int64_t i = b0 + g;
      const double dm = best > 0.0 ? best : 0.0;  // np.clip(.., 0, None)
      labels[i] = bk;
      d2min[i] = dm;
      if (prev != nullptr) changed += prev[i] != bk;
      if (dm > bmax) bmax = dm, barg = i;  // ascending i per lane: keeps the first max
    }
    __syncwarp();  // the staging is reused by the next step
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const int64_t oc = __shfl_xor_sync(kFM, changed, o), oa = __shfl_xor_sync(kFM, barg, o);
    const double om = __shfl_xor_sync(kFM, bmax, o);
    changed += oc;
    if (oa >= 0 && (om > bmax || (om == bmax && (barg < 0 || oa < barg)))) bmax = om, barg = oa;
  }
  __shared__ int64_t s_ch[kCoopWarps], s_arg[kCoopWarps];
  __shared__ double s_mx[kCoopWarps];
  if (lane == 0) s_ch[warp] = changed, s_mx[warp] = bmax, s_arg[warp] = barg;
  __syncthreads();
  if (threadIdx.x == 0) {
    int64_t c = 0, a = -1;
    double mx = -1.0;
    for (int w = 0; w < kCoopWarps; ++w) {
      c += s_ch[w];
      if (s_arg[w] >= 0 && (s_mx[w] > mx || (s_mx[w] == mx && (a < 0 || s_arg[w] < a)))) mx = s_mx[w], a = s_arg[w];
    }
    blk_changed[blockIdx.x] = c;
    blk_max[blockIdx.x] = mx;
    blk_arg[blockIdx.x] = a;
  }
}
static size_t coop_smem(int32_t p_pad, int KC, int m) {
  const int H = KC / 2, G = 32 / H;
  return (size_t)p_pad * KC * 16 + (size_t)kCoopWarps * G * m * 12;
}

// K5r: K5c with one table pass. The shared table holds mu itself ([p_pad + 1][H] pairs, half of
// K5c's two planes, loaded straight from the centres: no table kernel; row p_pad is zero); a lane
// keeps the mu values of its point's coordinates in registers for the second half of the chain.
// The terms are the reference's bit for bit: fl((-2 v) mu) = fl(v (-2 mu)) (both round the same
// real number, the factors of -2 are exact) and fl(mu mu) is the table's square. Rows are staged
// padded to MT entries with (coordinate p_pad, value 0): a padded term is (-0)(0) = -0 or
// (0)(0) = +0, and adding a zero leaves the accumulator as it is (it starts at +0 and so is
// never -0), so the unrolled loops need no predicates and the loads batch ahead of the chain.
// Same chain order as K5c / K5s: labels and d2min are bit-identical. m <= MT <= 32 (registers).
#ifndef SKC_REG_WARPS
#define SKC_REG_WARPS 8
#endif
constexpr int kRegWarps = SKC_REG_WARPS;
// H (pairs of centres per point) as a sum of powers of two, widest first: component c has width
// w(c) and starts at pair o(c) (the spread table layout of K5r)
template <int H>
struct RegDecomp {
  static constexpr int n = ((H >> 3) & 1) + ((H >> 2) & 1) + ((H >> 1) & 1) + (H & 1);
  static constexpr int w(int c) {
    int seen = 0;
    for (int b = 8; b >= 1; b >>= 1)
      if (H & b) {
        if (seen == c) return b;
        ++seen;
      }
    return 1;
  }
  static constexpr int o(int c) {
    int sum = 0;
    for (int i = 0; i < c; ++i) sum += w(i);
    return sum;
  }
  static constexpr int comp(int h) {
    int c = 0;
    while (c + 1 < n && h >= o(c + 1)) ++c;
    return c;
  }
};
template <typename V, int H, int MT, bool SPREAD>
__global__ void __launch_bounds__(kRegWarps * 32, 1) km_assign_reg_kernel(
    const int32_t* __restrict__ idx, const void* __restrict__ val, int64_t n, int m, const double* __restrict__ mu,
    int K, int p_pad, const int32_t* __restrict__ prev, int32_t* __restrict__ labels, double* __restrict__ d2min,
    int64_t* __restrict__ blk_changed, double* __restrict__ blk_max, int64_t* __restrict__ blk_arg) {
  constexpr int G = 32 / H;                 // points per warp step
  constexpr int NE = G * MT;                // staged entries per warp step
  constexpr int RS = MT | 1;                // staged row stride (odd: the G rows start in distinct banks)
  constexpr int PF = (NE + 31) / 32;        // per lane
  constexpr bool kPrefetch = PF <= 8;       // next step's rows in registers during this step's chains
  extern __shared__ __align__(16) unsigned char csm[];
  // Table layouts. Compact: [p_pad + 1][H] pairs (mu[j][2h], mu[j][2h+1]); the 16 H-byte rows of
  // the two or three points inside a quarter-warp overlap banks (~7.5 wavefronts per 16-byte read
  // at H = 5). Spread (when it fits): H splits into its powers of two, widest first; component c
  // (width w, first pair o) has its own table of 128-byte rows holding 8 / w replicas of the
  // row's w pairs, its lanes form one region (point g at lanes G o + g w ...), and a lane reads
  // the replica that puts it at bank 4 (lane mod 8): every quarter-warp covers the 32 banks
  // once, whatever rows its points read (4 wavefronts per read).
  using RD = RegDecomp<H>;
  constexpr int NC = SPREAD ? RD::n : 1;
  constexpr int kRowBytes = SPREAD ? 128 : 16 * H;
  const size_t tab_bytes = (size_t)NC * (p_pad + 1) * kRowBytes;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double* sval = reinterpret_cast<double*>(csm + tab_bytes) + (size_t)warp * G * RS;
  int* sidx = reinterpret_cast<int*>(reinterpret_cast<double*>(csm + tab_bytes) + (size_t)kRegWarps * G * RS) +
              (size_t)warp * G * RS;
  if constexpr (SPREAD) {
    double2* tab = reinterpret_cast<double2*>(csm);
    for (int e = threadIdx.x; e < NC * (p_pad + 1) * 8; e += blockDim.x) {
      const int q = e & 7, j = (e >> 3) % (p_pad + 1), c = (e >> 3) / (p_pad + 1);
      const int hh = RD::o(c) + q % RD::w(c), c2 = 2 * hh;
      const double* r = mu + (size_t)j * K;
      const bool row = j < p_pad;
      tab[e] = make_double2(row && c2 < K ? __ldg(r + c2) : 0.0, row && c2 + 1 < K ? __ldg(r + c2 + 1) : 0.0);
    }
  } else {
    double2* tab = reinterpret_cast<double2*>(csm);
    for (int e = threadIdx.x; e < (p_pad + 1) * H; e += blockDim.x) {
      const int j = e / H, c = 2 * (e - j * H);
      const double* r = mu + (size_t)j * K;
      const bool row = j < p_pad;
      tab[e] = make_double2(row && c < K ? __ldg(r + c) : 0.0, row && c + 1 < K ? __ldg(r + c + 1) : 0.0);
    }
  }
  __syncthreads();
  // lane -> (point slot g, pair h) and the lane's byte offset inside a table row
  int g = lane / H, h = lane - g * H;
  const unsigned char* tlane = csm + 16 * h;
  if constexpr (SPREAD) {
#pragma unroll
    for (int c = 0; c < NC; ++c) {
      const int lo = G * RD::o(c), hi = lo + G * RD::w(c);
      if (lane >= lo && lane < hi) {
        const int r = lane - lo;
        g = r / RD::w(c);
        h = RD::o(c) + r % RD::w(c);
        tlane = csm + (size_t)c * (p_pad + 1) * 128 + 16 * (lane & 7);
      }
    }
  }
  const V* const vals = reinterpret_cast<const V*>(val);
  int64_t changed = 0;
  double bmax = -1.0;
  int64_t barg = -1;
  const int64_t step = (int64_t)gridDim.x * kRegWarps * G;
  int pi[PF];
  V pv[PF];
  // entry e of a step: point e / MT, slot e % MT; slots past m are the zero row
  auto fetch = [&](int64_t b0) {
#pragma unroll
    for (int q = 0; q < PF; ++q) {
      const int e = lane + 32 * q, gp = e / MT, t = e - gp * MT;
      const bool ok = e < NE && t < m && b0 + gp < n;
      const int64_t at = (b0 + gp) * m + t;
      pi[q] = ok ? __ldg(idx + at) : p_pad;
      pv[q] = ok ? __ldg(vals + at) : (V)0;
    }
  };
  int64_t b0 = ((int64_t)blockIdx.x * kRegWarps + warp) * G;
  if (kPrefetch && b0 < n) fetch(b0);
  for (; b0 < n; b0 += step) {
    if (!kPrefetch) fetch(b0);
#pragma unroll
    for (int q = 0; q < PF; ++q) {
      const int e = lane + 32 * q, gp = e / MT;
      if (e < NE) sidx[e + gp * (RS - MT)] = pi[q], sval[e + gp * (RS - MT)] = (double)pv[q];
    }
    __syncwarp();
    if (kPrefetch && b0 + step < n) fetch(b0 + step);
    const int np = (int)min((int64_t)G, n - b0);
    const bool valid = lane < G * H && g < np;
    const int* ri = sidx + (lane < G * H ? g : 0) * RS;
    const double* rv = sval + (lane < G * H ? g : 0) * RS;
    double m0[MT], m1[MT];
    double a0 = 0.0, a1 = 0.0;
    // colsq in numpy's pairwise order from the same value reads: eight running sums over the
    // full groups of eight (t < m8), the tail added in order after their combine
    const int m8 = m < 8 ? 0 : m - (m & 7);
    double r8[8] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
#pragma unroll
    for (int t = 0; t < MT; ++t) {
      const double v = rv[t];
      if (t < 8) r8[t] = dmul(v, v);  // slots >= m8 are not used below
      else if (t < m8) r8[t & 7] = dadd(r8[t & 7], dmul(v, v));
      const double v2 = dmul(-2.0, v);
      const double2 u = *reinterpret_cast<const double2*>(tlane + (size_t)ri[t] * kRowBytes);
      m0[t] = u.x;
      m1[t] = u.y;
      a0 = dadd(a0, dmul(v2, u.x));
      a1 = dadd(a1, dmul(v2, u.y));
    }
#pragma unroll
    for (int t = 0; t < MT; ++t) {
      a0 = dadd(a0, dmul(m0[t], m0[t]));
      a1 = dadd(a1, dmul(m1[t], m1[t]));
    }
    double cs = 0.0;
    if (m8) cs = dadd(dadd(dadd(r8[0], r8[1]), dadd(r8[2], r8[3])), dadd(dadd(r8[4], r8[5]), dadd(r8[6], r8[7])));
    for (int t = m8; t < m; ++t) cs = dadd(cs, dmul(rv[t], rv[t]));
    const double d0 = dadd(a0, cs), d1 = dadd(a1, cs);
    double best = 0.0;
    int bk = 0;
#pragma unroll
    for (int q = 0; q < H; ++q) {
      const int src = (SPREAD ? G * RD::o(RD::comp(q)) + g * RD::w(RD::comp(q)) + q - RD::o(RD::comp(q)) : g * H + q) & 31;
      const double x = __shfl_sync(kFM, d0, src), y = __shfl_sync(kFM, d1, src);
      if (q == 0) best = x;
      else if (2 * q < K && x < best) best = x, bk = 2 * q;
      if (2 * q + 1 < K && y < best) best = y, bk = 2 * q + 1;
    }
    if (valid && h == 0) {
      const int64_t i = b0 + g;
      const double dm = best > 0.0 ? best : 0.0;  // np.clip(.., 0, None)
      labels[i] = bk;
      d2min[i] = dm;
      if (prev != nullptr) changed += prev[i] != bk;
      if (dm > bmax) bmax = dm, barg = i;  // ascending i per lane: keeps the first max
    }
    __syncwarp();  // the staging is reused by the next step
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const int64_t oc = __shfl_xor_sync(kFM, changed, o), oa = __shfl_xor_sync(kFM, barg, o);
    const double om = __shfl_xor_sync(kFM, bmax, o);
    changed += oc;
    if (oa >= 0 && (om > bmax || (om == bmax && (barg < 0 || oa < barg)))) bmax = om, barg = oa;
  }
  __shared__ int64_t s_ch[kRegWarps], s_arg[kRegWarps];
  __shared__ double s_mx[kRegWarps];
  if (lane == 0) s_ch[warp] = changed, s_mx[warp] = bmax, s_arg[warp] = barg;
  __syncthreads();
  if (threadIdx.x == 0) {
    int64_t c = 0, a = -1;
    double mx = -1.0;
    for (int w = 0; w < kRegWarps; ++w) {
      c += s_ch[w];
      if (s_arg[w] >= 0 && (s_mx[w] > mx || (s_mx[w] == mx && (a < 0 || s_arg[w] < a)))) mx = s_mx[w], a = s_arg[w];
    }
    blk_changed[blockIdx.x] = c;
    blk_max[blockIdx.x] = mx;
    blk_arg[blockIdx.x] = a;
  }
}
static int reg_mt(int m) { return m <= 8 ? 8 : m <= 16 ? 16 : m <= 24 ? 24 : m <= 28 ? 28 : 32; }
static size_t reg_smem(int32_t p_pad, int KC, int m, bool spread) {
  const int H = KC / 2, G = 32 / H;
  const int nc = ((H >> 3) & 1) + ((H >> 2) & 1) + ((H >> 1) & 1) + (H & 1);
  const size_t tab = spread ? (size_t)nc * (p_pad + 1) * 128 : (size_t)(p_pad + 1) * KC * 8;
  return tab + (size_t)kRegWarps * G * (reg_mt(m) | 1) * 12;
}

__global__ void km_assign_reduce_kernel(const int64_t* __restrict__ blk_changed, const double* __restrict__ blk_max,
                                        const int64_t* __restrict__ blk_arg, int nb, int64_t* out, double* d2max) {
  int64_t c = 0, a = -1;
  double mx = -1.0;
  for (int b = threadIdx.x; b < nb; b += blockDim.x) {
    c += blk_changed[b];
    if (blk_arg[b] >= 0 && (blk_max[b] > mx || (blk_max[b] == mx && blk_arg[b] < a))) {
      mx = blk_max[b];
      a = blk_arg[b];
    }
  }
  // warp then block combine: (max value, smallest index among ties), sum of changed
  __shared__ int64_t sc[32], sa[32];
  __shared__ double sm[32];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const int64_t oc = __shfl_xor_sync(kFM, c, o), oa = __shfl_xor_sync(kFM, a, o);
    const double om = __shfl_xor_sync(kFM, mx, o);
    c += oc;
    if (oa >= 0 && (om > mx || (om == mx && (a < 0 || oa < a)))) {
      mx = om;
      a = oa;
    }
  }
  const int w = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0) {
    sc[w] = c;
    sa[w] = a;
    sm[w] = mx;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    int64_t C = 0, A = -1;
    double M = -1.0;
    for (int i = 0; i < (int)(blockDim.x >> 5); ++i) {
      C += sc[i];
      if (sa[i] >= 0 && (sm[i] > M || (sm[i] == M && (A < 0 || sa[i] < A)))) {
        M = sm[i];
        A = sa[i];
      }
    }
    out[0] = C;
    out[1] = A;
    if (d2max) d2max[0] = M;
  }
}

// ======================================================================================
// K5f: exact assignment by filter and verify, for tables that do not fit shared memory
// (C5: p=2048, K=100). The exact kernel above is L2-bound there: every (point, centre)
// gathers 2m table doubles. Here a warp takes one point at a time:
//  filter  lanes = centres: d~ = colsq + sum_t fl32(v_t)*(-2 mu32) + mu32^2 with FMAs, and
//          S = colsq + sum_t |v_t*(-2 mu32)| + mu32^2. A rigorous bound on |d~ - d| for the
//          exact fp64 value d (reference order) is E = S ((2m+8) 2^-24 + (2m+1) 2^-53) 1.01:
//          input conversion (3 u per product), recursive summation (2m u), fp64's own error.
//          Every centre with d~ - E <= min(d~ + E) is a candidate; the exact argmin is one.
//  verify  queued (point, candidate) pairs, 32 at a time, get the exact fp64 value in the
//          reference order (the same arithmetic as km_assign_kernel), and each point takes
//          the first minimum over its candidates (np.argmin), d2min = max(d, 0).
// Labels, d2min, the changed count and the farthest point are bit-identical to K5.
// ======================================================================================
constexpr int kFiltWarps = 8;
// per warp queue of (point, candidate) pairs: flushed once it holds >= 32 (+ one point's K)
__host__ __device__ inline size_t filt_warp_bytes(int m, int K) { return (size_t)m * 16 + (size_t)(32 + K) * 24 + 33 * 16; }

// fp32 copy of mu as [p][K4] rows (K4 = K rounded up to 4, zero padded): a lane reads 4 centres
// with one 16-byte load
__global__ void km_tables32_kernel(const double* __restrict__ mu, int32_t p_pad, int K, int K4,
                                   float* __restrict__ t32) {
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= (int64_t)p_pad * K4) return;
  const int64_t j = e / K4;
  const int k = (int)(e - j * K4);
  t32[e] = k < K ? (float)mu[j * K + k] : 0.f;
}
__device__ __forceinline__ uint64_t fma2(uint64_t a, uint64_t b, uint64_t c) {
  uint64_t r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
  return r;
}
__device__ __forceinline__ uint64_t pk2(float lo, float hi) {
  uint64_t r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
  return r;
}
__device__ __forceinline__ void upk2(uint64_t x, float& lo, float& hi) {
  asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(x));
}

#ifndef SKC_FILT_MINB
#define SKC_FILT_MINB 4  // 4 CTAs per SM (64 registers), 8-deep unroll: measured best for C5 (tools/ab_c5.sh)
#endif
#ifndef SKC_FILT_UNROLL
#define SKC_FILT_UNROLL 8
#endif
constexpr int kFiltUnroll = SKC_FILT_UNROLL;
template <typename V, int NB>  // NB = ceil(K4 / 128) blocks of 4 centres per lane
__global__ void __launch_bounds__(kFiltWarps * 32, SKC_FILT_MINB)
    km_assign_filter_kernel(const int32_t* __restrict__ idx, const void* __restrict__ val, int64_t n, int m,
                            const float* __restrict__ t32, int K4, const double* __restrict__ tabx,
                            const double* __restrict__ taby, int K,
                            const int32_t* __restrict__ prev, int32_t* __restrict__ labels,
                            double* __restrict__ d2min, int64_t* __restrict__ blk_changed,
                            double* __restrict__ blk_max, int64_t* __restrict__ blk_arg,
                            const int64_t* __restrict__ list, const int32_t* __restrict__ list_n) {
  // list != nullptr: only the points list[0 .. *list_n) (K5t's unresolved points)
  extern __shared__ __align__(16) unsigned char sm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // per warp: sidx[m] (j*K), sval[m] (double), sv32[m], queue (i, k, colsq, d), point table
  const int qcap = 32 + K;
  unsigned char* wb = sm + filt_warp_bytes(m, K) * warp;
  double* sval = reinterpret_cast<double*>(wb);
  int* sidx = reinterpret_cast<int*>(wb + (size_t)m * 8);
  float* sv32 = reinterpret_cast<float*>(wb + (size_t)m * 12);
  double* qc = reinterpret_cast<double*>(wb + (size_t)m * 16);  // colsq per queued pair
  double* qd = qc + qcap;                                        // exact value per queued pair
  int* qk = reinterpret_cast<int*>(qd + qcap);                   // centre per queued pair
  int* qp = qk + qcap;                                           // point slot per queued pair
  int64_t* pi = reinterpret_cast<int64_t*>(qp + qcap);           // point index per slot (32)
  int* pstart = reinterpret_cast<int*>(pi + 33);                 // first queue entry per slot (33)
  const double eu = ((2.0 * m + 16.0) * 0x1p-24 + (2.0 * m + 1.0) * 0x1p-53) * 1.1;
  int64_t changed = 0;
  double bmax = -1.0;
  int64_t barg = -1;
  int qn = 0, np = 0;  // queued pairs, queued points
  auto flush = [&]() {
    // exact values: lanes = pairs (the reference order of km_assign_kernel)
    for (int q0 = 0; q0 < qn; q0 += 32) {
      const int q = q0 + lane;
      if (q < qn) {
        const int64_t i = pi[qp[q]];
        const int k = qk[q];
        const int32_t* ir = idx + i * m;
        const double* tkx = tabx + k;
        const double* tky = taby + k;
        double acc = 0.0;
        for (int t = 0; t < m; ++t) acc = dadd(acc, dmul(ldd<V>(val, i * m + t), tkx[(size_t)__ldg(ir + t) * K]));
        for (int t = 0; t < m; ++t) acc = dadd(acc, tky[(size_t)__ldg(ir + t) * K]);
        qd[q] = dadd(acc, qc[q]);
      }
    }
    __syncwarp();
    // each point: first minimum over its candidates (queued in ascending k)
    if (lane < np) {
      const int64_t i = pi[lane];
      double best = 0.0;
      int bk = -1;
      for (int q = pstart[lane]; q < pstart[lane + 1]; ++q)  // queued in any order: lowest k on ties
        if (bk < 0 || qd[q] < best || (qd[q] == best && qk[q] < bk)) best = qd[q], bk = qk[q];
      const double dm = best > 0.0 ? best : 0.0;  // np.clip(.., 0, None)
      labels[i] = bk;
      d2min[i] = dm;
      if (prev != nullptr) changed += prev[i] != bk;
      if (dm > bmax || (dm == bmax && (barg < 0 || i < barg))) bmax = dm, barg = i;
    }
    __syncwarp();
    qn = 0;
    np = 0;
  };
  const int64_t gw = (int64_t)blockIdx.x * kFiltWarps + warp, nw = (int64_t)gridDim.x * kFiltWarps;
  const int64_t cnt = list ? (int64_t)*list_n : n;
  for (int64_t li = gw; li < cnt; li += nw) {
    const int64_t i = list ? list[li] : li;
    __syncwarp();
    for (int t = lane; t < m; t += 32) {
      const double v = ldd<V>(val, i * m + t);
      sidx[t] = __ldg(idx + i * m + t) * K4;
      sval[t] = v;
      sv32[t] = (float)v;
    }
    __syncwarp();
    // colsq = (v*v).sum() in numpy's pairwise order (as km_assign_kernel)
    double colsq = 0.0;
    if (m < 8) {
      if (lane == 0)
        for (int t = 0; t < m; ++t) colsq = dadd(colsq, dmul(sval[t], sval[t]));
    } else if (m <= 128) {
      double r = 0.0;
      if (lane < 8) {
        r = dmul(sval[lane], sval[lane]);
        for (int t = 8 + lane; t < m - (m % 8); t += 8) r = dadd(r, dmul(sval[t], sval[t]));
      }
      const double r1 = __shfl_down_sync(kFM, r, 1);
      const double s01 = dadd(r, r1);
      const double s23 = __shfl_down_sync(kFM, s01, 2);
      const double q = dadd(s01, s23);
      const double q2 = __shfl_down_sync(kFM, q, 4);
      if (lane == 0) {
        colsq = dadd(q, q2);
        for (int t = m - (m % 8); t < m; ++t) colsq = dadd(colsq, dmul(sval[t], sval[t]));
      }
    } else if (lane == 0) {
      double* tmp = sval;  // square in place, restore after
      for (int t = 0; t < m; ++t) tmp[t] = dmul(sval[t], sval[t]);
      colsq = pw_rec(tmp, m);
      for (int t = 0; t < m; ++t) tmp[t] = ldd<V>(val, i * m + t);
    }
    __syncwarp();
    colsq = __shfl_sync(kFM, colsq, 0);
    // filter: lane owns centres k = lane + 32 b (b < NB), one walk over the support:
    // P = sum u^2 and Q = sum u v in fp32 (u = fl32(mu[j_t, k]), v = fl32(v_t)), d~ = P - 2Q + colsq.
    // Cauchy-Schwarz: sum |u v| <= sqrt(P colsq), so every term's magnitude sums to at most
    // S = P + 2 sqrt(P colsq) + colsq, and |d~ - d| <= E = S ((2m+16) 2^-24 + (2m+1) 2^-53) 1.1
    // (input conversion, fp32 accumulation and combination, fp64's own rounding).
    // P, Q as packed fp32 pairs: lane owns centres k = 128 b + 4 lane + c (c < 4)
    uint64_t P[NB][2], Q[NB][2];
#pragma unroll
    for (int b = 0; b < NB; ++b) P[b][0] = P[b][1] = Q[b][0] = Q[b][1] = 0;
    const float* tl = t32 + 4 * lane;
    bool okb[NB];
#pragma unroll
    for (int b = 0; b < NB; ++b) okb[b] = 128 * b + 4 * lane < K4;
    // unrolled: SKC_FILT_UNROLL * NB independent 16-byte gathers in flight per lane
#pragma unroll kFiltUnroll
    for (int t = 0; t < m; ++t) {
      const float* row = tl + sidx[t];
      const float v = sv32[t];
      const uint64_t vv = pk2(v, v);
#pragma unroll
      for (int b = 0; b < NB; ++b) {
        const float4 u = okb[b] ? __ldg(reinterpret_cast<const float4*>(row + 128 * b)) : make_float4(0.f, 0.f, 0.f, 0.f);
        const uint64_t u01 = pk2(u.x, u.y), u23 = pk2(u.z, u.w);
        P[b][0] = fma2(u01, u01, P[b][0]);
        P[b][1] = fma2(u23, u23, P[b][1]);
        Q[b][0] = fma2(u01, vv, Q[b][0]);
        Q[b][1] = fma2(u23, vv, Q[b][1]);
      }
    }
    float dl[NB][4], el[NB][4];
    float ub = __int_as_float(0x7F800000);
    const bool wide = !(colsq >= 0x1p-90 && colsq <= 0x1p100);
#pragma unroll
    for (int b = 0; b < NB; ++b) {
      float pf[4], qf[4];
      upk2(P[b][0], pf[0], pf[1]);
      upk2(P[b][1], pf[2], pf[3]);
      upk2(Q[b][0], qf[0], qf[1]);
      upk2(Q[b][1], qf[2], qf[3]);
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        dl[b][c] = __int_as_float(0x7F800000);
        el[b][c] = 0.f;
        if (128 * b + 4 * lane + c < K) {
          const double Pd = pf[c];
          dl[b][c] = (float)(Pd - 2.0 * (double)qf[c] + colsq);
          el[b][c] = (float)((Pd + 2.0 * sqrt(Pd * colsq) + colsq) * eu) * 1.001f;
          ub = fminf(ub, dl[b][c] + el[b][c]);
        }
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) ub = fminf(ub, __shfl_xor_sync(kFM, ub, o));  // over all centres
    // queue the candidates (the flush breaks ties by the lowest k, so any queue order works)
    if (lane == 0) pi[np] = i, pstart[np] = qn;
#pragma unroll
    for (int b = 0; b < NB; ++b) {
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const int k = 128 * b + 4 * lane + c;
        // outside the range the fp32 bound covers (colsq beyond [2^-90, 2^100], or a non-finite
        // estimate), every centre stays a candidate and the exact pass decides
        const bool cand = k < K && (wide || !isfinite(dl[b][c]) || !isfinite(el[b][c]) || dl[b][c] - el[b][c] <= ub);
        const unsigned mk = __ballot_sync(kFM, cand);
        if (cand) {
          const int q = qn + __popc(mk & ((1u << lane) - 1u));
          qk[q] = k;
          qp[q] = np;
          qc[q] = colsq;
        }
        qn += __popc(mk);
      }
    }
    ++np;
    if (lane == 0) pstart[np] = qn;
    __syncwarp();
    if (qn >= 32 || np == 32) flush();
  }
  if (np > 0) flush();
  // block reduction over all lanes: changed sum, (max, first index)
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const int64_t oc = __shfl_xor_sync(kFM, changed, o), oa = __shfl_xor_sync(kFM, barg, o);
    const double om = __shfl_xor_sync(kFM, bmax, o);
    changed += oc;
    if (oa >= 0 && (om > bmax || (om == bmax && (barg < 0 || oa < barg)))) bmax = om, barg = oa;
  }
  __shared__ int64_t s_ch[kFiltWarps], s_arg[kFiltWarps];
  __shared__ double s_mx[kFiltWarps];
  if (lane == 0) s_ch[warp] = changed, s_mx[warp] = bmax, s_arg[warp] = barg;
  __syncthreads();
  if (threadIdx.x == 0) {
    int64_t c = 0, a = -1;
    double mx = -1.0;
    for (int w = 0; w < kFiltWarps; ++w) {
      c += s_ch[w];
      if (s_arg[w] >= 0 && (s_mx[w] > mx || (s_mx[w] == mx && (a < 0 || s_arg[w] < a)))) mx = s_mx[w], a = s_arg[w];
    }
    blk_changed[blockIdx.x] = c;
    blk_max[blockIdx.x] = mx;
    blk_arg[blockIdx.x] = a;
  }
}

static int assign_grid(int64_t n) {
  int64_t g = (n + kAsgWarps - 1) / kAsgWarps;
  const int64_t cap = 4 * (int64_t)sm_count();
  if (g > cap) g = cap;
  return (int)(g < 1 ? 1 : g);
}

// tables: 2 p_pad * K doubles ([-2 mu] and [mu * mu] planes), or the padded planes of K5s
static size_t assign_tab_doubles(int32_t p_pad, int32_t K) { return (size_t)2 * p_pad * ((K + 1) & ~1); }
size_t assign_ws(int64_t n, int32_t p_pad, int32_t K) {
  // [tables][per-block changed/max/arg][fp32 table for K5f]
  return assign_tab_doubles(p_pad, K) * sizeof(double) + (size_t)assign_grid(n) * 24 +
         (size_t)p_pad * ((K + 3) & ~3) * 4 + 128;
}
// K5f instead of K5 when the packed table does not fit the shared-memory budget (SKC_ASSIGN_EXACT=1
// keeps K5, for A/B runs and the bit-equality test)
static bool use_filter(int32_t p_pad, int32_t K) {
  if (K > 256) return false;
  if (const char* e = getenv("SKC_ASSIGN_EXACT")) return e[0] != '1';
  // K5 packs 2 or 4 points per warp for K <= 16 and stays faster there (C2: 2.25 vs 2.95 ms)
  return K > 16 && (size_t)p_pad * K * 16 > 40 * 1024;
}

template <typename V, int KP>
static void launch_assign_kp(int G, const int32_t* idx, const void* val, int64_t n, int32_t m, const double* tx,
                             const double* ty,
                             int32_t K, int32_t p_pad, const int32_t* prev, int32_t* labels, double* d2min,
                             int64_t* bch, double* bmx, int64_t* barg, cudaStream_t st) {
  constexpr int GP = 32 / KP;
  const size_t per_warp = ((size_t)GP * m * 4 + 15) / 16 * 16 + (size_t)GP * m * 8;
  const size_t tab_bytes = (size_t)p_pad * K * 16;
  int warps = kAsgWarps;
  while (warps > 1 && per_warp * warps > 50 * 1024) warps >>= 1;  // 4 CTAs per SM
  if (tab_bytes + per_warp * warps <= 50 * 1024) {
    auto k = km_assign_kernel<V, KP, true>;
    const size_t smem = tab_bytes + per_warp * warps;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k<<<G, warps * 32, smem, st>>>(idx, val, n, m, tx, ty, K, p_pad, prev, labels, d2min, bch, bmx, barg);
  } else {
    auto k = km_assign_kernel<V, KP, false>;
    const size_t smem = per_warp * warps;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k<<<G, warps * 32, smem, st>>>(idx, val, n, m, tx, ty, K, p_pad, prev, labels, d2min, bch, bmx, barg);
  }
}

int assign_launch(const int32_t* idx, const void* val, int val_f64, int64_t n, int32_t m, const double* mu,
                  int32_t p_pad, int32_t K, const int32_t* prev, int32_t* labels, double* d2min, int64_t* out,
                  double* d2max, void* ws, cudaStream_t st) {
  double* tx = reinterpret_cast<double*>(ws);  // [-2 mu] plane, then the [mu * mu] plane
  double* ty = tx + (size_t)p_pad * K;
  const int G = assign_grid(n);
  int64_t* bch = reinterpret_cast<int64_t*>(tx + assign_tab_doubles(p_pad, K));
  // K5s for small tables: one point per thread (SKC_ASSIGN_SMALL=0 keeps the warp kernel)
  static const bool small_on = [] {
    const char* e = getenv("SKC_ASSIGN_SMALL");
    return !(e && e[0] == '0');
  }();
  if (n > 0 && small_on && K <= 16 && m <= 128 && !use_filter(p_pad, K)) {
    const int KC = (K + 1) & ~1;
    // K5r when m fits the register copy of the row's centres (SKC_ASSIGN_REG=0: K5c / K5s)
    const char* reg_env = getenv("SKC_ASSIGN_REG");  // read per call: tests compare the kernels
    const bool reg_on = !(reg_env && reg_env[0] == '0');
    // the spread (conflict-free) table when it fits beside the staging (SKC_ASSIGN_SPREAD=0: compact)
    const char* spr_env = getenv("SKC_ASSIGN_SPREAD");
    const bool spread = !(spr_env && spr_env[0] == '0') && reg_smem(p_pad, KC, m, true) <= 200 * 1024 &&
                        KC / 2 != 8;  // H = 8: a quarter-warp reads one 128-byte row as it is
    const size_t rsm = reg_smem(p_pad, KC, m, spread);
    if (reg_on && m <= 32 && rsm <= 200 * 1024) {
      const int H = KC / 2, Gp = 32 / H;
      int64_t Gc = (n + (int64_t)kRegWarps * Gp - 1) / ((int64_t)kRegWarps * Gp);
      const int64_t cap = (int64_t)sm_count();  // one CTA per SM (registers)
      if (Gc > cap) Gc = cap;
      if (Gc > G) Gc = G;  // the per-block arrays hold G entries
      auto gor = [&](auto kern) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)rsm);
        kern<<<(unsigned)Gc, kRegWarps * 32, rsm, st>>>(idx, val, n, m, mu, K, p_pad, prev, labels, d2min, bch,
                                                         reinterpret_cast<double*>(bch + G),
                                                         reinterpret_cast<int64_t*>(bch + 2 * G));
      };
#define SKC_REG_MT(HH, MM)                                                        \
  if (spread) {                                                                   \
    if (val_f64) gor(km_assign_reg_kernel<double, HH, MM, true>);                 \
    else gor(km_assign_reg_kernel<float, HH, MM, true>);                          \
  } else {                                                                        \
    if (val_f64) gor(km_assign_reg_kernel<double, HH, MM, false>);                \
    else gor(km_assign_reg_kernel<float, HH, MM, false>);                         \
  }
#define SKC_REG_CASE(HH)                                                          \
  case HH:                                                                        \
    switch (reg_mt(m)) {                                                          \
      case 8: SKC_REG_MT(HH, 8) break;                                            \
      case 16: SKC_REG_MT(HH, 16) break;                                          \
      case 24: SKC_REG_MT(HH, 24) break;                                          \
      case 28: SKC_REG_MT(HH, 28) break;                                          \
      default: SKC_REG_MT(HH, 32) break;                                          \
    }                                                                             \
    break;
      switch (H) {
        SKC_REG_CASE(1)
        SKC_REG_CASE(2)
        SKC_REG_CASE(3)
        SKC_REG_CASE(4)
        SKC_REG_CASE(5)
        SKC_REG_CASE(6)
        SKC_REG_CASE(7)
        SKC_REG_CASE(8)
      }
#undef SKC_REG_CASE
#undef SKC_REG_MT
      int rcr = check_launch("km_assign_reg_kernel");
      if (rcr) return rcr;
      km_assign_reduce_kernel<<<1, 1024, 0, st>>>(bch, reinterpret_cast<double*>(bch + G),
                                                  reinterpret_cast<int64_t*>(bch + 2 * G), (int)Gc, out, d2max);
      return check_launch("km_assign_reduce_kernel");
    }
    double* tx2 = tx;
    double* ty2 = tx + (size_t)p_pad * KC;
    const int64_t tot = (int64_t)p_pad * KC;
    km_tables_pad_kernel<<<(unsigned)((tot + 255) / 256), 256, 0, st>>>(mu, p_pad, K, KC, tx2, ty2);
    int rc = check_launch("km_tables_pad_kernel");
    if (rc) return rc;
    // K5c when the padded tables fit shared memory next to the row staging (SKC_ASSIGN_COOP=0: K5s)
    const char* coop_env = getenv("SKC_ASSIGN_COOP");  // read per call: tests compare both kernels
    const bool coop_on = !(coop_env && coop_env[0] == '0');
    const size_t csm = coop_smem(p_pad, KC, m);
    if (coop_on && m <= 64 && csm <= 110 * 1024) {
      const int H = KC / 2, Gp = 32 / H;
      int64_t Gc = (n + (int64_t)kCoopWarps * Gp - 1) / ((int64_t)kCoopWarps * Gp);
      const int64_t cap = 2 * (int64_t)sm_count();
      if (Gc > cap) Gc = cap;
      if (Gc > G) Gc = G;  // the per-block arrays hold G entries
      auto goc = [&](auto kern) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)csm);
        kern<<<(unsigned)Gc, kCoopWarps * 32, csm, st>>>(idx, val, n, m, tx2, ty2, K, p_pad, prev, labels, d2min, bch,
                                                          reinterpret_cast<double*>(bch + G),
                                                          reinterpret_cast<int64_t*>(bch + 2 * G));
      };
#define SKC_COOP_CASE(HH)                                              \
  case HH:                                                             \
    if (val_f64) goc(km_assign_coop_kernel<double, HH>);               \
    else goc(km_assign_coop_kernel<float, HH>);                        \
    break;
      switch (H) {
        SKC_COOP_CASE(1)
        SKC_COOP_CASE(2)
        SKC_COOP_CASE(3)
        SKC_COOP_CASE(4)
        SKC_COOP_CASE(5)
        SKC_COOP_CASE(6)
        SKC_COOP_CASE(7)
        SKC_COOP_CASE(8)
      }
#undef SKC_COOP_CASE
      if ((rc = check_launch("km_assign_coop_kernel"))) return rc;
      km_assign_reduce_kernel<<<1, 1024, 0, st>>>(bch, reinterpret_cast<double*>(bch + G),
                                                  reinterpret_cast<int64_t*>(bch + 2 * G), (int)Gc, out, d2max);
      return check_launch("km_assign_reduce_kernel");
    }
    int64_t Gs = (n + kSmallThreads - 1) / kSmallThreads;
    if (Gs > G) Gs = G;  // the per-block arrays hold G entries
    auto go = [&](auto kern) {
      kern<<<(unsigned)Gs, kSmallThreads, 0, st>>>(idx, val, n, m, tx2, ty2, K, prev, labels, d2min, bch,
                                         reinterpret_cast<double*>(bch + G), reinterpret_cast<int64_t*>(bch + 2 * G));
    };
#define SKC_SMALL_CASE(KK)                                                              \
  case KK:                                                                              \
    if (val_f64) go(km_assign_small_kernel<double, KK>);                                \
    else go(km_assign_small_kernel<float, KK>);                                         \
    break;
    switch (KC) {
      SKC_SMALL_CASE(2)
      SKC_SMALL_CASE(4)
      SKC_SMALL_CASE(6)
      SKC_SMALL_CASE(8)
      SKC_SMALL_CASE(10)
      SKC_SMALL_CASE(12)
      SKC_SMALL_CASE(14)
      SKC_SMALL_CASE(16)
    }
#undef SKC_SMALL_CASE
    if ((rc = check_launch("km_assign_small_kernel"))) return rc;
    km_assign_reduce_kernel<<<1, 1024, 0, st>>>(bch, reinterpret_cast<double*>(bch + G),
                                                reinterpret_cast<int64_t*>(bch + 2 * G), (int)Gs, out, d2max);
    return check_launch("km_assign_reduce_kernel");
  }
  double* bmx = reinterpret_cast<double*>(bch + G);
  int64_t* barg = reinterpret_cast<int64_t*>(bmx + G);
  const int64_t total = (int64_t)p_pad * K;
  km_tables2_kernel<<<(unsigned)((total + 255) / 256), 256, 0, st>>>(mu, total, tx, ty);
  int rc = check_launch("km_tables2_kernel");
  if (rc) return rc;
  if (n > 0 && use_filter(p_pad, K)) {
    float* t32 = reinterpret_cast<float*>((reinterpret_cast<uintptr_t>(barg + G) + 127) & ~(uintptr_t)127);
    const int K4 = (K + 3) & ~3;
    km_tables32_kernel<<<(unsigned)(((int64_t)p_pad * K4 + 255) / 256), 256, 0, st>>>(mu, p_pad, K, K4, t32);
    if ((rc = check_launch("km_tables32_kernel"))) return rc;
    const size_t smem = filt_warp_bytes(m, K) * kFiltWarps;
    int Gf = (int)((n + kFiltWarps - 1) / kFiltWarps);
    if (Gf > G) Gf = G;  // the per-block arrays hold G entries
    const int nb = (K4 + 127) / 128;
    auto go = [&](auto kern) {
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      kern<<<Gf, kFiltWarps * 32, smem, st>>>(idx, val, n, m, t32, K4, tx, ty, K, prev, labels, d2min, bch, bmx, barg,
                                               nullptr, nullptr);
    };
    if (val_f64) {
      switch (nb) {
        case 1: go(km_assign_filter_kernel<double, 1>); break;
        default: go(km_assign_filter_kernel<double, 2>); break;  // use_filter: K <= 256
      }
    } else {
      switch (nb) {
        case 1: go(km_assign_filter_kernel<float, 1>); break;
        default: go(km_assign_filter_kernel<float, 2>); break;  // use_filter: K <= 256
      }
    }
    if ((rc = check_launch("km_assign_filter_kernel"))) return rc;
    km_assign_reduce_kernel<<<1, 1024, 0, st>>>(bch, bmx, barg, Gf, out, d2max);
    return check_launch("km_assign_reduce_kernel");
  }
  if (n > 0) {
    if (val_f64) {
      if (K <= 8) launch_assign_kp<double, 8>(G, idx, val, n, m, tx, ty, K, p_pad, prev, labels, d2min, bch, bmx, barg, st);
      else if (K <= 16) launch_assign_kp<double, 16>(G, idx, val, n, m, tx, ty, K, p_pad, prev, labels, d2min, bch, bmx, barg, st);
      else launch_assign_kp<double, 32>(G, idx, val, n, m, tx, ty, K, p_pad, prev, labels, d2min, bch, bmx, barg, st);
    } else {
      if (K <= 8) launch_assign_kp<float, 8>(G, idx, val, n, m, tx, ty, K, p_pad, prev, labels, d2min, bch, bmx, barg, st);
      else if (K <= 16) launch_assign_kp<float, 16>(G, idx, val, n, m, tx, ty, K, p_pad, prev, labels, d2min, bch, bmx, barg, st);
      else launch_assign_kp<float, 32>(G, idx, val, n, m, tx, ty, K, p_pad, prev, labels, d2min, bch, bmx, barg, st);
    }
    rc = check_launch("km_assign_kernel");
    if (rc) return rc;
  }
  km_assign_reduce_kernel<<<1, 1024, 0, st>>>(bch, bmx, barg, n > 0 ? G : 0, out, d2max);
  return check_launch("km_assign_reduce_kernel");
}

// K5f over a device-side list of points (K5t's unresolved points), G blocks of partials
int assign_filter_list_launch(const int32_t* idx, const void* val, int val_f64, int64_t n, int32_t m,
                              const double* mu, int32_t p_pad, int32_t K, const int32_t* prev, int32_t* labels,
                              double* d2min, const int64_t* list, const int32_t* list_n, const double* tx,
                              const double* ty,
                              float* t32, int64_t* bch, double* bmx, int64_t* barg, int G, cudaStream_t st) {
  if (K > 256) return fail(SKC_EPARAM, "K5f list pass needs K <= 256");
  const int K4 = (K + 3) & ~3;
  km_tables32_kernel<<<(unsigned)(((int64_t)p_pad * K4 + 255) / 256), 256, 0, st>>>(mu, p_pad, K, K4, t32);
  int rc = check_launch("km_tables32_kernel");
  if (rc) return rc;
  const size_t smem = filt_warp_bytes(m, K) * kFiltWarps;
  auto go = [&](auto kern) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    kern<<<G, kFiltWarps * 32, smem, st>>>(idx, val, n, m, t32, K4, tx, ty, K, prev, labels, d2min, bch, bmx, barg, list,
                                            list_n);
  };
  const int nb = (K4 + 127) / 128;
  if (val_f64) {
    if (nb == 1) go(km_assign_filter_kernel<double, 1>);
    else go(km_assign_filter_kernel<double, 2>);
  } else {
    if (nb == 1) go(km_assign_filter_kernel<float, 1>);
    else go(km_assign_filter_kernel<float, 2>);
  }
  return check_launch("km_assign_filter_kernel (list)");
}

int assign_reduce_launch(const int64_t* bch, const double* bmx, const int64_t* barg, int G, int64_t* out,
                         double* d2max, cudaStream_t st) {
  km_assign_reduce_kernel<<<1, 1024, 0, st>>>(bch, bmx, barg, G, out, d2max);
  return check_launch("km_assign_reduce_kernel");
}

int tables2_launch(const double* mu, int32_t p_pad, int32_t K, double* tx, double* ty, cudaStream_t st) {
  const int64_t total = (int64_t)p_pad * K;
  km_tables2_kernel<<<(unsigned)((total + 255) / 256), 256, 0, st>>>(mu, total, tx, ty);
  return check_launch("km_tables2_kernel");
}

// ---------------------------------------------------------------------------------
// partials (exact): see the transposed-sketch section below
size_t csc_ws(int64_t n, int32_t m, int32_t p_pad, int val_f64);
size_t seg_ws(int64_t n, int32_t m, int32_t p_pad, int32_t K, int val_f64);
int csc_build_launch(const int32_t*, const void*, int, int64_t, int32_t, int32_t, void*, cudaStream_t);
int csc_partials_launch(const void*, int, int64_t, int32_t, int32_t, const int32_t*, int32_t, double*, int64_t*,
                        int64_t*, void*, cudaStream_t);

// skc_kmeans_partials: the exact path (transpose, then sequential per-chain sums)
size_t partials_ws(int64_t n, int32_t m, int32_t p_pad, int32_t K) {
  return ((csc_ws(n, m, p_pad, 1) + 255) & ~(size_t)255) + seg_ws(n, m, p_pad, K, 1);
}
int partials_launch(const int32_t* idx, const void* val, int val_f64, int64_t n, int32_t m, const int32_t* labels,
                    int32_t p_pad, int32_t K, double* sums, int64_t* counts, int64_t* sizes, void* ws,
                    cudaStream_t st) {
  int rc = csc_build_launch(idx, val, val_f64, n, m, p_pad, ws, st);
  if (rc) return rc;
  char* seg = static_cast<char*>(ws) + ((csc_ws(n, m, p_pad, 1) + 255) & ~(size_t)255);
  return csc_partials_launch(ws, val_f64, n, m, p_pad, labels, K, sums, counts, sizes, seg, st);
}

int partials_check(int32_t p_pad, int32_t K) {
  if ((size_t)p_pad * 8 > 96 * 1024) return fail(SKC_EPARAM, "p_pad too large for the K-means update kernel");
  if (K > 256) return fail(SKC_EPARAM, "K > 256 is not supported by the exact K-means update (byte labels)");
  return SKC_OK;
}

// ---------------------------------------------------------------------------------
// Exact partials (cluster.py:189-208). sums[j][k] is np.bincount's sum: sequential fp64 in
// ascending point index over the points labelled k (the stable label sort), at coordinate j.
// The sketch is transposed once (per sketch) into per-coordinate lists, ascending in point
// index: a stable counting sort by coordinate, where a warp takes a range of kCscRange
// points in order. Each iteration one warp walks one coordinate's list 32 entries at a time.
// Lanes with equal labels (match_any) are folded by their lowest lane, in lane order
// (= point order), into warp-private acc[k]. Every (j, k) sum is the reference's chain,
// bit for bit, and the counts come with it.
constexpr int kCscRange = 2048;  // points per warp range, at most
// Points per range: as small as keeps the [p_pad][R] offset table at <= 8M cells (64 MB), between
// 64 and kCscRange. A warp walks its range point by point, so the range count is the transpose's
// parallelism: C2 (200K points, p = 512) gets 3125 ranges of 64 instead of 98 of 2048; C5 (10M
// points, p = 2048) stays at 2048 (its scatter is bound by the scattered 4- and 8-byte stores).
static int csc_range(int64_t n, int32_t p_pad) {
  if (const char* e = getenv("SKC_CSC_RANGE")) return atoi(e) > 0 ? atoi(e) : kCscRange;  // A/B runs
  int64_t r = (n * (int64_t)p_pad + (8 << 20) - 1) / (8 << 20);
  r = (r + 63) / 64 * 64;
  return (int)(r < 64 ? 64 : r > kCscRange ? kCscRange : r);
}

struct CscLayout {
  int64_t R, nnz;
  int S;  // segments per coordinate list in the per-iteration label sort
  size_t off_off, off_rows, off_vals, off_temp, temp_bytes, total;
  size_t off_kbuf, off_sorted, off_seg, off_stemp, stemp_bytes;
};

static CscLayout csc_layout(int64_t n, int32_t m, int32_t p_pad, int val_f64) {
  CscLayout L{};
  const int range = csc_range(n, p_pad);
  L.R = (n + range - 1) / range;
  if (L.R < 1) L.R = 1;
  L.nnz = n * (int64_t)m;
  const int64_t cells = (int64_t)p_pad * L.R + 1;
  cub::DeviceScan::ExclusiveSum(nullptr, L.temp_bytes, (int64_t*)nullptr, (int64_t*)nullptr, (int)cells);
  size_t o = 0;
  auto take = [&](size_t bytes) {
    const size_t r = o;
    o += (bytes + 255) & ~(size_t)255;
    return r;
  };
  L.off_off = take((size_t)cells * 8);
  L.off_rows = take((size_t)(L.nnz > 0 ? L.nnz : 1) * 4);
  L.off_vals = take((size_t)(L.nnz > 0 ? L.nnz : 1) * (val_f64 ? 8 : 4));
  L.off_temp = take(L.temp_bytes);
  L.total = o;
  return L;
}

// per-iteration scratch of the exact partials for K clusters (separate from the transpose)
struct SegLayout {
  int S;
  size_t off_kbuf, off_sorted, off_seg, off_temp, temp_bytes, total;
};
static SegLayout seg_layout(int64_t n, int32_t m, int32_t p_pad, int32_t K, int val_f64) {
  SegLayout L{};
  const int64_t nnz = n * (int64_t)m;
  const int64_t avg = nnz / (p_pad > 0 ? p_pad : 1);
  int64_t S = (avg + 1023) / 1024;
  const int64_t smax = (int64_t)(4 << 20) / ((int64_t)p_pad * K);  // keep p*K*S counters <= 4M
  if (S > smax) S = smax;
  if (S < 1) S = 1;
  L.S = (int)S;
  const int64_t cells = (int64_t)p_pad * K * S + 1;
  cub::DeviceScan::ExclusiveSum(nullptr, L.temp_bytes, (int64_t*)nullptr, (int64_t*)nullptr, (int)cells);
  size_t o = 0;
  auto take = [&](size_t bytes) {
    const size_t r = o;
    o += (bytes + 255) & ~(size_t)255;
    return r;
  };
  L.off_kbuf = take((size_t)(nnz > 0 ? nnz : 1));
  L.off_sorted = take((size_t)(nnz > 0 ? nnz : 1) * (val_f64 ? 8 : 4));
  L.off_seg = take((size_t)cells * 8);
  L.off_temp = take(L.temp_bytes);
  L.total = o;
  return L;
}

// counts of range r at coordinate j -> off[j * R + r] (int64, scanned in place afterwards)
__global__ void km_csc_count_kernel(const int32_t* __restrict__ idx, int64_t n, int m, int32_t p_pad, int64_t R,
                                    int range, int64_t* __restrict__ off) {
  extern __shared__ int ccnt[];  // [warps][p_pad]
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  int* c = ccnt + (size_t)warp * p_pad;
  const int64_t r = blockIdx.x * (int64_t)nw + warp;
  for (int j = lane; j < p_pad; j += 32) c[j] = 0;
  __syncwarp();
  if (r < R) {
    const int64_t i1 = min(n, (r + 1) * (int64_t)range);
    for (int64_t i = r * (int64_t)range; i < i1; ++i)
      for (int t = lane; t < m; t += 32) atomicAdd(&c[__ldg(idx + i * m + t)], 1);
    __syncwarp();
    for (int j = lane; j < p_pad; j += 32) off[(int64_t)j * R + r] = c[j];
  }
}

// stable scatter: range r's entries of coordinate j go to off[j * R + r] ... in point order
template <typename V>
__global__ void km_csc_scatter_kernel(const int32_t* __restrict__ idx, const V* __restrict__ val, int64_t n, int m,
                                      int32_t p_pad, int64_t R, int range, const int64_t* __restrict__ off,
                                      int32_t* __restrict__ rows, V* __restrict__ vals) {
  extern __shared__ int64_t cpos[];  // [warps][p_pad]
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  int64_t* q = cpos + (size_t)warp * p_pad;
  const int64_t r = blockIdx.x * (int64_t)nw + warp;
  if (r >= R) return;
  for (int j = lane; j < p_pad; j += 32) q[j] = off[(int64_t)j * R + r];
  __syncwarp();
  const int64_t i1 = min(n, (r + 1) * (int64_t)range);
  for (int64_t i = r * (int64_t)range; i < i1; ++i) {
    for (int t = lane; t < m; t += 32) {
      const int j = __ldg(idx + i * m + t);
      const int64_t pos = q[j]++;
      rows[pos] = (int32_t)i;
      vals[pos] = __ldg(val + i * m + t);
    }
    __syncwarp();
  }
}

// Per iteration, with each coordinate's list cut into S segments (equal parts per
// coordinate): (A) a warp per segment gathers the labels (kept per entry) and counts them
// per cluster; (B) an exclusive scan over [coordinate][cluster][segment] makes every
// (coordinate, cluster) chain contiguous, in point order; (C) a warp per segment scatters
// its values stably (match_any ranks); (D) a thread per chain adds it sequentially. The
// order is np.bincount's, so sums are bit-identical, and thousands of segments / chains
// keep the GPU busy even at p = 512.
__device__ __forceinline__ void seg_bounds(const int64_t* __restrict__ off, int64_t R, int64_t j, int S, int s,
                                           int64_t* a, int64_t* b) {
  const int64_t e0 = off[j * R], e1 = off[(j + 1) * R];
  const int64_t len = e1 - e0, seg = (len + S - 1) / S;
  *a = min(e1, e0 + seg * s);
  *b = min(e1, e0 + seg * (s + 1));
}

__global__ void km_seg_hist_kernel(const int64_t* __restrict__ off, int64_t R, const int32_t* __restrict__ rows,
                                   const int32_t* __restrict__ labels, int32_t p_pad, int K, int S,
                                   uint8_t* __restrict__ kbuf, int64_t* __restrict__ cnt) {
  extern __shared__ int hcnt[];  // [warps][K]
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  int* h = hcnt + (size_t)warp * K;
  const int64_t w = blockIdx.x * (int64_t)nw + warp;
  if (w >= (int64_t)p_pad * S) return;
  const int64_t j = w / S;
  const int sg = (int)(w - j * S);
  for (int k = lane; k < K; k += 32) h[k] = 0;
  __syncwarp();
  int64_t a, b;
  seg_bounds(off, R, j, S, sg, &a, &b);
  for (int64_t e = a + lane; e < b; e += 32) {
    const int k = __ldg(labels + __ldg(rows + e));
    kbuf[e] = (uint8_t)k;
    atomicAdd(&h[k], 1);
  }
  __syncwarp();
  for (int k = lane; k < K; k += 32) cnt[(j * K + k) * S + sg] = h[k];
}

template <typename V>
__global__ void km_seg_scatter_kernel(const int64_t* __restrict__ off, int64_t R, const V* __restrict__ vals,
                                      const uint8_t* __restrict__ kbuf, int32_t p_pad, int K, int S,
                                      const int64_t* __restrict__ pos0, V* __restrict__ sorted) {
  extern __shared__ int64_t run[];  // [warps][K]
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  int64_t* q = run + (size_t)warp * K;
  const int64_t w = blockIdx.x * (int64_t)nw + warp;
  if (w >= (int64_t)p_pad * S) return;
  const int64_t j = w / S;
  const int sg = (int)(w - j * S);
  for (int k = lane; k < K; k += 32) q[k] = pos0[(j * K + k) * S + sg];
  __syncwarp();
  int64_t a, b;
  seg_bounds(off, R, j, S, sg, &a, &b);
  // 4 steps of 32 elements per round: their label and value loads are all in flight before the
  // (stable, in-order) placements
  constexpr int kR = 4;
  for (int64_t base = a; base < b; base += 32 * kR) {
    int kk[kR];
    V vv[kR];
#pragma unroll
    for (int r = 0; r < kR; ++r) {
      const int64_t e = base + 32 * r + lane;
      kk[r] = e < b ? (int)kbuf[e] : -1;
      vv[r] = e < b ? vals[e] : V(0);
    }
#pragma unroll
    for (int r = 0; r < kR; ++r) {
      const int k = kk[r];
      const uint32_t peers = __match_any_sync(kFM, k);
      if (k >= 0) {
        const int64_t at = q[k] + __popc(peers & lanemask_lt());
        sorted[at] = vv[r];
      }
      __syncwarp();
      if (k >= 0 && (peers & lanemask_lt()) == 0) q[k] += __popc(peers);
      __syncwarp();
    }
  }
}

// A thread adds one chain in order. Loads run one 16-value block ahead of the adds
// (software pipeline). One warp per CTA spreads the few chains of a small problem over
// every SM.
template <typename V>
__global__ void km_chain_sum_kernel(const int64_t* __restrict__ pos0, const V* __restrict__ sorted, int32_t p_pad,
                                    int K, int S, double* __restrict__ sums, int64_t* __restrict__ counts) {
  constexpr int B = 16;
  const int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;  // chain = j * K + k
  if (c >= (int64_t)p_pad * K) return;
  const int64_t a = pos0[c * S], b = pos0[(c + 1) * S];
  double acc = 0.0;
  double cur[B], nxt[B];
#pragma unroll
  for (int u = 0; u < B; ++u) cur[u] = a + u < b ? (double)__ldg(sorted + a + u) : 0.0;
  for (int64_t e = a; e < b; e += B) {
#pragma unroll
    for (int u = 0; u < B; ++u) nxt[u] = e + B + u < b ? (double)__ldg(sorted + e + B + u) : 0.0;
#pragma unroll
    for (int u = 0; u < B; ++u)
      if (e + u < b) acc = dadd(acc, cur[u]);
#pragma unroll
    for (int u = 0; u < B; ++u) cur[u] = nxt[u];
  }
  sums[c] = acc;
  counts[c] = b - a;
}

// Walk path (default where K fits shared memory): one warp walks one coordinate's whole
// list in order, 32 entries per step, with kWalkAhead steps of loads in flight (rows and
// values stream, labels are gathered). Lanes holding equal labels (match_any) add into the
// warp's acc[k] in rank order, one round per rank, so every (j, k) chain is still the
// sequential fp64 sum in ascending point index: no scatter, no scan, no sorted copy.
constexpr int kWalkWarps = 4;
#ifndef SKC_WALK_AHEAD
#define SKC_WALK_AHEAD 4
#endif
constexpr int kWalkAhead = SKC_WALK_AHEAD;  // steps of 32 entries per group; groups are software-pipelined
template <typename V>
__global__ void __launch_bounds__(kWalkWarps * 32) km_walk_kernel(const int64_t* __restrict__ off, int64_t R,
                                                                  const int32_t* __restrict__ rows,
                                                                  const V* __restrict__ vals,
                                                                  const int32_t* __restrict__ labels, int32_t p_pad,
                                                                  int K, double* __restrict__ sums,
                                                                  int64_t* __restrict__ counts) {
  extern __shared__ double wacc[];  // [warps][K] fp64 sums, then [warps][K] int32 counts
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t j = blockIdx.x * (int64_t)kWalkWarps + warp;
  if (j >= p_pad) return;
  double* acc = wacc + (size_t)warp * K;
  int* cnt = reinterpret_cast<int*>(wacc + (size_t)kWalkWarps * K) + (size_t)warp * K;
  for (int k = lane; k < K; k += 32) acc[k] = 0.0, cnt[k] = 0;
  __syncwarp();
  const int64_t a = off[j * R], b = off[(j + 1) * R];
  const uint32_t lt = lanemask_lt();
  constexpr int G = 32 * kWalkAhead;
  // three groups in flight: rows/values of group g+2 load, labels of group g+1 gather, group g adds.
  // The three register sets keep fixed roles per unrolled step: rotating them with register moves
  // would make each move wait for its load and collapse the pipeline.
  struct Set {
    int r[kWalkAhead], k[kWalkAhead];
    V v[kWalkAhead];
  };
  auto load_rv = [&](int64_t base, Set& S) {
#pragma unroll
    for (int s = 0; s < kWalkAhead; ++s) {
      const int64_t e = base + 32 * s + lane;
      S.r[s] = e < b ? __ldg(rows + e) : -1;
      S.v[s] = e < b ? __ldg(vals + e) : V(0);
    }
  };
  auto gather = [&](Set& S) {
#pragma unroll
    for (int s = 0; s < kWalkAhead; ++s) S.k[s] = S.r[s] >= 0 ? __ldg(labels + S.r[s]) : -1;
  };
  auto process = [&](const Set& S) {
    // the group's label matches are independent of the sums: all in flight before the adds
    uint32_t peers[kWalkAhead];
    int last[kWalkAhead];
#pragma unroll
    for (int s = 0; s < kWalkAhead; ++s) peers[s] = __match_any_sync(kFM, S.k[s]);
#pragma unroll
    for (int s = 0; s < kWalkAhead; ++s) last[s] = __reduce_max_sync(kFM, S.k[s] >= 0 ? __popc(peers[s]) : 0);
#pragma unroll
    for (int s = 0; s < kWalkAhead; ++s) {
      // the leader (lowest lane) of each label adds its peers' values in lane (= point) order
      const int k = S.k[s];
      const bool lead = k >= 0 && (peers[s] & lt) == 0;
      double t = lead ? acc[k] : 0.0;
      uint32_t rem = peers[s];
      for (int q = 0; q < last[s]; ++q) {
        const int src = rem ? __ffs(rem) - 1 : lane;
        const double vq = __shfl_sync(kFM, (double)S.v[s], src);
        if (lead && rem) t = dadd(t, vq);
        rem &= rem - 1;
      }
      if (lead) {
        acc[k] = t;
        cnt[k] += __popc(peers[s]);
      }
      __syncwarp();
    }
  };
  auto step = [&](int64_t base, Set& X, Set& Y, Set& Z) {
    gather(Y);                // labels of group g+1
    load_rv(base + 2 * G, Z);  // rows and values of group g+2
    process(X);               // group g
  };
  Set A, B, C;
  load_rv(a, A);
  load_rv(a + G, B);
  gather(A);
  for (int64_t base = a; base < b; base += 3 * G) {
    step(base, A, B, C);
    if (base + G < b) step(base + G, B, C, A);
    if (base + 2 * G < b) step(base + 2 * G, C, A, B);
  }
  __syncwarp();
  for (int k = lane; k < K; k += 32) {
    sums[j * K + k] = acc[k];
    counts[j * K + k] = cnt[k];
  }
}

// Tile path (default for K <= 256): a CTA per coordinate list, kTileE entries at a time. The tile's
// values and labels are staged in shared memory; a stable counting sort by label (per-warp
// counts over contiguous sub-ranges, a scan over (label, warp), match_any ranks inside each
// 32-entry step) makes every label's entries contiguous in point order; then thread k adds
// label k's run to its running fp64 sum, so each (j, k) chain is still the sequential sum in
// ascending point index. Loads are coalesced and the sort runs in shared memory, so the pass
// streams the transposed sketch instead of chasing one warp's latency chain per list.
#ifndef SKC_TILE_E
#define SKC_TILE_E 2048
#endif
#ifndef SKC_TILE_MINB
#define SKC_TILE_MINB 4
#endif
constexpr int kTileE = SKC_TILE_E;
constexpr int kTileWarps = 8;
constexpr int kTileThreads = kTileWarps * 32;
constexpr int kTileMaxK = 256;
static size_t tile_smem(int K) {
  return (size_t)kTileE * 8 * 2 + (size_t)kTileE + (size_t)kTileWarps * K * 4 + (size_t)(K + 1) * 4 * 2 + 64;
}
template <typename V>
__global__ void __launch_bounds__(kTileThreads, SKC_TILE_MINB) km_tile_walk_kernel(
    const int64_t* __restrict__ off, int64_t R, const int32_t* __restrict__ rows, const V* __restrict__ vals,
    const int32_t* __restrict__ labels, int32_t p_pad, int K, double* __restrict__ sums, int64_t* __restrict__ counts) {
  extern __shared__ __align__(16) unsigned char tsm[];
  double* tv = reinterpret_cast<double*>(tsm);  // tile values, list order
  double* ts = tv + kTileE;                     // tile values, sorted by label (stable)
  uint8_t* tl = reinterpret_cast<uint8_t*>(ts + kTileE);
  int* wc = reinterpret_cast<int*>(tl + kTileE);  // [warp][K]: counts, then placement cursors
  int* lb = wc + kTileWarps * K;                  // [K + 1]: label run starts
  int* lt = lb + K + 1;                           // [K]: label run lengths
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int64_t j = blockIdx.x;
  const int64_t a = off[j * R], b = off[(j + 1) * R];
  const uint32_t ltm = lanemask_lt();
  double acc[(kTileMaxK + kTileThreads - 1) / kTileThreads] = {0.0};
  int64_t cntk[(kTileMaxK + kTileThreads - 1) / kTileThreads] = {0};
  for (int64_t t0 = a; t0 < b; t0 += kTileE) {
    const int L = (int)min((int64_t)kTileE, b - t0);
    for (int q = tid; q < kTileWarps * K; q += kTileThreads) wc[q] = 0;
    // stage: values and gathered labels (all loads of a thread in flight together)
#pragma unroll 4
    for (int e = tid; e < L; e += kTileThreads) {
      tv[e] = (double)__ldg(vals + t0 + e);
      tl[e] = (uint8_t)__ldg(labels + __ldg(rows + t0 + e));
    }
    __syncthreads();
    // per-warp label counts over the warp's contiguous sub-range
    const int s0 = (int)((int64_t)L * warp / kTileWarps), s1 = (int)((int64_t)L * (warp + 1) / kTileWarps);
    for (int e = s0 + lane; e < s1; e += 32) atomicAdd(&wc[warp * K + tl[e]], 1);
    __syncthreads();
    // run lengths per label and the exclusive scan over labels (warp 0)
    for (int k = tid; k < K; k += kTileThreads) {
      int t = 0;
      for (int w = 0; w < kTileWarps; ++w) t += wc[w * K + k];
      lt[k] = t;
    }
    __syncthreads();
    if (warp == 0) {
      int run = 0;
      for (int k0 = 0; k0 < K; k0 += 32) {
        const int k = k0 + lane;
        const int c = k < K ? lt[k] : 0;
        int x = c;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const int y = __shfl_up_sync(kFM, x, o);
          if (lane >= o) x += y;
        }
        if (k < K) lb[k] = run + x - c;
        run += __shfl_sync(kFM, x, 31);
      }
      if (lane == 0) lb[K] = run;
    }
    __syncthreads();
    // cursors: label k's entries of warp w start after those of warps < w
    for (int k = tid; k < K; k += kTileThreads) {
      int pos = lb[k];
      for (int w = 0; w < kTileWarps; ++w) {
        const int c = wc[w * K + k];
        wc[w * K + k] = pos;
        pos += c;
      }
    }
    __syncthreads();
    // stable placement: warp sub-ranges in order, lanes in order inside each 32-entry step
    for (int e0 = s0; e0 < s1; e0 += 32) {
      const int e = e0 + lane;
      const int k = e < s1 ? (int)tl[e] : -1;
      const uint32_t peers = __match_any_sync(kFM, k);
      if (k >= 0) ts[wc[warp * K + k] + __popc(peers & ltm)] = tv[e];
      __syncwarp();
      if (k >= 0 && (peers & ltm) == 0) wc[warp * K + k] += __popc(peers);
      __syncwarp();
    }
    __syncthreads();
    // chains: thread k adds label k's run in order (loads ahead of the dependent adds)
#pragma unroll
    for (int u = 0; u < (kTileMaxK + kTileThreads - 1) / kTileThreads; ++u) {
      const int k = tid + u * kTileThreads;
      if (k < K) {
        const int r0 = lb[k], r1 = r0 + lt[k];
        double x = acc[u];
        int e = r0;
        for (; e + 8 <= r1; e += 8) {
          double w[8];
#pragma unroll
          for (int q = 0; q < 8; ++q) w[q] = ts[e + q];
#pragma unroll
          for (int q = 0; q < 8; ++q) x = dadd(x, w[q]);
        }
        for (; e < r1; ++e) x = dadd(x, ts[e]);
        acc[u] = x;
        cntk[u] += r1 - r0;
      }
    }
    __syncthreads();  // the next tile overwrites the staging
  }
#pragma unroll
  for (int u = 0; u < (kTileMaxK + kTileThreads - 1) / kTileThreads; ++u) {
    const int k = tid + u * kTileThreads;
    if (k < K) {
      sums[j * K + k] = acc[u];
      counts[j * K + k] = cntk[u];
    }
  }
}

static size_t walk_smem(int K) { return (size_t)kWalkWarps * K * 12; }
// The walk has one warp per coordinate list: it needs enough lists to fill the GPU (C5, p = 2048:
// 8.7 vs 24 ms per iteration); with few lists the segment path's thousands of segments win
// (C2, p = 512: 2.17 vs 2.44 ms per 6-iteration run).
// Path choice (measured): long lists (p_pad >= 1024: C5's 2048 lists of ~500K entries) take the walk
// (8.7 ms per C5 iteration; tile 12.5, segments 24); short ones (C2: 512 lists of ~10K) the
// tile path (1.94 ms per C2 run; segments 2.14, walk 2.40); K > 256 the segment path.
static bool use_walk(int32_t p_pad, int K) {
  if (const char* e = getenv("SKC_PARTIALS")) return e[0] == 'w';  // A/B: SKC_PARTIALS=seg|walk|tile
  return p_pad >= 1024 && walk_smem(K) <= 96 * 1024;
}
static bool use_tile(int32_t p_pad, int K) {
  if (const char* e = getenv("SKC_PARTIALS")) return e[0] == 't' && K <= kTileMaxK;
  return !use_walk(p_pad, K) && K <= kTileMaxK;
}

// cluster sizes: bincount(labels), exact
__global__ void km_sizes_kernel(const int32_t* __restrict__ labels, int64_t n, int K, int64_t* __restrict__ sizes) {
  extern __shared__ int hs[];
  for (int k = threadIdx.x; k < K; k += blockDim.x) hs[k] = 0;
  __syncthreads();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    atomicAdd(&hs[labels[i]], 1);
  __syncthreads();
  for (int k = threadIdx.x; k < K; k += blockDim.x)
    if (hs[k]) atomicAdd(reinterpret_cast<unsigned long long*>(sizes) + k, (unsigned long long)hs[k]);
}

size_t csc_ws(int64_t n, int32_t m, int32_t p_pad, int val_f64) { return csc_layout(n, m, p_pad, val_f64).total; }

static int csc_warps_for(int32_t p_pad, size_t bytes_per) {
  int w = 4;
  while (w > 1 && (size_t)w * p_pad * bytes_per > 96 * 1024) w >>= 1;
  return w;
}

int csc_build_launch(const int32_t* idx, const void* val, int val_f64, int64_t n, int32_t m, int32_t p_pad, void* ws,
                     cudaStream_t st) {
  const CscLayout L = csc_layout(n, m, p_pad, val_f64);
  char* w = reinterpret_cast<char*>(ws);
  int64_t* off = reinterpret_cast<int64_t*>(w + L.off_off);
  const int64_t cells = (int64_t)p_pad * L.R + 1;
  cudaMemsetAsync(off, 0, (size_t)cells * 8, st);
  int rc;
  if (n > 0) {
    const int wc = csc_warps_for(p_pad, 4);
    const size_t smc = (size_t)wc * p_pad * 4;
    cudaFuncSetAttribute(km_csc_count_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smc);
    km_csc_count_kernel<<<(unsigned)((L.R + wc - 1) / wc), wc * 32, smc, st>>>(idx, n, m, p_pad, L.R,
                                                                                csc_range(n, p_pad), off);
    if ((rc = check_launch("km_csc_count_kernel"))) return rc;
  }
  size_t tb = L.temp_bytes;
  if (cub::DeviceScan::ExclusiveSum(w + L.off_temp, tb, off, off, (int)cells, st) != cudaSuccess)
    return check_launch("csc offsets scan");
  if (n > 0) {
    const int ws_ = csc_warps_for(p_pad, 8);
    const size_t sms = (size_t)ws_ * p_pad * 8;
    const unsigned grid = (unsigned)((L.R + ws_ - 1) / ws_);
    if (val_f64) {
      cudaFuncSetAttribute(km_csc_scatter_kernel<double>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sms);
      km_csc_scatter_kernel<double><<<grid, ws_ * 32, sms, st>>>(idx, (const double*)val, n, m, p_pad, L.R,
                                                                  csc_range(n, p_pad), off,
                                                                  reinterpret_cast<int32_t*>(w + L.off_rows),
                                                                  reinterpret_cast<double*>(w + L.off_vals));
    } else {
      cudaFuncSetAttribute(km_csc_scatter_kernel<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sms);
      km_csc_scatter_kernel<float><<<grid, ws_ * 32, sms, st>>>(idx, (const float*)val, n, m, p_pad, L.R,
                                                                csc_range(n, p_pad), off,
                                                                reinterpret_cast<int32_t*>(w + L.off_rows),
                                                                reinterpret_cast<float*>(w + L.off_vals));
    }
    if ((rc = check_launch("km_csc_scatter_kernel"))) return rc;
  }
  return SKC_OK;
}

static int sizes_launch(const int32_t* labels, int64_t n, int32_t K, int64_t* sizes, cudaStream_t st) {
  if (sizes == nullptr) return SKC_OK;  // the caller derives them from the counts (sum_j counts[j][k] = m n_k)
  cudaMemsetAsync(sizes, 0, (size_t)K * 8, st);
  if (n > 0) {
    int64_t blocks = (n + 255) / 256;
    if (blocks > 4LL * sm_count()) blocks = 4LL * sm_count();
    cudaFuncSetAttribute(km_sizes_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(K * 4));
    km_sizes_kernel<<<(unsigned)blocks, 256, (size_t)K * 4, st>>>(labels, n, K, sizes);
    return check_launch("km_sizes_kernel");
  }
  return SKC_OK;
}

size_t seg_ws(int64_t n, int32_t m, int32_t p_pad, int32_t K, int val_f64) {
  if (use_walk(p_pad, K) || use_tile(p_pad, K)) return 256;  // the walk and tile paths need no per-iteration scratch
  return seg_layout(n, m, p_pad, K, val_f64).total;
}

int csc_partials_launch(const void* ws, int val_f64, int64_t n, int32_t m, int32_t p_pad, const int32_t* labels,
                        int32_t K, double* sums, int64_t* counts, int64_t* sizes, void* seg_ws_ptr, cudaStream_t st) {
  const CscLayout L = csc_layout(n, m, p_pad, val_f64);
  const SegLayout G = seg_layout(n, m, p_pad, K, val_f64);
  const char* w = reinterpret_cast<const char*>(ws);
  char* g = reinterpret_cast<char*>(seg_ws_ptr);
  const int64_t* off = reinterpret_cast<const int64_t*>(w + L.off_off);
  const int32_t* rows = reinterpret_cast<const int32_t*>(w + L.off_rows);
  int rc;
  if (use_tile(p_pad, K)) {
    const size_t tsm = tile_smem(K);
    if (val_f64) {
      cudaFuncSetAttribute(km_tile_walk_kernel<double>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)tsm);
      km_tile_walk_kernel<double><<<(unsigned)p_pad, kTileThreads, tsm, st>>>(
          off, L.R, rows, reinterpret_cast<const double*>(w + L.off_vals), labels, p_pad, K, sums, counts);
    } else {
      cudaFuncSetAttribute(km_tile_walk_kernel<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)tsm);
      km_tile_walk_kernel<float><<<(unsigned)p_pad, kTileThreads, tsm, st>>>(
          off, L.R, rows, reinterpret_cast<const float*>(w + L.off_vals), labels, p_pad, K, sums, counts);
    }
    if ((rc = check_launch("km_tile_walk_kernel"))) return rc;
    return sizes_launch(labels, n, K, sizes, st);
  }
  if (use_walk(p_pad, K)) {
    const unsigned wgrid = (unsigned)((p_pad + kWalkWarps - 1) / kWalkWarps);
    const size_t wsm = walk_smem(K);
    if (val_f64) {
      cudaFuncSetAttribute(km_walk_kernel<double>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)wsm);
      km_walk_kernel<double><<<wgrid, kWalkWarps * 32, wsm, st>>>(
          off, L.R, rows, reinterpret_cast<const double*>(w + L.off_vals), labels, p_pad, K, sums, counts);
    } else {
      cudaFuncSetAttribute(km_walk_kernel<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)wsm);
      km_walk_kernel<float><<<wgrid, kWalkWarps * 32, wsm, st>>>(
          off, L.R, rows, reinterpret_cast<const float*>(w + L.off_vals), labels, p_pad, K, sums, counts);
    }
    if ((rc = check_launch("km_walk_kernel"))) return rc;
    return sizes_launch(labels, n, K, sizes, st);
  }
  uint8_t* kbuf = reinterpret_cast<uint8_t*>(g + G.off_kbuf);
  int64_t* seg = reinterpret_cast<int64_t*>(g + G.off_seg);
  const int S = G.S;
  const int64_t items = (int64_t)p_pad * S;
  const int64_t cells = (int64_t)p_pad * K * S + 1;
  constexpr int kW = 4;  // warps per CTA (one segment each)
  const unsigned grid = (unsigned)((items + kW - 1) / kW);
  cudaMemsetAsync(seg + cells - 1, 0, 8, st);
  cudaFuncSetAttribute(km_seg_hist_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(kW * K * 4));
  km_seg_hist_kernel<<<grid, kW * 32, (size_t)kW * K * 4, st>>>(off, L.R, rows, labels, p_pad, K, S, kbuf, seg);
  if ((rc = check_launch("km_seg_hist_kernel"))) return rc;
  size_t tb = G.temp_bytes;
  if (cub::DeviceScan::ExclusiveSum(g + G.off_temp, tb, seg, seg, (int)cells, st) != cudaSuccess)
    return check_launch("segment offsets scan");
  const size_t ssm = (size_t)kW * K * 8;
  const unsigned cgrid = (unsigned)(((int64_t)p_pad * K + 31) / 32);  // one warp (32 chains) per CTA
  if (val_f64) {
    const double* vals = reinterpret_cast<const double*>(w + L.off_vals);
    double* sorted = reinterpret_cast<double*>(g + G.off_sorted);
    cudaFuncSetAttribute(km_seg_scatter_kernel<double>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ssm);
    km_seg_scatter_kernel<double><<<grid, kW * 32, ssm, st>>>(off, L.R, vals, kbuf, p_pad, K, S, seg, sorted);
    if ((rc = check_launch("km_seg_scatter_kernel"))) return rc;
    km_chain_sum_kernel<double><<<cgrid, 32, 0, st>>>(seg, sorted, p_pad, K, S, sums, counts);
  } else {
    const float* vals = reinterpret_cast<const float*>(w + L.off_vals);
    float* sorted = reinterpret_cast<float*>(g + G.off_sorted);
    cudaFuncSetAttribute(km_seg_scatter_kernel<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ssm);
    km_seg_scatter_kernel<float><<<grid, kW * 32, ssm, st>>>(off, L.R, vals, kbuf, p_pad, K, S, seg, sorted);
    if ((rc = check_launch("km_seg_scatter_kernel"))) return rc;
    km_chain_sum_kernel<float><<<cgrid, 32, 0, st>>>(seg, sorted, p_pad, K, S, sums, counts);
  }
  if ((rc = check_launch("km_chain_sum_kernel"))) return rc;
  return sizes_launch(labels, n, K, sizes, st);
}

// ---------------------------------------------------------------------------------
__global__ void km_centers_kernel(const double* __restrict__ sums, const int64_t* __restrict__ counts,
                                  const int64_t* __restrict__ sizes, const double* __restrict__ mu_prev, int32_t p_pad,
                                  int K, double* __restrict__ mu, int32_t* __restrict__ empty) {
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e < K) empty[e] = sizes[e] == 0;
  if (e >= (int64_t)p_pad * K) return;
  const int k = (int)(e % K);
  const int64_t c = counts[e];
  mu[e] = (sizes[k] == 0 || c == 0) ? mu_prev[e] : __ddiv_rn(sums[e], (double)c);
}

int centers_launch(const double* sums, const int64_t* counts, const int64_t* sizes, const double* mu_prev,
                   int32_t p_pad, int32_t K, double* mu, int32_t* empty, cudaStream_t st) {
  const int64_t tot = (int64_t)p_pad * K;
  const int64_t work = tot > K ? tot : K;
  km_centers_kernel<<<(unsigned)((work + 255) / 256), 256, 0, st>>>(sums, counts, sizes, mu_prev, p_pad, K, mu,
                                                                     empty);
  return check_launch("km_centers_kernel");
}

template <typename V>
__global__ void km_reseed_kernel(const int32_t* __restrict__ idx_c, const void* __restrict__ val_c, int m,
                                 const int32_t* __restrict__ empty, int32_t p_pad, int K, double* __restrict__ mu) {
  const int k = blockIdx.x;
  if (!empty[k]) return;
  for (int j = threadIdx.x; j < p_pad; j += blockDim.x) mu[(int64_t)j * K + k] = 0.0;
  __syncthreads();
  for (int t = threadIdx.x; t < m; t += blockDim.x) mu[(int64_t)idx_c[t] * K + k] = ldd<V>(val_c, t);
}

// the same with the farthest point's row read from device memory (*row, clamped at 0),
// so the Lloyd loop can enqueue the reseed before the host has read the argmax
template <typename V>
__global__ void km_reseed_at_kernel(const int32_t* __restrict__ idx, const void* __restrict__ val, int m,
                                    const long long* __restrict__ row, const int32_t* __restrict__ empty,
                                    int32_t p_pad, int K, double* __restrict__ mu) {
  const int k = blockIdx.x;
  if (!empty[k]) return;
  const long long r = *row > 0 ? *row : 0;
  for (int j = threadIdx.x; j < p_pad; j += blockDim.x) mu[(int64_t)j * K + k] = 0.0;
  __syncthreads();
  for (int t = threadIdx.x; t < m; t += blockDim.x) mu[(int64_t)idx[r * m + t] * K + k] = ldd<V>(val, r * m + t);
}

int reseed_at_launch(const int32_t* idx, const void* val, int val_f64, int32_t m, const long long* row,
                     const int32_t* empty, int32_t p_pad, int32_t K, double* mu, cudaStream_t st) {
  if (val_f64) km_reseed_at_kernel<double><<<K, 256, 0, st>>>(idx, val, m, row, empty, p_pad, K, mu);
  else km_reseed_at_kernel<float><<<K, 256, 0, st>>>(idx, val, m, row, empty, p_pad, K, mu);
  return check_launch("km_reseed_at_kernel");
}

int reseed_launch(const int32_t* idx_c, const void* val_c, int val_f64, int32_t m, const int32_t* empty,
                  int32_t p_pad, int32_t K, double* mu, cudaStream_t st) {
  if (val_f64) km_reseed_kernel<double><<<K, 256, 0, st>>>(idx_c, val_c, m, empty, p_pad, K, mu);
  else km_reseed_kernel<float><<<K, 256, 0, st>>>(idx_c, val_c, m, empty, p_pad, K, mu);
  return check_launch("km_reseed_kernel");
}

template <typename V>
__global__ void km_init_kernel(const int32_t* __restrict__ idx, const void* __restrict__ val, int m,
                               const int64_t* __restrict__ chosen, int K, int32_t p_pad, double* __restrict__ mu) {
  const int k = blockIdx.x;
  for (int j = threadIdx.x; j < p_pad; j += blockDim.x) mu[(int64_t)j * K + k] = 0.0;
  __syncthreads();
  const int64_t c = chosen[k];
  for (int t = threadIdx.x; t < m; t += blockDim.x) mu[(int64_t)idx[c * m + t] * K + k] = ldd<V>(val, c * m + t);
}

int init_launch(const int32_t* idx, const void* val, int val_f64, int32_t m, const int64_t* chosen, int32_t K,
                int32_t p_pad, double* mu, cudaStream_t st) {
  if (val_f64) km_init_kernel<double><<<K, 256, 0, st>>>(idx, val, m, chosen, K, p_pad, mu);
  else km_init_kernel<float><<<K, 256, 0, st>>>(idx, val, m, chosen, K, p_pad, mu);
  return check_launch("km_init_kernel");
}

// ---------------------------------------------------------------------------------
// K-means++ support: row norms and D^2 to one point (cluster.py:148, 169-173)
template <typename V>
__global__ void row_sqnorm_kernel(const void* __restrict__ val, int64_t n, int m, double* __restrict__ out) {
  extern __shared__ double sq_all[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double* sq = sq_all + (size_t)warp * m;
  const int64_t gw = (int64_t)blockIdx.x * (blockDim.x >> 5) + warp, nw = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t i = gw; i < n; i += nw) {
    for (int t = lane; t < m; t += 32) {
      const double v = ldd<V>(val, i * m + t);
      sq[t] = dmul(v, v);
    }
    __syncwarp();
    if (lane == 0) out[i] = pw_rec(sq, m);
    __syncwarp();
  }
}

template <typename V>
__global__ void dense_point_kernel(const int32_t* __restrict__ idx, const void* __restrict__ val, int m, int32_t p_pad,
                                   int64_t c, double* __restrict__ dense) {
  for (int j = threadIdx.x; j < p_pad; j += blockDim.x) dense[j] = 0.0;
  __syncthreads();
  for (int t = threadIdx.x; t < m; t += blockDim.x) dense[idx[c * m + t]] = ldd<V>(val, c * m + t);
}

template <typename V>
__global__ void d2_point_kernel(const int32_t* __restrict__ idx, const void* __restrict__ val, int64_t n, int m,
                                const double* __restrict__ csq, const double* __restrict__ colsq,
                                const double* __restrict__ dense, double scale, double* __restrict__ out) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  double cross = 0.0;
  for (int t = 0; t < m; ++t) cross = dadd(cross, dmul(ldd<V>(val, i * m + t), __ldg(dense + __ldg(idx + i * m + t))));
  const double d2 = dsub(dadd(colsq[i], *csq), dmul(2.0, cross));
  out[i] = dmul(scale, d2 > 0.0 ? d2 : 0.0);
}

int row_sqnorms_launch(const void* val, int val_f64, int64_t n, int32_t m, double* out, cudaStream_t st) {
  if (n == 0) return SKC_OK;
  const size_t smem = (size_t)8 * m * sizeof(double);
  if (smem > 200 * 1024) return fail(SKC_EPARAM, "m too large for the row-norm kernel");
  int64_t blocks = (n + 7) / 8;
  if (blocks > 8 * (int64_t)sm_count()) blocks = 8 * (int64_t)sm_count();
  auto kern = val_f64 ? row_sqnorm_kernel<double> : row_sqnorm_kernel<float>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  kern<<<(unsigned)blocks, 256, smem, st>>>(val, n, m, out);
  return check_launch("row_sqnorm_kernel");
}

int d2_dense_launch(const int32_t*, const void*, int, int64_t, int32_t, int32_t, const double*, const double*,
                    const double*, double*, cudaStream_t);

int d2_point_launch(const int32_t* idx, const void* val, int val_f64, int64_t n, int32_t m, int32_t p_pad, int64_t c,
                    const double* colsq, double* dense, double* out, cudaStream_t st) {
  const double scale = (double)p_pad / (double)m;
  if (val_f64) dense_point_kernel<double><<<1, 256, 0, st>>>(idx, val, m, p_pad, c, dense);
  else dense_point_kernel<float><<<1, 256, 0, st>>>(idx, val, m, p_pad, c, dense);
  int rc = check_launch("dense_point_kernel");
  if (rc) return rc;
  return d2_dense_launch(idx, val, val_f64, n, m, p_pad, dense, colsq + c, colsq, out, st);
}

// d2 of every point to a point given as its densified row and squared norm (a point of another
// shard: sharded K-means++ seeding, cluster.py:169-173 with W[:, c] supplied).
int d2_dense_launch(const int32_t* idx, const void* val, int val_f64, int64_t n, int32_t m, int32_t p_pad,
                    const double* dense, const double* csq, const double* colsq, double* out, cudaStream_t st) {
  if (n == 0) return SKC_OK;
  const double scale = (double)p_pad / (double)m;
  const unsigned blocks = (unsigned)((n + 255) / 256);
  if (val_f64) d2_point_kernel<double><<<blocks, 256, 0, st>>>(idx, val, n, m, csq, colsq, dense, scale, out);
  else d2_point_kernel<float><<<blocks, 256, 0, st>>>(idx, val, n, m, csq, colsq, dense, scale, out);
  return check_launch("d2_point_kernel");
}

}  // namespace skc
