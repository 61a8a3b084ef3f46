// K5/K6: sparsified K-means on the sketch (cluster.py:133-243).
//  assign   exact fp64 emulation of [values | ones] @ [-2 mu ; mu*mu] + colsq
//           (cluster.py:181-187), so labels and d2min are bit-exact
//  pairwise numpy pairwise summation of d2min (the objective, cluster.py:233)
//  partials stable counting sort by label, then fixed-size chunks summed by
//           warp-private shared-memory vectors; deterministic (cluster.py:189-208)
//  centers  divide / keep-previous / empty flags (cluster.py:196-210)
//  reseed   cluster.py:212-215;  init  cluster.py:175-179
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

constexpr int kPwDeep = 14;  // subtrees at depth 14: one thread each, 64 blocks

__global__ void __launch_bounds__(256) pairwise_leaves_kernel(const double* __restrict__ x, int64_t n,
                                                              double* __restrict__ res) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;  // path of depth kPwDeep
  int64_t off = 0, len = n;
  bool active = true;
  for (int d = 0; d < kPwDeep; ++d) {
    const int bit = (t >> (kPwDeep - 1 - d)) & 1;
    if (len <= 128) {  // leaf above the split depth: owned by the all-zero suffix path
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
  res[t] = active ? pw_rec(x + off, len) : 0.0;
}

__global__ void __launch_bounds__(1024) pairwise_combine_kernel(double* __restrict__ res, int64_t n,
                                                                double* __restrict__ out) {
  for (int d = kPwDeep - 1; d >= 0; --d) {
    for (int t = threadIdx.x; t < (1 << d); t += blockDim.x) {
      bool leaf_above;
      int64_t L = n;
      leaf_above = false;
      for (int k = 0; k < d; ++k) {
        if (L <= 128) {
          leaf_above = true;
          break;
        }
        int64_t n2 = L / 2;
        n2 -= n2 % 8;
        L = ((t >> (d - 1 - k)) & 1) ? L - n2 : n2;
      }
      if (!leaf_above && L > 128) {
        const int sh = kPwDeep - d;
        res[(size_t)t << sh] = dadd(res[(size_t)(2 * t) << (sh - 1)], res[(size_t)(2 * t + 1) << (sh - 1)]);
      }
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) out[0] = res[0];
}

size_t pairwise_ws() { return ((size_t)1 << kPwDeep) * sizeof(double); }

int pairwise_launch(const double* x, int64_t n, double* out, void* ws, cudaStream_t st) {
  double* res = reinterpret_cast<double*>(ws);
  pairwise_leaves_kernel<<<(1 << kPwDeep) / 256, 256, 0, st>>>(x, n, res);
  int rc = check_launch("pairwise_leaves_kernel");
  if (rc) return rc;
  pairwise_combine_kernel<<<1, 1024, 0, st>>>(res, n, out);
  return check_launch("pairwise_combine_kernel");
}

// ---------------------------------------------------------------------------------
// assign
constexpr int kAsgWarps = 8;

// packed per-(j,k) table: {-2 mu, mu*mu} (np.vstack([-2.0 * mu, mu * mu]), cluster.py:182)
__global__ void km_tables2_kernel(const double* __restrict__ mu, int64_t total, double2* __restrict__ tab) {
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= total) return;
  const double v = mu[e];
  tab[e] = make_double2(dmul(-2.0, v), dmul(v, v));
}

// A warp holds G = 32/KP points; lane = g*KP + k. For K > KP the lane loops over k += KP.
// colsq: numpy pairwise order on 8 lanes of the group (m <= 128), else pw_rec on one lane.
// d2[k] = sum_t v_t*(-2 mu[j_t,k]) then + sum_t mu[j_t,k]^2 (csr_matvecs axpy order) + colsq.
// SMEM_TAB: the packed (p, K) table is staged in shared memory (small p*K, e.g. C2).
template <typename V, int KP, bool SMEM_TAB>
__global__ void __launch_bounds__(kAsgWarps * 32, 4)
    km_assign_kernel(const int32_t* __restrict__ idx, const void* __restrict__ val, int64_t n, int m,
                     const double2* __restrict__ gtab, int K, int p_pad, const int32_t* __restrict__ prev,
                     int32_t* __restrict__ labels, double* __restrict__ d2min, int64_t* __restrict__ blk_changed,
                     double* __restrict__ blk_max, int64_t* __restrict__ blk_arg) {
  constexpr int G = 32 / KP;
  extern __shared__ __align__(16) unsigned char sm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane / KP, k0 = lane % KP;
  // layout: [table (SMEM_TAB)] [per warp: sidx G*m int | sval G*m double | msq 32*m double]
  size_t off = 0;
  const double2* tab = gtab;
  if constexpr (SMEM_TAB) {
    double2* st = reinterpret_cast<double2*>(sm);
    for (int e = threadIdx.x; e < p_pad * K; e += blockDim.x) st[e] = gtab[e];
    tab = st;
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
        const double2* tk = tab + k;
        double acc = 0.0;
        int t = 0;
        const double* tkx = reinterpret_cast<const double*>(tk);
        for (; t + 4 <= m; t += 4) {
          const double a0 = tkx[2 * si[t]], a1 = tkx[2 * si[t + 1]], a2 = tkx[2 * si[t + 2]], a3 = tkx[2 * si[t + 3]];
          acc = dadd(acc, dmul(sv[t], a0));
          acc = dadd(acc, dmul(sv[t + 1], a1));
          acc = dadd(acc, dmul(sv[t + 2], a2));
          acc = dadd(acc, dmul(sv[t + 3], a3));
        }
        for (; t < m; ++t) acc = dadd(acc, dmul(sv[t], tkx[2 * si[t]]));
        for (t = 0; t + 4 <= m; t += 4) {
          const double b0 = tkx[2 * si[t] + 1], b1 = tkx[2 * si[t + 1] + 1], b2 = tkx[2 * si[t + 2] + 1],
                       b3 = tkx[2 * si[t + 3] + 1];
          acc = dadd(acc, b0);
          acc = dadd(acc, b1);
          acc = dadd(acc, b2);
          acc = dadd(acc, b3);
        }
        for (; t < m; ++t) acc = dadd(acc, tkx[2 * si[t] + 1]);
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

static int assign_grid(int64_t n) {
  int64_t g = (n + kAsgWarps - 1) / kAsgWarps;
  const int64_t cap = 4 * (int64_t)sm_count();
  if (g > cap) g = cap;
  return (int)(g < 1 ? 1 : g);
}

size_t assign_ws(int64_t n, int32_t p_pad, int32_t K) {
  return (size_t)2 * p_pad * K * sizeof(double) + (size_t)assign_grid(n) * 24 + 64;
}

template <typename V, int KP>
static void launch_assign_kp(int G, const int32_t* idx, const void* val, int64_t n, int32_t m, const double2* tab,
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
    k<<<G, warps * 32, smem, st>>>(idx, val, n, m, tab, K, p_pad, prev, labels, d2min, bch, bmx, barg);
  } else {
    auto k = km_assign_kernel<V, KP, false>;
    const size_t smem = per_warp * warps;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k<<<G, warps * 32, smem, st>>>(idx, val, n, m, tab, K, p_pad, prev, labels, d2min, bch, bmx, barg);
  }
}

int assign_launch(const int32_t* idx, const void* val, int val_f64, int64_t n, int32_t m, const double* mu,
                  int32_t p_pad, int32_t K, const int32_t* prev, int32_t* labels, double* d2min, int64_t* out,
                  double* d2max, void* ws, cudaStream_t st) {
  double2* tab = reinterpret_cast<double2*>(ws);
  const int G = assign_grid(n);
  int64_t* bch = reinterpret_cast<int64_t*>(tab + (size_t)p_pad * K);
  double* bmx = reinterpret_cast<double*>(bch + G);
  int64_t* barg = reinterpret_cast<int64_t*>(bmx + G);
  const int64_t total = (int64_t)p_pad * K;
  km_tables2_kernel<<<(unsigned)((total + 255) / 256), 256, 0, st>>>(mu, total, tab);
  int rc = check_launch("km_tables2_kernel");
  if (rc) return rc;
  if (n > 0) {
    if (val_f64) {
      if (K <= 8) launch_assign_kp<double, 8>(G, idx, val, n, m, tab, K, p_pad, prev, labels, d2min, bch, bmx, barg, st);
      else if (K <= 16) launch_assign_kp<double, 16>(G, idx, val, n, m, tab, K, p_pad, prev, labels, d2min, bch, bmx, barg, st);
      else launch_assign_kp<double, 32>(G, idx, val, n, m, tab, K, p_pad, prev, labels, d2min, bch, bmx, barg, st);
    } else {
      if (K <= 8) launch_assign_kp<float, 8>(G, idx, val, n, m, tab, K, p_pad, prev, labels, d2min, bch, bmx, barg, st);
      else if (K <= 16) launch_assign_kp<float, 16>(G, idx, val, n, m, tab, K, p_pad, prev, labels, d2min, bch, bmx, barg, st);
      else launch_assign_kp<float, 32>(G, idx, val, n, m, tab, K, p_pad, prev, labels, d2min, bch, bmx, barg, st);
    }
    rc = check_launch("km_assign_kernel");
    if (rc) return rc;
  }
  km_assign_reduce_kernel<<<1, 1024, 0, st>>>(bch, bmx, barg, n > 0 ? G : 0, out, d2max);
  return check_launch("km_assign_reduce_kernel");
}

// ---------------------------------------------------------------------------------
// partials: stable counting sort by label + chunked warp-private accumulation
constexpr int kSortBlock = 1024;  // points per histogram/scatter block
constexpr int kPartWarps = 8;

struct PartLayout {
  int64_t nblk, nchunk_max, ch;
  size_t off_hist, off_base, off_perm, off_sizes, off_coff, off_cfirst, off_chunks, off_psum, off_pcnt, total;
};

static PartLayout part_layout(int64_t n, int32_t p_pad, int32_t K) {
  PartLayout L{};
  L.nblk = (n + kSortBlock - 1) / kSortBlock;
  if (L.nblk < 1) L.nblk = 1;
  int64_t ch = n / (2 * (int64_t)sm_count());
  const int64_t minch = (int64_t)32 * p_pad / 8;  // per-chunk setup ~ W*p words vs ch*m/32 work
  if (ch < minch) ch = minch;
  if (ch < 512) ch = 512;
  if (ch > 32768) ch = 32768;
  L.ch = ch;
  L.nchunk_max = (n + ch - 1) / ch + K;
  size_t o = 0;
  auto take = [&](size_t bytes) {
    size_t r = o;
    o += (bytes + 255) & ~(size_t)255;
    return r;
  };
  L.off_hist = take((size_t)L.nblk * K * 4);
  L.off_base = take((size_t)L.nblk * K * 8);
  L.off_perm = take((size_t)(n > 0 ? n : 1) * 4);
  L.off_sizes = take((size_t)K * 8);
  L.off_coff = take((size_t)(K + 1) * 8);
  L.off_cfirst = take((size_t)(K + 1) * 8);
  L.off_chunks = take((size_t)L.nchunk_max * 16);
  L.off_psum = take((size_t)L.nchunk_max * p_pad * 8);
  L.off_pcnt = take((size_t)L.nchunk_max * p_pad * 4);
  L.total = o;
  return L;
}

size_t partials_ws(int64_t n, int32_t p_pad, int32_t K) { return part_layout(n, p_pad, K).total; }

// hist[k][b] = # points of block b with label k
__global__ void km_hist_kernel(const int32_t* __restrict__ labels, int64_t n, int K, int64_t nblk,
                               int32_t* __restrict__ hist) {
  extern __shared__ int h[];
  for (int k = threadIdx.x; k < K; k += blockDim.x) h[k] = 0;
  __syncthreads();
  const int64_t b = blockIdx.x;
  for (int64_t i = b * kSortBlock + threadIdx.x; i < min(n, (b + 1) * (int64_t)kSortBlock); i += blockDim.x)
    atomicAdd(&h[labels[i]], 1);
  __syncthreads();
  for (int k = threadIdx.x; k < K; k += blockDim.x) hist[(int64_t)k * nblk + b] = h[k];
}

// per k: exclusive scan over blocks -> base[k][b]; sizes[k]
__global__ void km_scan_kernel(const int32_t* __restrict__ hist, int64_t nblk, int64_t* __restrict__ base,
                               int64_t* __restrict__ sizes) {
  const int k = blockIdx.x;
  __shared__ int64_t carry;
  __shared__ int64_t wsum[32];
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarp = blockDim.x >> 5;
  for (int64_t b0 = 0; b0 < nblk; b0 += blockDim.x) {
    const int64_t b = b0 + threadIdx.x;
    int64_t v = b < nblk ? hist[(int64_t)k * nblk + b] : 0;
    int64_t x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int64_t y = __shfl_up_sync(kFM, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) wsum[warp] = x;
    __syncthreads();
    int64_t before = carry;
    for (int w = 0; w < warp; ++w) before += wsum[w];
    if (b < nblk) base[(int64_t)k * nblk + b] = before + x - v;
    __syncthreads();
    if (threadIdx.x == 0) {
      int64_t s = 0;
      for (int w = 0; w < nwarp; ++w) s += wsum[w];
      carry += s;
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) sizes[k] = carry;
}

// cluster offsets, first chunk of each cluster, and the chunk table (cluster-major, fixed
// chunk length). One block: a warp-cooperative scan over K, then every thread fills the
// entries of its own clusters.
__global__ void km_offsets_kernel(const int64_t* __restrict__ sizes, int K, int64_t ch, int64_t nchunk_max,
                                  int64_t* __restrict__ coff, int64_t* __restrict__ cfirst,
                                  int64_t* __restrict__ chunks) {
  __shared__ int64_t carry_s, carry_c;
  if (threadIdx.x == 0) {
    carry_s = 0;
    carry_c = 0;
  }
  __syncthreads();
  const int lane = threadIdx.x & 31;
  if (threadIdx.x < 32) {
    for (int k0 = 0; k0 < K; k0 += 32) {
      const int k = k0 + lane;
      const int64_t sz = k < K ? sizes[k] : 0;
      const int64_t nc = (sz + ch - 1) / ch;
      int64_t is = sz, ic = nc;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int64_t ys = __shfl_up_sync(kFM, is, o), yc = __shfl_up_sync(kFM, ic, o);
        if (lane >= o) {
          is += ys;
          ic += yc;
        }
      }
      if (k < K) {
        coff[k] = carry_s + is - sz;
        cfirst[k] = carry_c + ic - nc;
      }
      __syncwarp();
      if (lane == 31) {
        carry_s += is;
        carry_c += ic;
      }
      __syncwarp();
    }
    if (lane == 0) {
      coff[K] = carry_s;
      cfirst[K] = carry_c;
    }
  }
  __syncthreads();
  for (int k = threadIdx.x; k < K; k += blockDim.x) {
    int64_t c = cfirst[k];
    for (int64_t s0 = 0; s0 < sizes[k]; s0 += ch, ++c) {
      chunks[2 * c] = coff[k] + s0;                                             // start in perm
      chunks[2 * c + 1] = ((int64_t)k << 32) | (uint32_t)min(ch, sizes[k] - s0);  // k | len
    }
  }
  for (int64_t c = cfirst[K] + threadIdx.x; c < nchunk_max; c += blockDim.x) {
    chunks[2 * c] = 0;
    chunks[2 * c + 1] = -1;
  }
}

// stable scatter: one warp per block walks its points in order
__global__ void km_scatter_kernel(const int32_t* __restrict__ labels, int64_t n, int K, int64_t nblk,
                                  const int64_t* __restrict__ base, const int64_t* __restrict__ coff,
                                  int32_t* __restrict__ perm) {
  extern __shared__ int64_t run[];
  const int lane = threadIdx.x;
  const int64_t b = blockIdx.x;
  for (int k = lane; k < K; k += 32) run[k] = coff[k] + base[(int64_t)k * nblk + b];
  __syncwarp();
  const int64_t end = min(n, (b + 1) * (int64_t)kSortBlock);
  for (int64_t i0 = b * kSortBlock; i0 < end; i0 += 32) {
    const int64_t i = i0 + lane;
    const bool ok = i < end;
    const int k = ok ? labels[i] : -1 - lane;
    const uint32_t same = __match_any_sync(kFM, k);
    if (ok) {
      const int rank = __popc(same & lanemask_lt());
      perm[run[k] + rank] = (int32_t)i;
    }
    __syncwarp();
    if (ok && (same & lanemask_lt()) == 0) run[k] += __popc(same);
    __syncwarp();
  }
}

template <typename V>
__global__ void __launch_bounds__(kPartWarps * 32)
    km_chunk_kernel(const int32_t* __restrict__ idx, const void* __restrict__ val, int m, int32_t p_pad,
                    const int32_t* __restrict__ perm, const int64_t* __restrict__ chunks, double* __restrict__ psum,
                    int32_t* __restrict__ pcnt) {
  extern __shared__ unsigned char sm[];
  const int c = blockIdx.x;
  const int64_t meta = chunks[2 * c + 1];
  if (meta < 0) return;
  const int64_t start = chunks[2 * c];
  const int len = (int)(meta & 0xFFFFFFFF);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double* ws = reinterpret_cast<double*>(sm) + (size_t)warp * p_pad;
  int* wc = reinterpret_cast<int*>(sm + (size_t)kPartWarps * p_pad * 8) + (size_t)warp * p_pad;
  for (int j = lane; j < p_pad; j += 32) {
    ws[j] = 0.0;
    wc[j] = 0;
  }
  __syncwarp();
  const int q0 = len * warp / kPartWarps, q1 = len * (warp + 1) / kPartWarps;
  int q = q0;
  if (m <= 64) {  // batches of 4 points: perm and row loads issued before the updates
    for (; q + 4 <= q1; q += 4) {
      int64_t pi[4];
#pragma unroll
      for (int b = 0; b < 4; ++b) pi[b] = perm[start + q + b];
      int jj[4][2];
      double vv[4][2];
#pragma unroll
      for (int b = 0; b < 4; ++b)
#pragma unroll
        for (int c2 = 0; c2 < 2; ++c2) {
          const int t = lane + 32 * c2;
          jj[b][c2] = -1;
          if (t < m) {
            jj[b][c2] = __ldg(idx + pi[b] * m + t);
            vv[b][c2] = ldd<V>(val, pi[b] * m + t);
          }
        }
#pragma unroll
      for (int b = 0; b < 4; ++b) {
#pragma unroll
        for (int c2 = 0; c2 < 2; ++c2)
          if (jj[b][c2] >= 0) {
            ws[jj[b][c2]] = dadd(ws[jj[b][c2]], vv[b][c2]);
            wc[jj[b][c2]] += 1;
          }
        __syncwarp();
      }
    }
  }
  for (; q < q1; ++q) {
    const int64_t i = perm[start + q];
    for (int t = lane; t < m; t += 32) {
      const int j = __ldg(idx + i * m + t);
      ws[j] = dadd(ws[j], ldd<V>(val, i * m + t));
      wc[j] += 1;
    }
    __syncwarp();
  }
  __syncthreads();
  double* os = psum + (size_t)c * p_pad;
  int32_t* oc = pcnt + (size_t)c * p_pad;
  for (int j = threadIdx.x; j < p_pad; j += blockDim.x) {
    double s = 0.0;
    int cnt = 0;
    for (int w = 0; w < kPartWarps; ++w) {
      s = dadd(s, reinterpret_cast<double*>(sm)[(size_t)w * p_pad + j]);
      cnt += reinterpret_cast<int*>(sm + (size_t)kPartWarps * p_pad * 8)[(size_t)w * p_pad + j];
    }
    os[j] = s;
    oc[j] = cnt;
  }
}

// sums[j][k] / counts[j][k]: chunks of cluster k added in order
__global__ void km_chunk_reduce_kernel(const double* __restrict__ psum, const int32_t* __restrict__ pcnt,
                                       const int64_t* __restrict__ cfirst, int32_t p_pad, int K,
                                       double* __restrict__ sums, int64_t* __restrict__ counts) {
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= (int64_t)p_pad * K) return;
  const int j = (int)(e / K), k = (int)(e % K);
  double s = 0.0;
  int64_t cnt = 0;
  for (int64_t c = cfirst[k]; c < cfirst[k + 1]; ++c) {
    s = dadd(s, psum[(size_t)c * p_pad + j]);
    cnt += pcnt[(size_t)c * p_pad + j];
  }
  sums[e] = s;
  counts[e] = cnt;
}

int partials_launch(const int32_t* idx, const void* val, int val_f64, int64_t n, int32_t m, const int32_t* labels,
                    int32_t p_pad, int32_t K, double* sums, int64_t* counts, int64_t* sizes, void* ws,
                    cudaStream_t st) {
  const PartLayout L = part_layout(n, p_pad, K);
  char* w = reinterpret_cast<char*>(ws);
  int32_t* hist = reinterpret_cast<int32_t*>(w + L.off_hist);
  int64_t* base = reinterpret_cast<int64_t*>(w + L.off_base);
  int32_t* perm = reinterpret_cast<int32_t*>(w + L.off_perm);
  int64_t* coff = reinterpret_cast<int64_t*>(w + L.off_coff);
  int64_t* cfirst = reinterpret_cast<int64_t*>(w + L.off_cfirst);
  int64_t* chunks = reinterpret_cast<int64_t*>(w + L.off_chunks);
  double* psum = reinterpret_cast<double*>(w + L.off_psum);
  int32_t* pcnt = reinterpret_cast<int32_t*>(w + L.off_pcnt);
  int rc;
  const size_t hsm = (size_t)K * 4;
  cudaFuncSetAttribute(km_hist_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)hsm);
  if (n > 0) {
    km_hist_kernel<<<(unsigned)L.nblk, 256, hsm, st>>>(labels, n, K, L.nblk, hist);
    if ((rc = check_launch("km_hist_kernel"))) return rc;
  } else {
    cudaMemsetAsync(hist, 0, (size_t)L.nblk * K * 4, st);
  }
  km_scan_kernel<<<K, 256, 0, st>>>(hist, L.nblk, base, sizes);
  if ((rc = check_launch("km_scan_kernel"))) return rc;
  km_offsets_kernel<<<1, 1024, 0, st>>>(sizes, K, L.ch, L.nchunk_max, coff, cfirst, chunks);
  if ((rc = check_launch("km_offsets_kernel"))) return rc;
  if (n > 0) {
    const size_t ssm = (size_t)K * 8;
    cudaFuncSetAttribute(km_scatter_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ssm);
    km_scatter_kernel<<<(unsigned)L.nblk, 32, ssm, st>>>(labels, n, K, L.nblk, base, coff, perm);
    if ((rc = check_launch("km_scatter_kernel"))) return rc;
    const size_t csm = (size_t)kPartWarps * p_pad * 12;
    auto kk = val_f64 ? km_chunk_kernel<double> : km_chunk_kernel<float>;
    cudaFuncSetAttribute(kk, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)csm);
    kk<<<(unsigned)L.nchunk_max, kPartWarps * 32, csm, st>>>(idx, val, m, p_pad, perm, chunks, psum, pcnt);
    if ((rc = check_launch("km_chunk_kernel"))) return rc;
  }
  const int64_t tot = (int64_t)p_pad * K;
  km_chunk_reduce_kernel<<<(unsigned)((tot + 255) / 256), 256, 0, st>>>(psum, pcnt, cfirst, p_pad, K, sums,
                                                                          counts);
  return check_launch("km_chunk_reduce_kernel");
}

int partials_check(int32_t p_pad, int32_t K) {
  if ((size_t)kPartWarps * p_pad * 12 > 227 * 1024)
    return fail(SKC_EPARAM, "p_pad too large for the K-means update kernel");
  if ((size_t)K * 8 > 227 * 1024) return fail(SKC_EPARAM, "K too large for the K-means update kernel");
  return SKC_OK;
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
                                int64_t c, const double* __restrict__ colsq, const double* __restrict__ dense,
                                double scale, double* __restrict__ out) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  double cross = 0.0;
  for (int t = 0; t < m; ++t) cross = dadd(cross, dmul(ldd<V>(val, i * m + t), __ldg(dense + __ldg(idx + i * m + t))));
  const double d2 = dsub(dadd(colsq[i], colsq[c]), dmul(2.0, cross));
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

int d2_point_launch(const int32_t* idx, const void* val, int val_f64, int64_t n, int32_t m, int32_t p_pad, int64_t c,
                    const double* colsq, double* dense, double* out, cudaStream_t st) {
  const double scale = (double)p_pad / (double)m;
  if (val_f64) dense_point_kernel<double><<<1, 256, 0, st>>>(idx, val, m, p_pad, c, dense);
  else dense_point_kernel<float><<<1, 256, 0, st>>>(idx, val, m, p_pad, c, dense);
  int rc = check_launch("dense_point_kernel");
  if (rc) return rc;
  const unsigned blocks = (unsigned)((n + 255) / 256);
  if (val_f64) d2_point_kernel<double><<<blocks, 256, 0, st>>>(idx, val, n, m, c, colsq, dense, scale, out);
  else d2_point_kernel<float><<<blocks, 256, 0, st>>>(idx, val, n, m, c, colsq, dense, scale, out);
  return check_launch("d2_point_kernel");
}

}  // namespace skc
