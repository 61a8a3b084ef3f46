// K2 moments (mean accumulation + value statistics), K3 covariance band accumulation,
// K4 covariance finalize, K7 adjoint transform (mean / PCs / centres).
// Reference: estimators.py:30-66, transform.py:92-200.
#include <math.h>
#include <stdio.h>
#include <stdlib.h>

#include <map>
#include <mutex>
#include <tuple>

#include "common.cuh"

namespace skc {

constexpr uint32_t kFullMask = 0xFFFFFFFFu;

// ======================================================================================
// K2: acc[j] += sum of values with index j (estimators.py:39-43), plus sum of squares and
// max |v| for K3's fixed-point scale. Each warp owns a private fp64 p-vector in smem and
// walks a fixed contiguous range of rows. Indices are distinct within a row, so lanes
// never collide. Warps combine in order, then CTAs combine in order, so the result is
// deterministic.
// ======================================================================================
int moments_grid(int64_t n) {
  int64_t g = (n + 255) / 256;
  const int64_t cap = 3 * (int64_t)sm_count();  // 3 CTAs (24 warps) per SM at p_pad <= 1024
  if (g > cap) g = cap;
  if (g < 1) g = 1;
  return (int)g;
}
static int moments_warps(int32_t p_pad) {
  int w = 8;
  while (w > 1 && (size_t)w * p_pad * 8 > 128 * 1024) w >>= 1;
  return w;
}

template <typename V, int MAXC>  // MAXC lane-chunks per row cover m <= 32 * MAXC from registers
__global__ void moments_kernel(const int32_t* __restrict__ idx, const V* __restrict__ val, int64_t n, int32_t m,
                               int32_t p_pad, double* __restrict__ part) {
  extern __shared__ double wvec[];  // [warps][p_pad]
  const int warps = blockDim.x >> 5, warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double* mine = wvec + (size_t)warp * p_pad;
  for (int j = lane; j < p_pad; j += 32) mine[j] = 0.0;
  __syncwarp();
  const int64_t c0 = n * blockIdx.x / gridDim.x, c1 = n * (blockIdx.x + 1) / gridDim.x;
  const int64_t r0 = c0 + (c1 - c0) * warp / warps, r1 = c0 + (c1 - c0) * (warp + 1) / warps;
  double sqc[MAXC], mx = 0.0;  // one square-sum chain per lane-chunk (they only feed K3's scale)
#pragma unroll
  for (int c = 0; c < MAXC; ++c) sqc[c] = 0.0;
  // rows in batches of kB: all loads of a batch are issued before the shared-memory updates
  constexpr int kB = 8;
  int64_t r = r0;
  if (m <= 32 * MAXC) {
    for (; r + kB <= r1; r += kB) {
      int jj[kB][MAXC];
      double vv[kB][MAXC];
#pragma unroll
      for (int b = 0; b < kB; ++b)
#pragma unroll
        for (int c = 0; c < MAXC; ++c) {
          const int t = lane + 32 * c;
          jj[b][c] = -1;
          vv[b][c] = 0.0;
          if (t < m) {
            jj[b][c] = __ldg(idx + (r + b) * m + t);
            vv[b][c] = (double)__ldg(val + (r + b) * m + t);
          }
        }
#pragma unroll
      for (int b = 0; b < kB; ++b) {
#pragma unroll
        for (int c = 0; c < MAXC; ++c) {
          if (jj[b][c] >= 0) {
            const double v = vv[b][c];
            mine[jj[b][c]] = dadd(mine[jj[b][c]], v);
            sqc[c] = dadd(sqc[c], dmul(v, v));
            mx = fmax(mx, fabs(v));
          }
        }
        __syncwarp();
      }
    }
  }
  for (; r < r1; ++r) {
    for (int t = lane; t < m; t += 32) {
      const int j = __ldg(idx + r * m + t);
      const double v = (double)__ldg(val + r * m + t);
      mine[j] = dadd(mine[j], v);
      sqc[0] = dadd(sqc[0], dmul(v, v));
      mx = fmax(mx, fabs(v));
    }
    __syncwarp();
  }
  double sq = sqc[0];
#pragma unroll
  for (int c = 1; c < MAXC; ++c) sq = dadd(sq, sqc[c]);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    sq = dadd(sq, __shfl_xor_sync(kFullMask, sq, o));
    mx = fmax(mx, __shfl_xor_sync(kFullMask, mx, o));
  }
  __shared__ double wsq[32], wmx[32];
  if (lane == 0) {
    wsq[warp] = sq;
    wmx[warp] = mx;
  }
  __syncthreads();
  double* out = part + (size_t)blockIdx.x * (p_pad + 2);
  for (int j = threadIdx.x; j < p_pad; j += blockDim.x) {
    double s = 0.0;
    for (int w = 0; w < warps; ++w) s = dadd(s, wvec[(size_t)w * p_pad + j]);
    out[j] = s;
  }
  if (threadIdx.x == 0) {
    double s = 0.0, x = 0.0;
    for (int w = 0; w < warps; ++w) {
      s = dadd(s, wsq[w]);
      x = fmax(x, wmx[w]);
    }
    out[p_pad] = s;
    out[p_pad + 1] = x;
  }
}

__global__ void moments_reduce_kernel(const double* __restrict__ part, int G, int32_t p_pad, int64_t n,
                                      double* __restrict__ acc, double* __restrict__ stats) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j < p_pad) {
    double s = 0.0;
    for (int g = 0; g < G; ++g) s = dadd(s, part[(size_t)g * (p_pad + 2) + j]);
    acc[j] = dadd(acc[j], s);
  } else if (j == p_pad && stats != nullptr) {
    double s = 0.0, x = 0.0;
    for (int g = 0; g < G; ++g) {
      s = dadd(s, part[(size_t)g * (p_pad + 2) + p_pad]);
      x = fmax(x, part[(size_t)g * (p_pad + 2) + p_pad + 1]);
    }
    stats[0] = dadd(stats[0], s);
    stats[1] = fmax(stats[1], x);
    stats[2] = dadd(stats[2], (double)n);
  }
}

size_t moments_ws(int64_t n, int32_t p_pad) { return (size_t)moments_grid(n) * (p_pad + 2) * sizeof(double); }

int moments_launch(const int32_t* idx, const void* val, int val_f64, int64_t n, int32_t m, int32_t p_pad,
                   double* acc, double* stats, void* ws, cudaStream_t st) {
  const int G = moments_grid(n);
  const int W = moments_warps(p_pad);
  const size_t smem = (size_t)W * p_pad * sizeof(double);
  double* part = reinterpret_cast<double*>(ws);
  if (n > 0) {
    if (val_f64) {
      if (m <= 64) {
        cudaFuncSetAttribute(moments_kernel<double, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        moments_kernel<double, 2><<<G, W * 32, smem, st>>>(idx, (const double*)val, n, m, p_pad, part);
      } else {
        cudaFuncSetAttribute(moments_kernel<double, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        moments_kernel<double, 4><<<G, W * 32, smem, st>>>(idx, (const double*)val, n, m, p_pad, part);
      }
    } else {
      if (m <= 64) {
        cudaFuncSetAttribute(moments_kernel<float, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        moments_kernel<float, 2><<<G, W * 32, smem, st>>>(idx, (const float*)val, n, m, p_pad, part);
      } else {
        cudaFuncSetAttribute(moments_kernel<float, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        moments_kernel<float, 4><<<G, W * 32, smem, st>>>(idx, (const float*)val, n, m, p_pad, part);
      }
    }
    int rc = check_launch("moments_kernel");
    if (rc) return rc;
    moments_reduce_kernel<<<(p_pad + 1 + 255) / 256, 256, 0, st>>>(part, G, p_pad, n, acc, stats);
    return check_launch("moments_reduce_kernel");
  }
  return SKC_OK;
}

// ======================================================================================
// K3: raw W W^T upper triangle (estimators.py:59-61), in row bands that fit shared memory.
// CTA (band b, group g) with 32 warps holds band b as an int32 "low word" per entry. Each
// product w_a*w_b is scaled by 2^S (|q| <= 2^30 for |w| <= tau) and added with a native
// ATOMS.ADD whose returned old value yields the carry. A nonzero carry/borrow (~1 in 2^8
// adds) goes to the group's int64 partial in global memory with a native REDG.ADD.64.
// A row holding a value above tau sends its products (fp64, then scaled to int64)
// straight to that REDG path. Every sum is integer, so the result is exact in the fixed
// point and independent of order (deterministic). At the end the CTA adds its low words
// into the same int64 partial. A reduce kernel sums the groups in int64 and scales to fp64.
// tau = 8 * rms(values), from K2's statistics. Quantum 2^-S ~ 6e-8 * tau^2.
// Band boundaries of the flat kernel adapt to measured per-band time (band_plan below); the
// sums do not depend on them.
// Two kernels share this scheme: cov_flat_kernel (m <= 64, the default; lean per-visit work and
// a packed pair table) and cov_band_kernel (m > 64, or SKC_COV_KERNEL=band). Both are bound by
// the shared-memory pipe: an ATOMS wavefront costs about two load wavefronts, and random 32-lane
// atomics average 3.3 wavefronts of bank conflicts (profiles/round2/notes.md).
// ======================================================================================
#ifndef SKC_COV_UNROLL
#define SKC_COV_UNROLL 1  // unroll of the flat pair loop (experiments)
#endif
#ifndef SKC_COV_SMEM_KB
#define SKC_COV_SMEM_KB 226
#endif
#ifndef SKC_COV_WARPS
#define SKC_COV_WARPS 32
#endif
constexpr int kCovUnroll = SKC_COV_UNROLL;
constexpr int kSmemBudget = SKC_COV_SMEM_KB * 1024;  // dynamic smem per CTA
constexpr int kCovWarps = SKC_COV_WARPS;
constexpr int kMaxBands = 511;

__host__ __device__ inline int64_t tri_off(int64_t a, int64_t p) { return a * p - a * (a - 1) / 2; }

// visit pair table (m <= 64): bytes t[f], u[f] of the f-th pair (t <= u) in t-major order,
// so the pairs of rows t in [nlo, nhi) are the contiguous range [tri_off(nlo), tri_off(nhi)),
// followed by the u16 table F(t) = tri_off(t) for t = 0..m (the flat kernel's loop bounds)
static size_t pair_table_bytes(int32_t m) {
  return m <= 64 ? (((size_t)m * (m + 1) / 2 + 1) & ~(size_t)1) * 4 + (((size_t)m + 4) & ~(size_t)3) * 2 : 0;
}
// band kernel for m <= 64: 'f' flat pair table (default) or 'b' the round-1 band kernel
// (SKC_COV_KERNEL=band, A/B runs); m > 64: 'b'.
static char band_kind(int32_t m) {
  if (m > 64) return 'b';
  const char* k = getenv("SKC_COV_KERNEL");
  return (k && k[0] == 'b') ? 'b' : 'f';
}
static size_t flat_ptab_bytes(int32_t m) { return (((size_t)m * (m + 1) / 2 + 1) & ~(size_t)1) * 4; }
static int band_capacity(int32_t m, int32_t p_pad) {
  if (band_kind(m) == 'f')  // lo words + the pair table + per-warp U staging
    return (int)(((size_t)kSmemBudget - (size_t)kCovWarps * m * 8 - flat_ptab_bytes(m)) / 4);
  // int32 entries left after the per-warp row staging, the row table and the pair table
  return (int)(((size_t)kSmemBudget - (size_t)kCovWarps * m * 16 - 4 * (size_t)p_pad - pair_table_bytes(m)) / 4);
}
// greedy row bands of <= cap entries; returns the count, fills out[0..count] if given
static int greedy_bands(int32_t p_pad, int64_t cap, int* out) {
  int nb = 0, a = 0;
  while (a < p_pad) {
    int64_t e = 0;
    int r = a;
    while (r < p_pad && e + (p_pad - r) <= cap) {
      e += p_pad - r;
      ++r;
    }
    if (r == a) r = a + 1;
    if (out && nb < kMaxBands) out[nb] = a;
    ++nb;
    a = r;
  }
  if (out && nb <= kMaxBands) out[nb] = p_pad;
  return nb;
}
// as few bands as the capacity allows, balanced: the smallest per-band bound that keeps the
// greedy count (equal entries = equal expected pairs per band)
static int make_bands(int32_t p_pad, int cap, int* out) {
  const int nb = greedy_bands(p_pad, cap, nullptr);
  const int64_t total = tri_off(p_pad, p_pad);
  int64_t t = (total + nb - 1) / nb;
  while (t < cap && greedy_bands(p_pad, t, nullptr) > nb) t += (t >> 6) + 1;
  if (t > cap) t = cap;
  return greedy_bands(p_pad, t, out);
}

struct CovParams {
  const int32_t* idx;
  const void* val;
  int64_t n;
  int32_t m, p_pad;
  const double* stats;
  double* tri;               // output triangle (wide-range / huge products go here in fp64)
  unsigned long long* part;  // [groups][tri_total] int64 fixed-point partials
  int nbands, groups;
  int aligned;               // idx/val 16-byte aligned: tiles may use bulk copies
  int band_rows[kMaxBands + 1];
  unsigned long long* cyc;   // [groups][nbands] end stamps per band CTA + the start stamp, ns (measuring launches)
};

template <typename V>
__device__ __forceinline__ double ldv64(const void* p, int64_t i) {
  return (double)__ldg(reinterpret_cast<const V*>(p) + i);
}

// predicated 64-bit global reduction without a branch (the carry path is rare)
__device__ __forceinline__ void red_if(bool p, unsigned long long* addr, unsigned long long v) {
  asm volatile(
      "{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %0, 0;\n\t@q red.global.add.u64 [%1], %2;\n\t}" ::"r"((unsigned)p),
      "l"(addr), "l"(v)
      : "memory");
}

// S from the value statistics; identical in every CTA and in the reduce kernel. Products are
// w_a * w_b * 2^S, |q| <= 2^30 for |w| <= tau; S is even and each factor carries 2^(S/2) as a
// float. Outside |S| <= kWideS (rms below ~2^-105 or above ~2^135, e.g. fp64 sketches of
// extreme data) the factors are not representable as scaled floats, and every product takes
// the exact fp64 path instead (cov_wide).
constexpr int kWideS = 240;
__device__ __forceinline__ int cov_scale(const double* stats, int m, double* tau_out) {
  const double cnt = stats[2] * (double)m;
  const double rms = cnt > 0 ? sqrt(stats[0] / cnt) : 0.0;
  double tau = 8.0 * rms;
  if (!(tau > 0.0) || !(tau <= 1.0e300)) tau = 1.0;  // zero, NaN or overflowed statistics
  *tau_out = tau;
  const int S = (int)floor(30.0 - 2.0 * log2(tau));
  return max(-1000, min(1000, S)) & ~1;
}
__device__ __forceinline__ bool cov_wide(int S) { return S > kWideS || S < -kWideS; }
// exact fp64 fallback for one product: int64 fixed point when it fits, else (huge outliers,
// NaN/inf, or a wide-range scale) an fp64 atomic straight into the output triangle
__device__ __forceinline__ void cov_add_exact(double va, double vb, double full_s, bool wide,
                                              unsigned long long* part_e, double* tri_e) {
  const double pr = dmul(va, vb);
  const double q = dmul(pr, full_s);
  if (!wide && fabs(q) < 4.611686018427387904e18) atomicAdd(part_e, (unsigned long long)__double2ll_rn(q));
  else atomicAdd(tri_e, pr);
}

// Each warp streams its own rows (no CTA-wide synchronisation), prefetching the next row
// into registers while the current one is processed. Lanes own columns u of the row, so
// b_u and w_u stay in registers, and the loop runs over the band's rows t < u. Per update:
// IADD, FMUL, F2I, ATOMS and a carry test. The low words carry a 2^31 bias, so a carry
// needs a drift of 2^31 quanta and is rare even for entries whose sum hovers around zero.
constexpr uint32_t kBias = 0x80000000u;


template <typename V, bool WIDE>  // WIDE: m > 64 (columns beyond the two register chunks)
__global__ void __launch_bounds__(kCovWarps * 32, 1) cov_band_kernel(const __grid_constant__ CovParams P) {
  extern __shared__ int smem_i[];
  const int m = P.m;
  const int band = blockIdx.x % P.nbands, group = blockIdx.x / P.nbands;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int r0 = P.band_rows[band], r1 = P.band_rows[band + 1];
  const int64_t e0 = tri_off(r0, P.p_pad), e1 = tri_off(r1, P.p_pad);
  const int ne = (int)(e1 - e0);
  uint32_t* lo = reinterpret_cast<uint32_t*>(smem_i);
  int* rowbase = smem_i + ((ne + 1) & ~1);  // [r1 - r0]: entry (a, b) sits at rowbase[a - r0] + b
  // per-warp staging, 4*m words: the general path uses [sidx: m][sval: m], the flat path
  // reuses it as int2 T[m], U[m]
  const int npair = !WIDE ? m * (m + 1) / 2 : 0;
  uint8_t* ptt = reinterpret_cast<uint8_t*>(rowbase + ((r1 - r0 + 1) & ~1));
  uint8_t* ptu = ptt + npair;
  int* stage = reinterpret_cast<int*>(ptt + ((2 * npair + 7) & ~7)) + (size_t)warp * 4 * m;
  int* sidx = stage;
  float* sval = reinterpret_cast<float*>(stage + m);
  unsigned long long* part = P.part + (size_t)group * tri_off(P.p_pad, P.p_pad) + e0;

  double tau;
  const int S = cov_scale(P.stats, m, &tau);
  const bool wide = cov_wide(S);
  const float sh = wide ? 1.0f : (float)ldexp(1.0, S / 2);  // 2^(S/2) on each factor
  const double full_s = ldexp(1.0, S);
  const float ftau = wide ? -1.0f : (float)tau;  // wide: every row takes the exact path
  double* tri_b = P.tri + e0;

  for (int e = threadIdx.x; e < ne; e += blockDim.x) lo[e] = kBias;
  for (int a = r0 + threadIdx.x; a < r1; a += blockDim.x) rowbase[a - r0] = (int)(tri_off(a, P.p_pad) - e0) - a;
  if (npair && threadIdx.x < m) {
    const int t = threadIdx.x, f0 = t * m - ((t * (t - 1)) >> 1);
    for (int u = t; u < m; ++u) ptt[f0 + u - t] = (uint8_t)t, ptu[f0 + u - t] = (uint8_t)(m + u);  // U = T + m
  }
  __syncthreads();

  const int64_t g0 = P.n * group / P.groups, g1 = P.n * (group + 1) / P.groups;
  const V* val = reinterpret_cast<const V*>(P.val);
  const uint32_t lo_sh = (uint32_t)__cvta_generic_to_shared(lo);
  // lanes hold columns lane and lane + 32 of a row; the next row loads into registers
  // while the warp processes the current one (a two-set ping-pong measured slower: code size)
  const int64_t stride = (int64_t)kCovWarps * m;
  const int32_t* ip = P.idx + (g0 + warp) * (int64_t)m + lane;  // lane's column in the row
  const V* vp = val + (g0 + warp) * (int64_t)m + lane;
  const bool has0 = lane < m, has1 = lane + 32 < m;
  int aj0 = 0x7FFFFFFF, aj1 = 0x7FFFFFFF;
  V av0 = 0, av1 = 0;
  auto load = [&](int64_t r, const int32_t* ipr, const V* vpr, int& j0, int& j1, V& v0, V& v1) {
    if (r < g1) {
      if (has0) j0 = __ldg(ipr), v0 = __ldg(vpr);
      if (has1) j1 = __ldg(ipr + 32), v1 = __ldg(vpr + 32);
    }
  };
  // per-warp staging, 4*m words: the flat path uses int2 T[m] = (shared byte address of
  // row t's entries, w_t * 2^S) and U[m] = (4 * b_u, w_u); the general path [sidx][sval]
  int2* T = reinterpret_cast<int2*>(sidx);
  int2* U = T + m;
  auto visit = [&](const int64_t r, const int j0, const int j1, const float v0, const float v1) {
    int nlo = __popc(__ballot_sync(kFullMask, j0 < r0)) + __popc(__ballot_sync(kFullMask, j1 < r0));
    int nhi = __popc(__ballot_sync(kFullMask, j0 < r1)) + __popc(__ballot_sync(kFullMask, j1 < r1));
    bool big = !(fabsf(v0) <= ftau) || !(fabsf(v1) <= ftau);  // lanes past m hold 0; NaN is big
    if constexpr (WIDE) {
      for (int t0 = 64; t0 < m; t0 += 32) {  // columns beyond the two register chunks
        const int t = t0 + lane;
        const int j = t < m ? __ldg(P.idx + r * m + t) : 0x7FFFFFFF;
        if (t < m) big |= !(fabsf((float)__ldg(val + r * m + t)) <= ftau);
        nlo += __popc(__ballot_sync(kFullMask, j < r0));
        nhi += __popc(__ballot_sync(kFullMask, j < r1));
      }
    }
    if (nlo == nhi) return;  // none of this row's indices fall in the band
    const bool any_big = __any_sync(kFullMask, big);
    if (!WIDE && !any_big) {
      // the visit's pairs {(t, u): nlo <= t < nhi, t <= u < m} are the contiguous range
      // [tri_off(nlo), tri_off(nhi)) of the t-major pair table; lane f takes pair f
      const float s0 = v0 * sh, s1 = v1 * sh;  // exact power-of-two scalings
      if (has0) U[lane] = make_int2(j0 << 2, __float_as_int(s0));
      if (has1) U[lane + 32] = make_int2(j1 << 2, __float_as_int(s1));
      if (lane >= nlo && lane < nhi) T[lane] = make_int2((int)lo_sh + 4 * rowbase[j0 - r0], __float_as_int(s0));
      if (lane + 32 >= nlo && lane + 32 < nhi)
        T[lane + 32] = make_int2((int)lo_sh + 4 * rowbase[j1 - r0], __float_as_int(s1));
      __syncwarp();
      const int F1 = nhi * m - ((nhi * (nhi - 1)) >> 1);
#pragma unroll kCovUnroll
      for (int f = nlo * m - ((nlo * (nlo - 1)) >> 1) + lane; f < F1; f += 32) {
        const int2 tt = T[ptt[f]], uu = T[ptu[f]];
        const uint32_t addr = (uint32_t)(tt.x + uu.x);
        const int q = __float2int_rn(__int_as_float(tt.y) * __int_as_float(uu.y));
        uint32_t old;
        asm volatile("atom.shared.add.u32 %0, [%1], %2;" : "=r"(old) : "r"(addr), "r"((uint32_t)q) : "memory");
        if ((old + (uint32_t)q < old) != (q < 0))  // carry (q >= 0) / borrow (q < 0): rare
          atomicAdd(part + ((addr - lo_sh) >> 2), (unsigned long long)((long long)(q < 0 ? -1 : 1) << 32));
      }
      __syncwarp();
      return;
    }
    // general path (m > 64, or a value above tau): stage the row in shared memory
    const int32_t* ir = P.idx + r * m;
    const V* vr = val + r * m;
    if (has0) {
      sidx[lane] = j0;
      sval[lane] = v0 * sh;
    }
    if (has1) {
      sidx[lane + 32] = j1;
      sval[lane + 32] = v1 * sh;
    }
    for (int t0 = 64; t0 < m; t0 += 32) {
      const int t = t0 + lane;
      if (t < m) {
        sidx[t] = __ldg(ir + t);
        sval[t] = (float)__ldg(vr + t) * sh;
      }
    }
    __syncwarp();
    if (!any_big) {
      for (int c0 = 0; c0 < m; c0 += 32) {
        const int u = c0 + lane;
        const int tmax = min(nhi, c0 + 32);  // rows t <= u within this chunk
        if (nlo >= tmax) continue;
        const int bu = u < m ? sidx[u] : 0;
        const float vu = u < m ? sval[u] : 0.f;
        for (int t = nlo; t < tmax; ++t) {
          const int base = rowbase[sidx[t] - r0];
          const float va = sval[t];
          if (t <= u && u < m) {
            const int e = base + bu;
            const int q = __float2int_rn(va * vu);
            const uint32_t old = atomicAdd(lo + e, (uint32_t)q);
            if ((old + (uint32_t)q < old) != (q < 0))  // carry (q >= 0) / borrow (q < 0): rare
              atomicAdd(part + e, (unsigned long long)((long long)(q < 0 ? -1 : 1) << 32));
          }
        }
      }
    } else {
      // a value above tau (or a wide-range scale): exact fp64 products
      for (int t = nlo; t < nhi; ++t) {
        const double va = (double)__ldg(vr + t);
        const int base = rowbase[sidx[t] - r0];
        for (int u = t + lane; u < m; u += 32)
          cov_add_exact(va, (double)__ldg(vr + u), full_s, wide, part + base + sidx[u], tri_b + base + sidx[u]);
      }
    }
    __syncwarp();
  };
  int64_t r = g0 + warp;
  load(r, ip, vp, aj0, aj1, av0, av1);
  while (r < g1) {
    const int j0 = aj0, j1 = aj1;
    const float v0 = (float)av0, v1 = (float)av1;
    ip += stride;
    vp += stride;
    load(r + kCovWarps, ip, vp, aj0, aj1, av0, av1);
    visit(r, j0, j1, v0, v1);
    r += kCovWarps;
  }
  __syncthreads();
  for (int e = threadIdx.x; e < ne; e += blockDim.x) {
    const long long q = (long long)lo[e] - (long long)kBias;
    if (q != 0) atomicAdd(part + e, (unsigned long long)q);
  }
}

// K3 flat kernel (m <= 64, the configs' shapes): the same fixed-point band accumulation as
// cov_band_kernel, with the per-visit work cut to what the pair loop needs.
//  * A warp stages only U[u] = (4 j_u, w_u 2^(S/2)) per row; pair (t, u) reads U[t] and U[u]
//    and forms the shared address of band row j_t in registers (a (p - 1) - a (a - 1) / 2), as it
//    does F(t): no row-address or offset tables, half the staging, so the band holds more entries
//    (10 bands at C3 instead of 11, one row visit fewer).
//  * Rows are walked with 32-bit counters and pointer bumps; band membership of a lane's
//    element is one unsigned compare (indices are sorted, so in-band lanes are [nlo, nhi)).
//  * The pair loop's induction variable is the pair-table pointer.
// Rows holding a value above tau (or a wide-range scale) take the exact fp64 path.
__device__ __forceinline__ unsigned long long global_timer_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// MEASURE: the launch stamps every block's end time for the adaptive band plan (BandPlan). A
// separate instantiation, because even this one store after all the work moves the kernel's code
// enough to cost ~2% (8.75 -> 8.90 ms at p = 512, 6.44 -> 6.58 ms at p = 256); the steady-state
// launches run the kernel without it.
template <typename V, bool PK, bool MEASURE>  // PK (p_pad <= 2048): U.x packs (row offset of j) << 11 | j
__global__ void __launch_bounds__(kCovWarps * 32, 1) cov_flat_kernel(const __grid_constant__ CovParams P) {
  extern __shared__ int smem_i[];
  const int m = P.m;
  const int band = blockIdx.x % P.nbands, group = blockIdx.x / P.nbands;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int r0 = P.band_rows[band], r1 = P.band_rows[band + 1];
  const int64_t e0 = tri_off(r0, P.p_pad), e1 = tri_off(r1, P.p_pad);
  const int ne = (int)(e1 - e0);
  uint32_t* lo = reinterpret_cast<uint32_t*>(smem_i);
  const int npair = m * (m + 1) / 2;
  // pair f: byte offsets of U[t] and U[u] in the warp's staging, 8 t | 8 u << 16
  uint32_t* ptab = lo + ((ne + 1) & ~1);
  int2* S = reinterpret_cast<int2*>(ptab + ((npair + 1) & ~1)) + (size_t)warp * m;  // U[m]
  unsigned long long* part = P.part + (size_t)group * tri_off(P.p_pad, P.p_pad) + e0;
  const uint32_t lo_sh = (uint32_t)__cvta_generic_to_shared(lo);

  double tau;
  const int S_ = cov_scale(P.stats, m, &tau);
  const bool wide = cov_wide(S_);
  const float sh = wide ? 1.0f : (float)ldexp(1.0, S_ / 2);  // 2^(S/2) on each factor
  const double full_s = ldexp(1.0, S_);
  const float ftau = wide ? -1.0f : (float)tau;  // wide: every row takes the exact path
  double* tri_b = P.tri + e0;

  for (int e = threadIdx.x; e < ne; e += blockDim.x) lo[e] = kBias;
  // band-row addresses and the pair-list offsets F(t) are computed in registers (fewer shared
  // loads per visit: ~7% of the kernel's shared-memory wavefronts)
  const uint32_t rb = lo_sh - 4u * (uint32_t)e0;  // entry (a, 0) at rb + 4 (a (p - 1) - a (a - 1) / 2)
  const uint32_t pm1 = (uint32_t)P.p_pad - 1u;
  if (threadIdx.x < m) {
    const int t = threadIdx.x, f0 = t * m - ((t * (t - 1)) >> 1);
    for (int u = t; u < m; ++u) ptab[f0 + u - t] = (uint32_t)(8 * t) | ((uint32_t)(8 * u) << 16);
  }
  __syncthreads();

  const int64_t g0 = P.n * group / P.groups, g1 = P.n * (group + 1) / P.groups;
  const int nrows = (int)(g1 - g0);
  const V* val = reinterpret_cast<const V*>(P.val);
  // lane's element pointers for row i of the group: gi + i * m (the prefetch of row i + 32
  // is clamped to the last row instead of branched around)
  const int32_t* const gi = P.idx + g0 * (int64_t)m + lane;
  const V* const gv = val + g0 * (int64_t)m + lane;
  const bool has0 = lane < m, has1 = lane + 32 < m;
  const uint32_t bw = (uint32_t)(r1 - r0);
  const uint32_t S_sh = (uint32_t)__cvta_generic_to_shared(S);
  int aj0 = 0x7FFFFFFF, aj1 = 0x7FFFFFFF;
  V av0 = 0, av1 = 0;
  if (warp < nrows) {
    const int32_t* ip = gi + (int64_t)warp * m;
    const V* vp = gv + (int64_t)warp * m;
    if (has0) aj0 = __ldg(ip), av0 = __ldg(vp);
    if (has1) aj1 = __ldg(ip + 32), av1 = __ldg(vp + 32);
  }
  for (int i = warp; i < nrows; i += kCovWarps) {
    const int j0 = aj0, j1 = aj1;
    const float v0 = (float)av0, v1 = (float)av1;
    {
      const uint32_t off = (uint32_t)min(i + kCovWarps, nrows - 1) * (uint32_t)m;  // < 2^31 per launch
      const int32_t* ip = gi + off;
      const V* vp = gv + off;
      if (has0) aj0 = __ldg(ip), av0 = __ldg(vp);
      if (has1) aj1 = __ldg(ip + 32), av1 = __ldg(vp + 32);
    }
    const int nlo = __popc(__ballot_sync(kFullMask, j0 < r0)) + __popc(__ballot_sync(kFullMask, j1 < r0));
    const int nhi = __popc(__ballot_sync(kFullMask, j0 < r1)) + __popc(__ballot_sync(kFullMask, j1 < r1));
    if (nlo == nhi) continue;  // none of this row's indices fall in the band
    const bool big = !(fabsf(v0) <= ftau) || !(fabsf(v1) <= ftau);  // lanes past m hold 0; NaN is big
    if (__any_sync(kFullMask, big)) {
      // exact fp64 products for this row's band pairs
      const int64_t r = g0 + i;
      const int32_t* ir = P.idx + r * m;
      const V* vr = val + r * m;
      for (int t = nlo; t < nhi; ++t) {
        const double va = (double)__ldg(vr + t);
        const uint32_t a = (uint32_t)__ldg(ir + t);
        const int base = (int)(a * pm1 - ((a * (a - 1u)) >> 1)) - (int)e0;  // signed: entry (a, 0) may precede e0
        for (int u = t + lane; u < m; u += 32) {
          const int e = base + __ldg(ir + u);
#ifdef SKC_COV_DEBUG
          if (e < 0 || e >= ne) {
            printf("cov_flat big: bad e %d ne %d band %d row %d t %d u %d\n", e, ne, band, i, t, u);
            __trap();
          }
#endif
          cov_add_exact(va, (double)__ldg(vr + u), full_s, wide, part + e, tri_b + e);
        }
      }
      continue;
    }
    const float s0 = v0 * sh, s1 = v1 * sh;  // exact power-of-two scalings
    if constexpr (PK) {
      // U.x = rowoff(j) << 11 | j, rowoff(a) = a (p - 1) - a (a - 1) / 2 < 2^21 for p <= 2048:
      // a pair's entry is then rb + 4 (rowoff(j_t) + j_u), four instructions per pair
      const uint32_t a0 = (uint32_t)j0, a1 = (uint32_t)j1;
      if (has0) S[lane] = make_int2((int)(((a0 * pm1 - ((a0 * (a0 - 1u)) >> 1)) << 11) | a0), __float_as_int(s0));
      if (has1)
        S[lane + 32] = make_int2((int)(((a1 * pm1 - ((a1 * (a1 - 1u)) >> 1)) << 11) | a1), __float_as_int(s1));
    } else {
      if (has0) S[lane] = make_int2(j0 << 2, __float_as_int(s0));
      if (has1) S[lane + 32] = make_int2(j1 << 2, __float_as_int(s1));
    }
    __syncwarp();
    const uint32_t* tp = ptab + (nlo * m - ((nlo * (nlo - 1)) >> 1)) + lane;  // F(t) in registers
    const uint32_t* const te = ptab + (nhi * m - ((nhi * (nhi - 1)) >> 1));
    for (; tp < te; tp += 32) {
      const uint32_t pe = *tp;
      int tx, ty, ux, uy;
      asm volatile("ld.shared.v2.s32 {%0, %1}, [%2];" : "=r"(tx), "=r"(ty) : "r"(S_sh + (pe & 0xFFFFu)));
      asm volatile("ld.shared.v2.s32 {%0, %1}, [%2];" : "=r"(ux), "=r"(uy) : "r"(S_sh + (pe >> 16)));
      uint32_t addr;
      if constexpr (PK) {
        addr = rb + 4u * (((uint32_t)tx >> 11) + ((uint32_t)ux & 0x7FFu));
      } else {
        const uint32_t ta = (uint32_t)tx >> 2;  // j_t: the band row's address in registers
        addr = rb + 4u * (ta * pm1 - ((ta * (ta - 1u)) >> 1)) + (uint32_t)ux;
      }
#ifdef SKC_COV_DEBUG
      if (addr < lo_sh || addr >= lo_sh + 4u * (uint32_t)ne || (addr & 3)) {
        printf("cov_flat: bad addr %u (lo %u ne %d) band %d row %d t %d u %d nlo %d nhi %d\n", addr, lo_sh, ne, band,
               i, (int)(pe & 0xFFFF) / 8, (int)(pe >> 16) / 8 - m, nlo, nhi);
        __trap();
      }
#endif
      const int q = __float2int_rn(__int_as_float(ty) * __int_as_float(uy));
      uint32_t old;
      asm volatile("atom.shared.add.u32 %0, [%1], %2;" : "=r"(old) : "r"(addr), "r"((uint32_t)q) : "memory");
      if ((old + (uint32_t)q < old) != (q < 0))  // carry (q >= 0) / borrow (q < 0): rare
        atomicAdd(part + ((addr - lo_sh) >> 2), (unsigned long long)((long long)(q < 0 ? -1 : 1) << 32));
    }
    __syncwarp();
  }
  __syncthreads();
  for (int e = threadIdx.x; e < ne; e += blockDim.x) {
    const long long q = (long long)lo[e] - (long long)kBias;
    if (q != 0) atomicAdd(part + e, (unsigned long long)q);
  }
  // every block stamps its end (%globaltimer); the start stamp comes from cov_stamp_kernel,
  // launched just before
  if constexpr (MEASURE) {
    if (threadIdx.x == 0) P.cyc[blockIdx.x] = global_timer_ns();
  }
}
__global__ void cov_stamp_kernel(unsigned long long* out) { *out = global_timer_ns(); }

__global__ void cov_reduce_kernel(const unsigned long long* __restrict__ part, int groups, int64_t total, int m,
                                  const double* __restrict__ stats, double* __restrict__ tri) {
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= total) return;
  double tau;
  const int S = cov_scale(stats, m, &tau);
  long long s = 0;
  for (int g = 0; g < groups; ++g) s += (long long)part[(size_t)g * total + e];
  tri[e] = dadd(tri[e], (double)s * ldexp(1.0, -S));
}

// ======================================================================================
// K3g: no bands. The triangle is an L2-resident int64 fixed-point array (p = 4096: 67 MB),
// and each product goes in with one red.global.add.u64: no carry logic, still exact and
// order-independent. A row is visited once: one warp per row enumerates all m(m+1)/2 pairs
// flatly (row x folded with row m-1-x into width m+1). For large p_pad the banded kernel's
// per-visit overhead dominates (p = 4096: 153 bands, ~22 products per visit), and this
// path replaces it (cov_launch chooses by band count).
// ======================================================================================
constexpr int kCovGWarps = 8;
constexpr int kCovGlobalBands = 24;  // more bands than this: the global path (tools/cov_probe.py crossover)

template <typename V>
__global__ void __launch_bounds__(kCovGWarps * 32) cov_global_kernel(const int32_t* __restrict__ idx,
                                                                    const V* __restrict__ val, int64_t n, int m,
                                                                    int32_t p_pad, const double* __restrict__ stats,
                                                                    unsigned long long* __restrict__ acc,
                                                                    double* __restrict__ tri) {
  extern __shared__ int2 gst[];  // per warp: T[m] = (tri_off(j) - j, w * 2^S), U[m] = (j, w)
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  int2* T = gst + (size_t)warp * 2 * m;
  int2* U = T + m;
  double tau;
  const int S = cov_scale(stats, m, &tau);
  const bool wide = cov_wide(S);
  const float sh = wide ? 1.0f : (float)ldexp(1.0, S / 2);  // 2^(S/2) on each factor
  const double full_s = ldexp(1.0, S);
  const float ftau = wide ? -1.0f : (float)tau;
  const int Lp = m + 1;
  const int F = m * (m + 1) / 2;
  float inv;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(inv) : "f"((float)Lp));
  const int64_t warps = (int64_t)gridDim.x * kCovGWarps;
  for (int64_t r = blockIdx.x * (int64_t)kCovGWarps + warp; r < n; r += warps) {
    const int32_t* ir = idx + r * m;
    const V* vr = val + r * m;
    bool big = false;
    for (int t = lane; t < m; t += 32) {
      const int j = __ldg(ir + t);
      const float w = (float)__ldg(vr + t);
      big |= !(fabsf(w) <= ftau);
      U[t] = make_int2(j, __float_as_int(w * sh));
      T[t] = make_int2((int)(tri_off(j, p_pad) - j), __float_as_int(w * sh));
    }
    const bool any_big = __any_sync(kFullMask, big);
    __syncwarp();
    if (!any_big) {
      float ff = (float)lane + 0.5f;
      for (int f = lane; f < F; f += 32, ff += 32.0f) {
        int rr = (int)(ff * inv);
        int c = f - rr * Lp;
        if (c < 0) c += Lp, --rr;  // guard the approximate reciprocal
        if (c >= Lp) c -= Lp, ++rr;
        const bool first = c < m - rr;
        const int t = first ? rr : m - 1 - rr;
        const int u = first ? rr + c : c - 1;
        const int2 tt = T[t], uu = U[u];
        const long long q = __float2ll_rn(__int_as_float(tt.y) * __int_as_float(uu.y));
        asm volatile("red.global.add.u64 [%0], %1;" ::"l"(acc + (tt.x + uu.x)), "l"(q) : "memory");
      }
    } else {  // a value above tau: exact fp64 products
      for (int t = 0; t < m; ++t) {
        const double va = (double)__ldg(vr + t);
        const int base = T[t].x;
        for (int u = t + lane; u < m; u += 32)
          cov_add_exact(va, (double)__ldg(vr + u), full_s, wide, acc + (base + U[u].x), tri + (base + U[u].x));
      }
    }
    __syncwarp();
  }
}

static int cov_launch_global(const int32_t* idx, const void* val, int val_f64, int64_t n, int32_t m, int32_t p_pad,
                             const double* stats, double* tri, void* ws, cudaStream_t st) {
  const int64_t total = tri_off(p_pad, p_pad);
  unsigned long long* acc = reinterpret_cast<unsigned long long*>(ws);
  cudaMemsetAsync(acc, 0, (size_t)total * 8, st);
  const size_t smem = (size_t)kCovGWarps * 2 * m * sizeof(int2);
  int64_t grid = (n + kCovGWarps - 1) / kCovGWarps;
  const int64_t cap = 8LL * sm_count();
  if (grid > cap) grid = cap;
  int rc;
  if (val_f64) {
    cudaFuncSetAttribute(cov_global_kernel<double>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cov_global_kernel<double><<<(unsigned)grid, kCovGWarps * 32, smem, st>>>(idx, (const double*)val, n, m, p_pad,
                                                                              stats, acc, tri);
  } else {
    cudaFuncSetAttribute(cov_global_kernel<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cov_global_kernel<float><<<(unsigned)grid, kCovGWarps * 32, smem, st>>>(idx, (const float*)val, n, m, p_pad,
                                                                            stats, acc, tri);
  }
  if ((rc = check_launch("cov_global_kernel"))) return rc;
  cov_reduce_kernel<<<(unsigned)((total + 255) / 256), 256, 0, st>>>(acc, 1, total, m, stats, tri);
  return check_launch("cov_reduce_kernel");
}

static int cov_groups(int nbands, int64_t n) {
  int g = sm_count() / nbands;
  if (g < 1) g = 1;
  const int64_t maxg = (n + 4095) / 4096;
  if (g > maxg) g = (int)(maxg < 1 ? 1 : maxg);
  return g;
}

// K3t (cov_tc.cu): the tensor-core path for large m/p
bool covtc_supported(int32_t p_pad);
size_t covtc_ws(int64_t n, int32_t m, int32_t p_pad);
int covtc_launch(const int32_t* idx, const void* val, int val_f64, int64_t n, int32_t m, int32_t p_pad,
                 const double* stats, double* tri, void* ws, cudaStream_t st);
// Smallest m at which the tensor-core path beats the scatter paths, per log2(p_pad) = 8..13
// (dense MMA work is independent of m, the scatter's grows as m^2). Measured on one B200,
// tools/covtc_probe.py (profiles/round1_covtc.log): p = 256: m 36, 512: 50, 1024: 70,
// 2048: 75 (against K3g), 4096: 140 (K3g; 272 units run as two waves); 8192 extrapolated.
static int tc_min_m(int32_t p_pad) {
  static const int t[6] = {36, 50, 70, 75, 140, 280};
  int l = 0;
  while ((1 << l) < p_pad) ++l;
  return l < 8 ? 1 << 30 : t[l > 13 ? 5 : l - 8];
}

// Band count of the banded path. The flat kernel takes one band more than the capacity needs
// when the entry-balanced bands would sit within 5% of it and the launch is long enough to be
// measured: the adaptive plan below then has room to move boundaries (SKC_COV_ADAPT=0, or a launch
// under 2^20 rows: the minimum count, entry-balanced, as before).
static bool cov_adapt_on() {
  const char* e = getenv("SKC_COV_ADAPT");
  return !(e && e[0] == '0');
}
constexpr int64_t kPlanMinRows = (int64_t)1 << 20;  // shorter launches measure start-up, not the bands
static int band_count(int32_t p_pad, int32_t m, int64_t n) {
  const int cap = band_capacity(m, p_pad);
  int nb = make_bands(p_pad, cap, nullptr);
  if (band_kind(m) == 'f' && cov_adapt_on() && n >= kPlanMinRows && nb >= 4 && nb < kMaxBands &&
      (double)nb * cap < 1.05 * (double)tri_off(p_pad, p_pad))
    ++nb;
  return nb;
}
// The starting plan: nb bands (at least the capacity's minimum count) balanced on the weight
// (p - a) + kappa p / m per row a -- its entries plus a fixed cost per row, which is what the
// measured per-band times at C3 fit (kappa ~ 1; the converged C3 plan gives its last band 8.5%
// fewer entries than its first). kappa = 0: balanced by entries. The measurements correct it.
static void bands_by_entries(int32_t p_pad, int nb, int cap, int32_t m, int* out) {
  double kappa = 1.0;
  if (const char* e = getenv("SKC_COV_KAPPA")) kappa = atof(e);
  const double c = kappa > 0.0 ? kappa * (double)p_pad / (double)m : 0.0;
  auto pack = [&](double W, int* o) {
    int count = 0, a = 0;
    while (a < p_pad) {
      int64_t e = 0;
      double w = 0.0;
      int r = a;
      while (r < p_pad && e + (p_pad - r) <= cap && w + (p_pad - r) + c <= W) {
        e += p_pad - r;
        w += (p_pad - r) + c;
        ++r;
      }
      if (r == a) r = a + 1;
      if (o && count < nb) o[count] = a;
      ++count;
      a = r;
    }
    if (o && count <= nb) o[count] = p_pad;
    return count;
  };
  double lo = 0.0, hi = (double)tri_off(p_pad, p_pad) + c * p_pad + 1.0;
  for (int it = 0; it < 60; ++it) {
    const double mid = 0.5 * (lo + hi);
    if (pack(mid, nullptr) <= nb) hi = mid;
    else lo = mid;
  }
  int tmp[kMaxBands + 1];
  const int got = pack(hi, tmp);
  for (int b = 0; b <= nb; ++b) out[b] = b <= got ? tmp[b] : p_pad;  // fewer bands than asked (tiny p): empty tail
}

// Adaptive band plan (flat kernel). Equal entries are equal expected pairs, but a band CTA also
// pays per in-band element of a row, so bands of many short rows run slower (3.9% between the
// fastest and slowest of C3's ten bands). The slowest band sets the kernel time, and bands of a
// group that drift apart re-read its rows from DRAM once their distance exceeds what L2 holds.
// Every flat-kernel CTA records its elapsed cycles; the next launch of the same shape moves the
// band boundaries so that the measured time per band evens out (time taken as uniform per entry
// inside a band), a few times, then keeps the plan. Results do not depend on the boundaries (the
// fixed-point sums are exact), only the time and the DRAM traffic do.
struct BandPlan {
  int nb = 0, updates = 0, groups = 0;
  int rows[kMaxBands + 1];
  int best_rows[kMaxBands + 1];  // the measured plan with the fastest slowest band
  double best_max = 0.0;         // its slowest band, cycles per row of the launch
  int64_t n_meas = 1;            // rows of the measured launch
  unsigned long long* h_cyc = nullptr;  // pinned
  cudaEvent_t ev = nullptr;
  bool pending = false;
};
constexpr int kPlanUpdates = 2;  // proposals; every one is measured, the best measured plan stays (at C3 the
                                 // second is the best: later ones, and damped steps, measured worse)
constexpr int kPlanMaxCtas = 1023;  // + the start stamp
static std::mutex g_plan_mu;
static std::map<std::tuple<int, int, int, int, int>, BandPlan> g_plans;

static void plan_update(BandPlan& B, int32_t p_pad, int cap) {
  // mean cycles per band over the groups of the measured launch
  double T[kMaxBands], tot = 0.0, mx = 0.0;
  for (int b = 0; b < B.nb; ++b) {
    double sum = 0.0;  // mean end stamp of the band's CTAs, from the launch's start stamp (ns)
    const unsigned long long t0 = B.h_cyc[(size_t)B.groups * B.nb];
    for (int g = 0; g < B.groups; ++g) sum += (double)(B.h_cyc[(size_t)g * B.nb + b] - t0);
    T[b] = t0 ? sum / B.groups : 0.0;
    if (!(T[b] > 0.0)) return;  // no measurement
    tot += T[b];
    if (T[b] > mx) mx = T[b];
  }
  mx /= (double)B.n_meas;
  if (B.best_max == 0.0 || mx < B.best_max) {
    B.best_max = mx;
    for (int b = 0; b <= B.nb; ++b) B.best_rows[b] = B.rows[b];
  }
  if (getenv("SKC_COV_PLAN_LOG")) {
    fprintf(stderr, "band plan update %d: slowest %.0f ns, spread %.2f%%, rows", B.updates, mx * (double)B.n_meas,
            100.0 * (mx * (double)B.n_meas * B.nb / tot - 1.0));
    for (int b = 0; b <= B.nb; ++b) fprintf(stderr, " %d", B.rows[b]);
    fprintf(stderr, "\n");
  }
  if (B.updates >= kPlanUpdates) {  // the last proposal has been measured: keep the best plan
    for (int b = 0; b <= B.nb; ++b) B.rows[b] = B.best_rows[b];
    return;
  }
  // time per entry taken as uniform inside a band (interpolating it between band centres
  // measured worse: 26 GB / 35.04 ms against 20 GB / 34.75 ms at C3)
  double dens[kMaxBands];
  for (int b = 0; b < B.nb; ++b) dens[b] = T[b] / (double)(tri_off(B.rows[b + 1], p_pad) - tri_off(B.rows[b], p_pad));
  auto cost = [&](int r) {
    int k = 0;
    while (k + 1 < B.nb && r >= B.rows[k + 1]) ++k;
    return dens[k] * (double)(p_pad - r);
  };
  double pred = 0.0;
  for (int r = 0; r < p_pad; ++r) pred += cost(r);
  const double target = pred / B.nb;
  int out[kMaxBands + 1];
  int nbo = 0, a = 0;
  out[0] = 0;
  while (a < p_pad && nbo < B.nb) {
    double w = 0.0;
    int64_t e = 0;
    int r = a;
    const bool last = nbo == B.nb - 1;
    while (r < p_pad) {
      const double wr = cost(r);
      if (e + (p_pad - r) > cap) break;
      if (!last && w + 0.5 * wr > target) break;
      w += wr;
      e += p_pad - r;
      ++r;
    }
    if (r == a) ++r;
    out[++nbo] = r;
    a = r;
  }
  if (a < p_pad || nbo != B.nb) return;  // the capacity could not take the remainder: keep the plan
  for (int b = 0; b <= B.nb; ++b) B.rows[b] = out[b];
}

// 'b' banded scatter (K3), 'g' global L2 scatter (K3g), 't' tensor cores (K3t).
// SKC_COV_PATH=b|g|t forces a path where it applies.
constexpr int64_t kCovSmallRows = (int64_t)1 << 18;  // below: the band partials' reduce dominates (C1: 0.29 vs 0.05 ms)
static char cov_path(int32_t m, int32_t p_pad, int64_t n) {
  const int cap = band_capacity(m, p_pad);
  const bool tc = covtc_supported(p_pad);
  if (const char* f = getenv("SKC_COV_PATH")) {
    if (f[0] == 't' && tc) return 't';
    if (f[0] == 'g') return 'g';
    if (f[0] == 'b' && cap >= p_pad) return 'b';
  }
  if (tc && (m >= tc_min_m(p_pad) || cap < p_pad)) return 't';
  if (cap < p_pad) return 'g';
  if (n < kCovSmallRows && (size_t)kCovGWarps * 2 * m * sizeof(int2) <= 200 * 1024) return 'g';
  return make_bands(p_pad, cap, nullptr) > kCovGlobalBands ? 'g' : 'b';
}

int cov_check(int32_t p_pad, int32_t m) {
  const char path = cov_path(m, p_pad, kCovSmallRows);
  if (path == 't') return SKC_OK;
  if (path == 'g') return (size_t)kCovGWarps * 2 * m * sizeof(int2) <= 200 * 1024
                              ? SKC_OK
                              : fail(SKC_EPARAM, "m too large for the covariance kernels");
  if (band_count(p_pad, m, kPlanMinRows) > kMaxBands) return fail(SKC_EPARAM, "too many covariance bands for p_pad");
  return SKC_OK;
}

size_t cov_ws(int64_t n, int32_t m, int32_t p_pad) {
  const char path = cov_path(m, p_pad, n);
  if (path == 't') return covtc_ws(n, m, p_pad);
  if (path == 'g') return (size_t)tri_off(p_pad, p_pad) * sizeof(unsigned long long);
  // a split launch's tail part may fall under kPlanMinRows and take the smaller band count
  const int ga = cov_groups(band_count(p_pad, m, n), n), gb = cov_groups(band_count(p_pad, m, 0), n);
  return (size_t)(ga > gb ? ga : gb) * tri_off(p_pad, p_pad) * sizeof(unsigned long long) + (size_t)(kPlanMaxCtas + 1) * 8;
}

static int cov_launch_part(const int32_t* idx, const void* val, int val_f64, int64_t n, int32_t m, int32_t p_pad,
                           const double* stats, double* tri, void* ws, cudaStream_t st) {
  CovParams H;
  const int cap = band_capacity(m, p_pad);
  const bool flat = band_kind(m) == 'f';
  H.nbands = band_count(p_pad, m, n);
  H.groups = cov_groups(H.nbands, n);
  H.cyc = nullptr;
  bool measure = false;
  BandPlan* plan = nullptr;
  if (flat && cov_adapt_on() && n >= kPlanMinRows && H.nbands * H.groups <= kPlanMaxCtas) {
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> lk(g_plan_mu);
    BandPlan& B = g_plans[std::make_tuple(dev, (int)p_pad, (int)m, val_f64, H.nbands)];
    if (B.nb != H.nbands) {  // first use (or the count changed with the environment)
      B.nb = H.nbands;
      B.updates = 0;
      B.best_max = 0.0;
      B.pending = false;
      bands_by_entries(p_pad, B.nb, cap, m, B.rows);
      if (B.h_cyc == nullptr && cudaMallocHost(&B.h_cyc, (size_t)(kPlanMaxCtas + 1) * 8) != cudaSuccess) B.h_cyc = nullptr;
      if (B.ev == nullptr && cudaEventCreateWithFlags(&B.ev, cudaEventDisableTiming) != cudaSuccess) B.ev = nullptr;
      cudaGetLastError();
    }
    if (B.pending && cudaEventQuery(B.ev) == cudaSuccess) {
      B.pending = false;
      plan_update(B, p_pad, cap);
      ++B.updates;
    }
    cudaGetLastError();  // cudaEventQuery's cudaErrorNotReady is not an error
    for (int b = 0; b <= B.nb; ++b) H.band_rows[b] = B.rows[b];
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    cudaStreamIsCapturing(st, &cs);
    measure = B.h_cyc && B.ev && !B.pending && B.updates <= kPlanUpdates && cs == cudaStreamCaptureStatusNone &&
              n >= kPlanMinRows;
    plan = &B;
  } else {
    H.nbands = make_bands(p_pad, cap, H.band_rows);
    H.groups = cov_groups(H.nbands, n);
  }
  H.idx = idx;
  H.val = val;
  H.n = n;
  H.m = m;
  H.p_pad = p_pad;
  H.stats = stats;
  H.tri = tri;
  H.part = reinterpret_cast<unsigned long long*>(ws);
  if (measure) H.cyc = H.part + (size_t)H.groups * tri_off(p_pad, p_pad);
  H.aligned = (reinterpret_cast<uintptr_t>(idx) % 16 == 0) && (reinterpret_cast<uintptr_t>(val) % 16 == 0);
  const int64_t total = tri_off(p_pad, p_pad);
  cudaMemsetAsync(ws, 0, (size_t)H.groups * total * 8, st);
  int maxe = 0, maxr = 0;
  for (int b = 0; b < H.nbands; ++b) {
    const int e = (int)(tri_off(H.band_rows[b + 1], p_pad) - tri_off(H.band_rows[b], p_pad));
    if (e > maxe) maxe = e;
    if (H.band_rows[b + 1] - H.band_rows[b] > maxr) maxr = H.band_rows[b + 1] - H.band_rows[b];
  }
  const size_t smem = flat ? (size_t)((maxe + 1) & ~1) * 4 + flat_ptab_bytes(m) + (size_t)kCovWarps * m * 8
                           : (size_t)((maxe + 1) & ~1) * 4 + (size_t)((maxr + 1) & ~1) * 4 + pair_table_bytes(m) +
                                 (size_t)kCovWarps * m * 16;
  const bool pk = p_pad <= 2048;  // the packed U.x of the flat kernel
  auto flat_kernel = [&](auto v) {
    using V = decltype(v);
    return pk ? (measure ? cov_flat_kernel<V, true, true> : cov_flat_kernel<V, true, false>)
              : (measure ? cov_flat_kernel<V, false, true> : cov_flat_kernel<V, false, false>);
  };
  auto k = val_f64 ? (m > 64 ? cov_band_kernel<double, true> : flat ? flat_kernel(double()) : cov_band_kernel<double, false>)
                   : (m > 64 ? cov_band_kernel<float, true> : flat ? flat_kernel(float()) : cov_band_kernel<float, false>);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (measure) cov_stamp_kernel<<<1, 1, 0, st>>>(H.cyc + (size_t)H.nbands * H.groups);
  k<<<H.nbands * H.groups, kCovWarps * 32, smem, st>>>(H);
  int rc = check_launch("cov_band_kernel");
  if (rc) return rc;
  if (measure) {
    std::lock_guard<std::mutex> lk(g_plan_mu);
    plan->groups = H.groups;
    plan->n_meas = n;
    if (cudaMemcpyAsync(plan->h_cyc, H.cyc, ((size_t)H.nbands * H.groups + 1) * 8, cudaMemcpyDeviceToHost, st) == cudaSuccess &&
        cudaEventRecord(plan->ev, st) == cudaSuccess)
      plan->pending = true;
    cudaGetLastError();
  }
  cov_reduce_kernel<<<(unsigned)((total + 255) / 256), 256, 0, st>>>(H.part, H.groups, total, m, stats, tri);
  return check_launch("cov_reduce_kernel");
}

int cov_launch(const int32_t* idx, const void* val, int val_f64, int64_t n, int32_t m, int32_t p_pad,
               const double* stats, double* tri, void* ws, cudaStream_t st) {
  if (n == 0) return SKC_OK;
  // path: banded shared-memory accumulation, or (many bands) the L2-resident global path
  const char path = cov_path(m, p_pad, n);
  if (path == 't') return covtc_launch(idx, val, val_f64, n, m, p_pad, stats, tri, ws, st);
  if (path == 'g') return cov_launch_global(idx, val, val_f64, n, m, p_pad, stats, tri, ws, st);
  // the kernel addresses a group's rows with 32-bit element offsets: split huge inputs
  const int ga = cov_groups(band_count(p_pad, m, n), n), gb = cov_groups(band_count(p_pad, m, 0), n);
  const int groups = ga < gb ? ga : gb;
  int64_t max_rows = (int64_t)groups * ((((int64_t)1 << 31) / m) - kCovWarps);
  if (const char* e = getenv("SKC_COV_SPLIT_ROWS")) max_rows = atoll(e) > 0 ? atoll(e) : max_rows;  // tests
  const size_t vsz = val_f64 ? 8 : 4;
  for (int64_t r0 = 0; r0 < n; r0 += max_rows) {
    const int64_t c = n - r0 < max_rows ? n - r0 : max_rows;
    const int rc = cov_launch_part(idx + r0 * m, static_cast<const char*>(val) + (size_t)(r0 * m) * vsz, val_f64, c,
                                   m, p_pad, stats, tri, ws, st);
    if (rc) return rc;
  }
  return SKC_OK;
}

// ======================================================================================
// K4: estimators.py:62-65 on the packed triangle
// ======================================================================================
__global__ void cov_finalize_kernel(const double* __restrict__ tri, int32_t p, double f, double dfac,
                                    double* __restrict__ C) {
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= (int64_t)p * p) return;
  const int a = (int)(e / p), b = (int)(e % p);
  const int lo = min(a, b), hi = max(a, b);
  const double c = dmul(tri[tri_off(lo, p) + (hi - lo)], f);
  C[e] = (a == b) ? dmul(c, dfac) : c;
}

int cov_finalize_launch(const double* tri, int32_t p_pad, int32_t m, int64_t n_total, double* C, cudaStream_t st) {
  // (p * (p - 1)) / (m * (m - 1)) / n  and  1.0 - (p - m) / (p - 1), evaluated as Python does
  const double f = ((double)((int64_t)p_pad * (p_pad - 1)) / (double)((int64_t)m * (m - 1))) / (double)n_total;
  const double dfac = 1.0 - (double)(p_pad - m) / (double)(p_pad - 1);
  const int64_t total = (int64_t)p_pad * p_pad;
  cov_finalize_kernel<<<(unsigned)((total + 255) / 256), 256, 0, st>>>(tri, p_pad, f, dfac, C);
  return check_launch("cov_finalize_kernel");
}

// ======================================================================================
// K7: adjoint D^T H^T per row, fp64, reference stage order (transform.py:92-110, 192-200).
// One CTA per row, the row staged in shared memory. pre_scale != 0 first maps
// y <- (pre_scale * y) / pre_div (the estimate_mean scaling, estimators.py:44).
// ======================================================================================
__global__ void adjoint_kernel(const double* __restrict__ Y, int32_t p_pad, int use_signs, uint64_t sign_state,
                               int32_t p_out, double pre_scale, double pre_div, double* __restrict__ X) {
  extern __shared__ double b[];
  const int64_t row = blockIdx.x;
  for (int j = threadIdx.x; j < p_pad; j += blockDim.x) {
    double v = Y[row * p_pad + j];
    if (pre_scale != 0.0) v = __ddiv_rn(dmul(pre_scale, v), pre_div);
    b[j] = v;
  }
  __syncthreads();
  for (int h = 1; h < p_pad; h <<= 1) {
    for (int q = threadIdx.x; q < p_pad / 2; q += blockDim.x) {
      const int i = (q / h) * 2 * h + (q % h);
      const double u = b[i], v = b[i + h];
      b[i] = dadd(u, v);
      b[i + h] = dsub(u, v);
    }
    __syncthreads();
  }
  const double c = 1.0 / sqrt((double)p_pad);
  for (int j = threadIdx.x; j < p_out; j += blockDim.x) {
    double v = dmul(b[j], c);
    if (use_signs) {
      const uint64_t bit = mix64(sign_state + kGamma * (uint64_t)(j + 1)) >> 63;
      v = dmul(v, 1.0 - 2.0 * (double)bit);
    }
    X[row * p_out + j] = v;
  }
}

// identity kind: copy with truncation and optional pre-scaling
__global__ void copy_rows_kernel(const double* __restrict__ Y, int64_t n, int32_t p_pad, int32_t p_out,
                                 double pre_scale, double pre_div, double* __restrict__ X) {
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= n * p_out) return;
  const int64_t r = e / p_out;
  const int j = (int)(e % p_out);
  double v = Y[r * p_pad + j];
  if (pre_scale != 0.0) v = __ddiv_rn(dmul(pre_scale, v), pre_div);
  X[e] = v;
}

int adjoint_launch(const double* Y, int64_t n, int32_t p_pad, int32_t kind, uint64_t sign_seed, int32_t p_out,
                   double pre_scale, double pre_div, double* X, cudaStream_t st) {
  if (n == 0) return SKC_OK;
  if (kind < 0) {  // plain WHT, no signs
    const size_t smem = (size_t)p_pad * sizeof(double);
    cudaFuncSetAttribute(adjoint_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    adjoint_kernel<<<(unsigned)n, 256, smem, st>>>(Y, p_pad, 0, 0, p_out, 0.0, 1.0, X);
    return check_launch("adjoint_kernel");
  }
  if (kind == SKC_KIND_NONE) {
    const int64_t tot = n * p_out;
    copy_rows_kernel<<<(unsigned)((tot + 255) / 256), 256, 0, st>>>(Y, n, p_pad, p_out, pre_scale, pre_div, X);
    return check_launch("copy_rows_kernel");
  }
  const size_t smem = (size_t)p_pad * sizeof(double);
  cudaFuncSetAttribute(adjoint_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  adjoint_kernel<<<(unsigned)n, 256, smem, st>>>(Y, p_pad, 1, mix64(sign_seed ^ kTagSign), p_out, pre_scale,
                                                 pre_div, X);
  return check_launch("adjoint_kernel");
}

// D diagonal as fp64 (transform.py:71-82)
__global__ void signs_kernel(uint64_t sign_state, int32_t p_pad, int use_signs, double* out) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= p_pad) return;
  out[j] = use_signs ? 1.0 - 2.0 * (double)(mix64(sign_state + kGamma * (uint64_t)(j + 1)) >> 63) : 1.0;
}

int signs_launch(uint64_t sign_seed, int32_t p_pad, int32_t kind, double* out, cudaStream_t st) {
  signs_kernel<<<(p_pad + 255) / 256, 256, 0, st>>>(mix64(sign_seed ^ kTagSign), p_pad, kind == SKC_KIND_HADAMARD,
                                                   out);
  return check_launch("signs_kernel");
}

}  // namespace skc
