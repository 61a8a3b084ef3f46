// K1: fused single-pass precondition + sparsify (sketch.py:196-223) for sm_100a.
//
// One CTA (8 warps) streams tiles of S = 8192 / p_pad samples:
//   phase 1  coalesced vector loads of the tile -> XOR-swizzled shared memory (zero pad)
//   phase 2  signs + normalised WHT. Each thread owns E = 32 elements of one sample
//            (L = p_pad/32 threads per sample). Butterfly stages run in registers
//            inside a 5-bit "window" of the element index. Windows are changed by a
//            conflict-free transpose through the swizzled tile. Stages run in the
//            reference order h = 1, 2, 4, ... (transform.py:162-169), so the fp64
//            instantiation is bit-exact.
//   phase 3  one warp per sample: splitmix64 keys of all p_pad coordinates, a
//            threshold prefilter into a per-warp candidate list, then an exact bucket
//            select of the m smallest keys (sketch.py:53-56). Kept (index, value) pairs
//            are written in ascending index order with coalesced stores.
#include <math.h>

#include "common.cuh"

namespace skc {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr int kTileElems = 8192;
constexpr uint32_t kFull = 0xFFFFFFFFu;

enum SampleMode { kSelect = 0, kFullSet = 1, kSlowExact = 2, kNoSample = 3 };

struct SketchParams {
  const void* X;
  int64_t ld, n;
  int32_t p, m;
  int32_t pk;          // key range of the sampling plan (plan.p; = p_pad except kind none)
  int32_t x_f64;       // input dtype
  int32_t vec;         // 1: rows allow aligned vector loads
  uint64_t sign_state; // mix64(sign_seed ^ TAG_SIGN), used when use_signs
  int32_t use_signs;
  uint64_t s_tag;      // mix64(master ^ TAG_SAMPLE)
  int64_t col0;
  int32_t* idx_out;
  void* val_out;
  int32_t val_f64;
  double* y_out;       // optional full transformed rows (n, p_pad) fp64
  uint32_t t_lim;      // candidate iff (key >> 32) <= t_lim
  int32_t cap;         // per-warp candidate capacity (multiple of 32)
  int32_t mode;        // SampleMode
  int64_t num_tiles;
};

template <int LOGP>
struct Geo {
  static constexpr int P = 1 << LOGP;
  static constexpr int LOGE = LOGP < 5 ? LOGP : 5;
  static constexpr int E = 1 << LOGE;
  static constexpr int L = P / E;  // threads per sample
  static constexpr int S = kTileElems / P;
  static constexpr int NWIN = LOGE == 0 ? 1 : (LOGP + LOGE - 1) / LOGE;
  static constexpr int ITEMS = S * L;  // (sample, thread) work items per tile
  // conflict-free XOR swizzle inside each 32-element block ("K1 layout")
  static __device__ __forceinline__ int phys(int s, int i) {
    if constexpr (LOGP < 5) {
      return s * P + i;
    } else {
      return s * P + (i ^ (((i >> 5) ^ (s * L)) & 31));
    }
  }
  static __device__ __forceinline__ int elem(int k, int u, int e) {
    const int bk = (k * LOGE < LOGP - LOGE) ? k * LOGE : LOGP - LOGE;
    const int low = (1 << bk) - 1;
    return (u & low) | (e << bk) | ((u >> bk) << (bk + LOGE));
  }
};

// ------------------------------------------------------------------------------------
// phase 2: WHT of one window for one (sample, thread) item
template <int LOGP, typename T, int K>
__device__ __forceinline__ void wht_window(T* xs, const uint32_t* sgn, int s, int u, T scale) {
  using G = Geo<LOGP>;
  using A = Arith<T>;
  constexpr int bk = (K * G::LOGE < LOGP - G::LOGE) ? K * G::LOGE : LOGP - G::LOGE;
  constexpr int first = K * G::LOGE;  // first stage bit not yet applied
  T v[G::E];
#pragma unroll
  for (int e = 0; e < G::E; ++e) v[e] = xs[G::phys(s, G::elem(K, u, e))];
  if constexpr (K == 0) {
    if (sgn != nullptr) {
      // window 0 holds elements [u*E, u*E + E): E consecutive bits of the sign mask
      const int base = u * G::E;
      const uint32_t bits = sgn[base >> 5] >> (base & 31);
#pragma unroll
      for (int e = 0; e < G::E; ++e) v[e] = A::flip(v[e], (bits >> e) & 1u);
    }
  }
#pragma unroll
  for (int b = first; b < bk + G::LOGE; ++b) {
    const int h = 1 << (b - bk);
#pragma unroll
    for (int e = 0; e < G::E; ++e) {
      if ((e & h) == 0) {
        const T a = v[e], c = v[e + h];
        v[e] = A::add(a, c);
        v[e + h] = A::sub(a, c);
      }
    }
  }
  if constexpr (K == G::NWIN - 1) {
#pragma unroll
    for (int e = 0; e < G::E; ++e) v[e] = A::mul(v[e], scale);
  }
#pragma unroll
  for (int e = 0; e < G::E; ++e) xs[G::phys(s, G::elem(K, u, e))] = v[e];
}

template <int LOGP, typename T, int K>
__device__ __forceinline__ void wht_all_windows(T* xs, const uint32_t* sgn, T scale) {
  using G = Geo<LOGP>;
  if constexpr (K < G::NWIN) {
    for (int it = threadIdx.x; it < G::ITEMS; it += kThreads) {
      const int s = it / G::L, u = it % G::L;
      wht_window<LOGP, T, K>(xs, sgn, s, u, scale);
    }
    __syncthreads();
    wht_all_windows<LOGP, T, K + 1>(xs, sgn, scale);
  }
}

// ------------------------------------------------------------------------------------
// phase 3 helpers
__device__ __forceinline__ uint64_t key_of(uint64_t ci, int j) {
  return mix64(ci + kGamma * (uint64_t)(j + 1));
}

template <typename T>
__device__ __forceinline__ void store_val(void* out, int64_t pos, T v, int val_f64) {
  if (val_f64) reinterpret_cast<double*>(out)[pos] = (double)v;
  else reinterpret_cast<float*>(out)[pos] = (float)v;
}

// Exact fallback: binary search the m-th smallest key by re-hashing (64 passes). Used
// only when the prefilter misses (probability ~1e-7 per sample) or cap would overflow.
template <int LOGP, typename T>
__device__ void emit_slow_exact(const SketchParams& P, const T* xs, int s, int64_t row, uint64_t ci) {
  using G = Geo<LOGP>;
  const int lane = threadIdx.x & 31;
  uint64_t lo = 0, hi = ~0ull;
  while (lo < hi) {
    const uint64_t mid = lo + ((hi - lo) >> 1);
    int c = 0;
    for (int j = lane; j < P.pk; j += 32) c += key_of(ci, j) <= mid;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(kFull, c, o);
    if (c >= P.m) hi = mid;
    else lo = mid + 1;
  }
  int base = 0;
  for (int j0 = 0; j0 < P.pk; j0 += 32) {
    const int j = j0 + lane;
    const bool keep = j < P.pk && key_of(ci, j) <= lo;
    const uint32_t bal = __ballot_sync(kFull, keep);
    if (keep) {
      const int64_t pos = row * P.m + base + __popc(bal & lanemask_lt());
      P.idx_out[pos] = j;
      if (P.val_out) store_val<T>(P.val_out, pos, xs[G::phys(s, j)], P.val_f64);
    }
    base += __popc(bal);
  }
}

template <int LOGP, typename T>
__device__ void sample_one(const SketchParams& P, const T* xs, int s, int64_t row, uint64_t* ck, uint16_t* cj,
                           uint64_t* memk, int* hist) {
  using G = Geo<LOGP>;
  const int lane = threadIdx.x & 31;
  if (P.mode == kFullSet) {  // m == p: SamplingPlan shortcut, sketch.py:51-52
    for (int j = lane; j < P.pk; j += 32) {
      const int64_t pos = row * P.m + j;
      P.idx_out[pos] = j;
      if (P.val_out) store_val<T>(P.val_out, pos, xs[G::phys(s, j)], P.val_f64);
    }
    return;
  }
  const uint64_t ci = mix64(P.s_tag + kGamma * (uint64_t)(P.col0 + row + 1));  // _hash.py:54
  if (P.mode == kSlowExact) {
    emit_slow_exact<LOGP, T>(P, xs, s, row, ci);
    return;
  }
  // 1. prefilter: candidates in ascending j order
  int count = 0;
  uint64_t kin = ci + kGamma * (uint64_t)(lane + 1);
#pragma unroll 4
  for (int j0 = 0; j0 < P.pk; j0 += 32) {
    const int j = j0 + lane;
    const uint64_t key = mix64(kin);
    kin += 32ull * kGamma;
    const bool cand = (j < P.pk) && ((uint32_t)(key >> 32) <= P.t_lim);
    const uint32_t bal = __ballot_sync(kFull, cand);
    if (cand) {
      const int pos = count + __popc(bal & lanemask_lt());
      if (pos < P.cap) {
        ck[pos] = key;
        cj[pos] = (uint16_t)j;
      }
    }
    count += __popc(bal);
  }
  if (count < P.m || count > P.cap) {
    __syncwarp();
    emit_slow_exact<LOGP, T>(P, xs, s, row, ci);
    return;
  }
  __syncwarp();
  // 2. exact select of the m smallest keys: 32 key-monotone buckets, then rank inside
  //    the bucket that holds the m-th smallest
  uint64_t kth = ~0ull;
  if (count > P.m) {
    hist[lane] = 0;
    __syncwarp();
    const float bscale = 32.0f / ((float)P.t_lim + 1.0f);
    for (int q = lane; q < count; q += 32) {
      const int b = min(31, (int)((float)(uint32_t)(ck[q] >> 32) * bscale));
      atomicAdd(&hist[b], 1);
    }
    __syncwarp();
    const int h = hist[lane];
    int incl = h;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int t = __shfl_up_sync(kFull, incl, o);
      if (lane >= o) incl += t;
    }
    const int B = __ffs(__ballot_sync(kFull, incl >= P.m)) - 1;
    const int hB = __shfl_sync(kFull, h, B);
    const int r = P.m - __shfl_sync(kFull, incl - h, B);  // keep the r smallest of bucket B
    if (hB > 32) {
      emit_slow_exact<LOGP, T>(P, xs, s, row, ci);
      return;
    }
    int nb = 0;
    for (int q0 = 0; q0 < count; q0 += 32) {
      const int q = q0 + lane;
      bool in = false;
      uint64_t key = 0;
      if (q < count) {
        key = ck[q];
        in = min(31, (int)((float)(uint32_t)(key >> 32) * bscale)) == B;
      }
      const uint32_t bal = __ballot_sync(kFull, in);
      if (in) memk[nb + __popc(bal & lanemask_lt())] = key;
      nb += __popc(bal);
    }
    __syncwarp();
    const uint64_t mine = lane < hB ? memk[lane] : ~0ull;
    int rank = 0;
    for (int o = 0; o < hB; ++o) {
      const uint64_t other = __shfl_sync(kFull, mine, o);
      rank += other < mine;
    }
    const uint32_t hit = __ballot_sync(kFull, lane < hB && rank == r - 1);
    kth = __shfl_sync(kFull, mine, __ffs(hit) - 1);
  }
  // 3. emit kept coordinates in ascending order (candidates are already j-sorted)
  int base = 0;
  for (int q0 = 0; q0 < count; q0 += 32) {
    const int q = q0 + lane;
    const bool keep = q < count && ck[q] <= kth;
    const uint32_t bal = __ballot_sync(kFull, keep);
    if (keep) {
      const int j = cj[q];
      const int64_t pos = row * P.m + base + __popc(bal & lanemask_lt());
      P.idx_out[pos] = j;
      if (P.val_out) store_val<T>(P.val_out, pos, xs[G::phys(s, j)], P.val_f64);
    }
    base += __popc(bal);
  }
  __syncwarp();
}

// ------------------------------------------------------------------------------------
template <int LOGP, typename T>
__global__ void __launch_bounds__(kThreads) sketch_kernel(const SketchParams P) {
  using G = Geo<LOGP>;
  extern __shared__ __align__(16) unsigned char smem[];
  T* xs = reinterpret_cast<T*>(smem);
  uint32_t* sgn = reinterpret_cast<uint32_t*>(smem + sizeof(T) * kTileElems);
  constexpr int kSignWords = (G::P + 31) / 32;
  unsigned char* wbase = smem + sizeof(T) * kTileElems + 4 * ((kSignWords + 3) & ~3);
  const int warp = threadIdx.x >> 5;
  const size_t per_warp = (size_t)P.cap * 10 + 32 * 8 + 32 * 4;
  unsigned char* mine = wbase + per_warp * warp;
  uint64_t* ck = reinterpret_cast<uint64_t*>(mine);
  uint64_t* memk = reinterpret_cast<uint64_t*>(mine + (size_t)P.cap * 8);
  int* hist = reinterpret_cast<int*>(mine + (size_t)P.cap * 8 + 256);
  uint16_t* cj = reinterpret_cast<uint16_t*>(mine + (size_t)P.cap * 8 + 256 + 128);

  const bool has_x = P.X != nullptr;
  if (has_x && P.use_signs) {  // D diagonal, _hash.py:38-43, regenerated per CTA
    for (int w = threadIdx.x; w < kSignWords; w += kThreads) {
      uint32_t bits = 0;
      for (int b = 0; b < 32 && w * 32 + b < G::P; ++b) {
        const int j = w * 32 + b;
        bits |= (uint32_t)(mix64(P.sign_state + kGamma * (uint64_t)(j + 1)) >> 63) << b;
      }
      sgn[w] = bits;
    }
  }
  const T scale = (T)(1.0 / sqrt((double)G::P));  // transform.py:170

  for (int64_t tile = blockIdx.x; tile < P.num_tiles; tile += gridDim.x) {
    const int64_t row0 = tile * G::S;
    __syncthreads();  // previous tile's phase 3 done with xs; signs visible
    if (has_x) {
      // ---- phase 1: load (zero pad p..p_pad and rows >= n) ----
      if (P.vec && !P.x_f64) {
        constexpr int NV = kTileElems / 4 / kThreads;
        float4 buf[NV];
#pragma unroll
        for (int k = 0; k < NV; ++k) {
          const int f = (threadIdx.x + k * kThreads) * 4;
          const int s = f >> LOGP, i = f & (G::P - 1);
          const int64_t row = row0 + s;
          buf[k] = row < P.n ? __ldg(reinterpret_cast<const float4*>(reinterpret_cast<const float*>(P.X) +
                                                                    row * P.ld + i))
                             : make_float4(0.f, 0.f, 0.f, 0.f);
        }
#pragma unroll
        for (int k = 0; k < NV; ++k) {
          const int f = (threadIdx.x + k * kThreads) * 4;
          const int s = f >> LOGP, i = f & (G::P - 1);
          xs[G::phys(s, i + 0)] = (T)buf[k].x;
          xs[G::phys(s, i + 1)] = (T)buf[k].y;
          xs[G::phys(s, i + 2)] = (T)buf[k].z;
          xs[G::phys(s, i + 3)] = (T)buf[k].w;
        }
      } else {
        for (int f = threadIdx.x; f < kTileElems; f += kThreads) {
          const int s = f >> LOGP, i = f & (G::P - 1);
          const int64_t row = row0 + s;
          T v = (T)0;
          if (row < P.n && i < P.p) {
            v = P.x_f64 ? (T)__ldg(reinterpret_cast<const double*>(P.X) + row * P.ld + i)
                        : (T)__ldg(reinterpret_cast<const float*>(P.X) + row * P.ld + i);
          }
          xs[G::phys(s, i)] = v;
        }
      }
      __syncthreads();
      // ---- phase 2: D then WHT then scale ----
      wht_all_windows<LOGP, T, 0>(xs, P.use_signs ? sgn : nullptr, scale);
      if (P.y_out) {
        for (int f = threadIdx.x; f < kTileElems; f += kThreads) {
          const int s = f >> LOGP, i = f & (G::P - 1);
          const int64_t row = row0 + s;
          if (row < P.n) P.y_out[row * G::P + i] = (double)xs[G::phys(s, i)];
        }
      }
    }
    // ---- phase 3: sample + emit, one warp per sample ----
    if (P.mode != kNoSample) {
      for (int s = warp; s < G::S; s += kWarps) {
        const int64_t row = row0 + s;
        if (row >= P.n) break;
        sample_one<LOGP, T>(P, xs, s, row, ck, cj, memk, hist);
      }
    }
  }
}

// ------------------------------------------------------------------------------------
template <int LOGP, typename T>
static int launch_sketch_t(SketchParams P, cudaStream_t st) {
  using G = Geo<LOGP>;
  const size_t sign_bytes = 4 * (((G::P + 31) / 32 + 3) & ~3);
  const size_t per_warp = (size_t)P.cap * 10 + 32 * 8 + 32 * 4;
  const size_t smem = sizeof(T) * kTileElems + sign_bytes + per_warp * kWarps;
  auto kern = sketch_kernel<LOGP, T>;
  if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
    return check_launch("sketch smem attribute");
  int occ = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, kThreads, smem);
  if (occ < 1) occ = 1;
  P.num_tiles = (P.n + G::S - 1) / G::S;
  int64_t grid = (int64_t)sm_count() * occ;
  if (grid > P.num_tiles) grid = P.num_tiles;
  if (grid < 1) return SKC_OK;
  kern<<<(unsigned)grid, kThreads, smem, st>>>(P);
  return check_launch("sketch_kernel");
}

template <typename T>
static int launch_sketch_logp(int logp, const SketchParams& P, cudaStream_t st) {
  switch (logp) {
    case 0: return launch_sketch_t<0, T>(P, st);
    case 1: return launch_sketch_t<1, T>(P, st);
    case 2: return launch_sketch_t<2, T>(P, st);
    case 3: return launch_sketch_t<3, T>(P, st);
    case 4: return launch_sketch_t<4, T>(P, st);
    case 5: return launch_sketch_t<5, T>(P, st);
    case 6: return launch_sketch_t<6, T>(P, st);
    case 7: return launch_sketch_t<7, T>(P, st);
    case 8: return launch_sketch_t<8, T>(P, st);
    case 9: return launch_sketch_t<9, T>(P, st);
    case 10: return launch_sketch_t<10, T>(P, st);
    case 11: return launch_sketch_t<11, T>(P, st);
    case 12: return launch_sketch_t<12, T>(P, st);
  }
  return fail(SKC_EPARAM, "p_pad exceeds the largest instantiated transform (4096)");
}

// Host: prefilter threshold and candidate capacity for (p_pad, m)
static void plan_select(int32_t p_pad, int32_t m, SketchParams& P) {
  if (m == p_pad) {
    P.mode = kFullSet;
    P.cap = 32;
    P.t_lim = 0xFFFFFFFFu;
    return;
  }
  const double mu = m + 5.0 * sqrt((double)m) + 8.0;  // expected candidates (mean - 5 sigma >= m)
  if (mu >= 0.5 * p_pad) {
    P.t_lim = 0xFFFFFFFFu;  // every coordinate is a candidate
    P.cap = (p_pad + 31) & ~31;
  } else {
    double t = floor(mu / p_pad * 4294967296.0) - 1.0;
    P.t_lim = (uint32_t)t;
    double cap = mu + 6.0 * sqrt(mu) + 32.0;
    P.cap = ((int)cap + 31) & ~31;
  }
  P.mode = kSelect;
  if (P.cap > 1024) {
    P.mode = kSlowExact;
    P.cap = 32;
  }
}

int sketch_launch(const void* X, int32_t x_dtype, int64_t ld, int64_t n, int32_t p, int32_t p_pad, int32_t kind,
                  uint64_t sign_seed, uint64_t master_seed, int64_t col0, int32_t m, int32_t compute_dtype,
                  int32_t* idx_out, void* val_out, int32_t val_dtype, double* y_out, cudaStream_t st) {
  SketchParams P{};
  P.X = X;
  P.ld = ld;
  P.n = n;
  P.p = p;
  P.m = m;
  P.pk = p_pad;
  P.x_f64 = x_dtype == SKC_F64;
  P.use_signs = kind == SKC_KIND_HADAMARD;
  P.sign_state = mix64(sign_seed ^ kTagSign);
  P.s_tag = mix64(master_seed ^ kTagSample);
  P.col0 = col0;
  P.idx_out = idx_out;
  P.val_out = val_out;
  P.val_f64 = val_dtype == SKC_F64;
  P.y_out = y_out;
  int logp = 0;
  while ((1 << logp) < p_pad) ++logp;  // transform template; the sampler uses pk = p_pad
  const uintptr_t xa = reinterpret_cast<uintptr_t>(X);
  P.vec = X != nullptr && p == p_pad && p_pad >= 4 && (ld % 4) == 0 && (xa % 16) == 0;
  if (idx_out == nullptr) {
    P.mode = kNoSample;
    P.cap = 32;
  } else {
    plan_select(p_pad, m, P);
  }
  if (kind == SKC_KIND_NONE && X != nullptr) {
    // identity transform: no signs, no WHT, no scale (transform.py:225-227)
    return fail(SKC_EPARAM, "internal: kind none is routed through sketch_identity");
  }
  if (compute_dtype == SKC_F64) return launch_sketch_logp<double>(logp, P, st);
  return launch_sketch_logp<float>(logp, P, st);
}

// kind == none: values are the raw (zero-padded) coordinates. Reuses the sampler with a
// gather kernel instead of the transform.
__global__ void gather_identity_kernel(const void* X, int x_f64, int64_t ld, int64_t n, int32_t p, int32_t m,
                                       const int32_t* idx, void* val_out, int val_f64, double* y_out,
                                       int32_t p_pad) {
  const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (val_out != nullptr && tid < n * m) {
    const int64_t row = tid / m;
    const int j = idx[tid];
    double v = 0.0;
    if (j < p) v = x_f64 ? reinterpret_cast<const double*>(X)[row * ld + j]
                         : (double)reinterpret_cast<const float*>(X)[row * ld + j];
    if (val_f64) reinterpret_cast<double*>(val_out)[tid] = v;
    else reinterpret_cast<float*>(val_out)[tid] = (float)v;
  }
  if (y_out != nullptr && tid < n * p_pad) {
    const int64_t row = tid / p_pad;
    const int j = (int)(tid % p_pad);
    double v = 0.0;
    if (j < p) v = x_f64 ? reinterpret_cast<const double*>(X)[row * ld + j]
                         : (double)reinterpret_cast<const float*>(X)[row * ld + j];
    y_out[tid] = v;
  }
}

int sketch_identity(const void* X, int32_t x_dtype, int64_t ld, int64_t n, int32_t p, int32_t p_pad,
                    uint64_t master_seed, int64_t col0, int32_t m, int32_t* idx_out, void* val_out,
                    int32_t val_dtype, double* y_out, cudaStream_t st) {
  if (idx_out != nullptr) {
    int rc = sketch_launch(nullptr, x_dtype, ld, n, p, p_pad, SKC_KIND_HADAMARD, 0, master_seed, col0, m, SKC_F32,
                           idx_out, nullptr, val_dtype, nullptr, st);
    if (rc != SKC_OK) return rc;
  }
  const int64_t wv = val_out != nullptr ? n * m : 0, wy = y_out != nullptr ? n * p_pad : 0;
  const int64_t work = wv > wy ? wv : wy;
  if (work == 0) return SKC_OK;
  const int64_t blocks = (work + 255) / 256;
  gather_identity_kernel<<<(unsigned)blocks, 256, 0, st>>>(X, x_dtype == SKC_F64, ld, n, p, m, idx_out, val_out,
                                                           val_dtype == SKC_F64, y_out, p_pad);
  return check_launch("gather_identity_kernel");
}

}  // namespace skc
