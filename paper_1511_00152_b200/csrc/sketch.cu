// K1: fused single-pass precondition + sparsify (sketch.py:196-223) for sm_100a.
//
// A CTA (8 warps) streams tiles of S = 8192 / P samples (P = 2^LOGP = p_pad):
//   phase 1  coalesced 16-byte loads of the tile into a padded shared-memory layout:
//            element i of sample s sits at word  s*SP + (i>>5)*33 + (i&31),  SP=(P/32)*33.
//            That address is linear over disjoint index bits, so every register of a
//            window below is "thread base + immediate". The 33-word rows make every
//            window conflict-free, including windows whose lanes span several samples.
//   phase 2  signs + normalised WHT. A thread owns E = 32 elements of one sample (a
//            5-bit "window" of the index bits); butterfly stages run in registers;
//            windows change through the tile. Stages run in the reference order
//            h = 1, 2, 4, ... (transform.py:101-108), so the fp64 instantiation is
//            bit-exact.
//   phase 3  one warp per sample. Pass 1 hashes all keys of the plan (splitmix64,
//            _hash.py:46-56) and keeps the high word only for a threshold test, as a
//            per-lane bitmask. Pass 2 re-hashes the ~m+5sqrt(m) candidates in full into
//            a per-warp list. An exact bucket select finds the m smallest keys
//            (sketch.py:53-56); the kept set becomes a row bitmask, and each lane emits
//            its rows' elements at prefix-sum slots in ascending index order.
#include <math.h>
#include <stdlib.h>

#include <type_traits>

#include "common.cuh"

namespace skc {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr int kTileElems = 8192;
constexpr uint32_t kFull = 0xFFFFFFFFu;

enum SampleMode { kSelect = 0, kFullSet = 1, kSlowExact = 2, kNoSample = 3, kGiven = 4 };

struct SketchParams {
  const void* X;
  int64_t ld, n;
  int32_t p, m;
  int32_t pk;          // key range of the sampling plan (plan.p; = p_pad except kind none)
  int32_t x_f64;       // input dtype
  int32_t vec;         // 1: rows allow aligned 16-byte loads
  uint64_t sign_state; // mix64(sign_seed ^ TAG_SIGN), used when use_signs
  int32_t use_signs;
  uint64_t s_tag;      // mix64(master ^ TAG_SAMPLE)
  int64_t col0;
  int32_t* idx_out;
  const int32_t* idx_in;  // kGiven: the kept indices (n, m), sorted per row
  void* val_out;
  int32_t val_f64;
  double* y_out;       // optional full transformed rows (n, p_pad) fp64
  uint32_t t_hi;       // candidate iff (key >> 32) < t_hi  (t_all: every key)
  int32_t t_all;
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
  static constexpr int ITEMS = S * L;
  // Padded layout: each 32-element row of a sample takes 36 words, and consecutive samples
  // sit SP words apart with SP = 4 (mod 32). Rows start 16-byte aligned, so 4-element
  // groups move as single 16-byte copies and vector LDS/STS. Every window access below is
  // bank-conflict-free, including windows whose lanes span several samples.
  static constexpr int SP0 = LOGP < 5 ? P : (P / 32) * 36;
  static constexpr int SP = LOGP < 5 ? P : SP0 + ((4 - SP0 % 32) + 32) % 32;  // words per sample
  static constexpr int WORDS = S * SP;
  // padded address of element i (linear over disjoint bit sets of i)
  static __host__ __device__ constexpr int addr(int i) { return LOGP < 5 ? i : i + 4 * (i >> 5); }
  static __host__ __device__ constexpr int bk(int k) { return (k * LOGE < LOGP - LOGE) ? k * LOGE : LOGP - LOGE; }
  // the thread bits of window k: u fills every index bit outside [bk, bk+LOGE)
  static __device__ __forceinline__ int u_part(int k, int u) {
    const int b = bk(k);
    return (u & ((1 << b) - 1)) | ((u >> b) << (b + LOGE));
  }
};

// ------------------------------------------------------------------------------------
// packed fp32 pairs (sm_100 FADD2 / FMUL2)
__device__ __forceinline__ uint64_t pack2(float lo, float hi) {
  uint64_t r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
  return r;
}
__device__ __forceinline__ void unpack2(uint64_t x, float& lo, float& hi) {
  asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(x));
}
__device__ __forceinline__ uint64_t add2(uint64_t a, uint64_t b) {
  uint64_t r;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ uint64_t sub2(uint64_t a, uint64_t b) {
  uint64_t r;
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ uint64_t mul2(uint64_t a, uint64_t b) {
  uint64_t r;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}

// ------------------------------------------------------------------------------------
// phase 2: one window of the WHT for one (sample, thread) item
template <int LOGP, typename T, int K>
__device__ __forceinline__ void wht_window(T* xs, const uint32_t* sgn, int s, int u, T scale) {
  using G = Geo<LOGP>;
  using A = Arith<T>;
  constexpr int bk = G::bk(K);
  constexpr int first = K * G::LOGE;  // first stage bit not yet applied
  T* base = xs + s * G::SP + G::addr(G::u_part(K, u));
  T v[G::E];
  // window 0 of a padded layout reads E = 32 consecutive, 16-byte aligned elements
  using V16 = typename std::conditional<sizeof(T) == 4, float4, double2>::type;
  constexpr int PER = 16 / sizeof(T);
  constexpr bool kVec = bk == 0 && G::E == 32;
  if constexpr (kVec) {
#pragma unroll
    for (int c = 0; c < G::E / PER; ++c) {
      const V16 t = reinterpret_cast<const V16*>(base)[c];
      const T* tp = reinterpret_cast<const T*>(&t);
#pragma unroll
      for (int q = 0; q < PER; ++q) v[c * PER + q] = tp[q];
    }
  } else {
#pragma unroll
    for (int e = 0; e < G::E; ++e) v[e] = base[G::addr(e << bk)];
  }
  if constexpr (K == 0) {
    if (sgn != nullptr) {
      // window 0 holds elements [u*E, u*E + E): E consecutive bits of the sign mask
      const int b0 = u * G::E;
      const uint32_t bits = sgn[b0 >> 5] >> (b0 & 31);
#pragma unroll
      for (int e = 0; e < G::E; ++e) v[e] = A::flip(v[e], (bits >> e) & 1u);
    }
  }
  if constexpr (std::is_same<T, float>::value && G::E >= 4) {
    // fp32: stages with h >= 2 run on packed pairs (v[e], v[e+1]) with FADD2; each lane is
    // an IEEE add/sub/mul with round-to-nearest, so results equal the scalar order exactly
    uint64_t w[G::E / 2];
#pragma unroll
    for (int k = 0; k < G::E / 2; ++k) w[k] = pack2(v[2 * k], v[2 * k + 1]);
#pragma unroll
    for (int b = first; b < bk + G::LOGE; ++b) {
      const int h = 1 << (b - bk);
      if (h == 1) {
#pragma unroll
        for (int k = 0; k < G::E / 2; ++k) {
          float a, c;
          unpack2(w[k], a, c);
          w[k] = pack2(fadd(a, c), fsub(a, c));
        }
      } else {
        const int hp = h >> 1;
#pragma unroll
        for (int k = 0; k < G::E / 2; ++k) {
          if (((2 * k) & h) == 0) {
            const uint64_t x = w[k], y = w[k + hp];
            w[k] = add2(x, y);
            w[k + hp] = sub2(x, y);
          }
        }
      }
    }
    if constexpr (K == G::NWIN - 1) {
      const uint64_t sc = pack2(scale, scale);
#pragma unroll
      for (int k = 0; k < G::E / 2; ++k) w[k] = mul2(w[k], sc);
    }
#pragma unroll
    for (int k = 0; k < G::E / 2; ++k) unpack2(w[k], v[2 * k], v[2 * k + 1]);
  } else {
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
  }
  if constexpr (kVec) {
#pragma unroll
    for (int c = 0; c < G::E / PER; ++c) {
      V16 t;
      T* tp = reinterpret_cast<T*>(&t);
#pragma unroll
      for (int q = 0; q < PER; ++q) tp[q] = v[c * PER + q];
      reinterpret_cast<V16*>(base)[c] = t;
    }
  } else {
#pragma unroll
    for (int e = 0; e < G::E; ++e) base[G::addr(e << bk)] = v[e];
  }
}

template <int LOGP, typename T, int K>
__device__ __forceinline__ void wht_all_windows(T* xs, const uint32_t* sgn, T scale) {
  using G = Geo<LOGP>;
  if constexpr (K < G::NWIN) {
    for (int it = threadIdx.x; it < G::ITEMS; it += kThreads) wht_window<LOGP, T, K>(xs, sgn, it / G::L, it % G::L, scale);
    __syncthreads();
    wht_all_windows<LOGP, T, K + 1>(xs, sgn, scale);
  }
}

// ------------------------------------------------------------------------------------
// phase 3 helpers
// per-warp scratch: keys [cap] u64, bucket keys [32] u64, histogram [32], kept-row
// bitmask [P/32] u32, candidate indices [cap] u16 (16-byte multiple)
// The kept-set masks of all the warp's samples in a tile stay live from selection (before
// the transform) to emission (after it): max(P/32, 32) words for P >= 32.
template <int LOGP>
__host__ __device__ constexpr int mask_words() {
  return LOGP < 5 ? 1 : ((1 << LOGP) / 32 > 32 ? (1 << LOGP) / 32 : 32);
}
template <int LOGP>
__host__ __device__ constexpr size_t warp_bytes(int cap) {
  return ((size_t)cap * 10 + 256 + 128 + 4 * mask_words<LOGP>() + 15) & ~(size_t)15;
}
__device__ __forceinline__ uint64_t key_of(uint64_t ci, int j) { return mix64(ci + kGamma * (uint64_t)(j + 1)); }

// High 32 bits of mix64(z) before its last xor-shift: for t <= 2^31,
// (key >> 32) < t  <=>  hi32(z2) < t, because the last step only flips bit 0 of the high
// word when bit 63 is set. Skips the low word of the final product and shift.
__device__ __forceinline__ uint32_t mix64_hi_pre(uint64_t z) {
  z = (z ^ (z >> 30)) * kMix1;
  z = z ^ (z >> 27);
  return (uint32_t)((z * kMix2) >> 32);
}

template <typename T>
__device__ __forceinline__ void store_val(void* out, int64_t pos, T v, int val_f64) {
  if (val_f64) reinterpret_cast<double*>(out)[pos] = (double)v;
  else reinterpret_cast<float*>(out)[pos] = (float)v;
}

template <int LOGP, typename T>
__device__ __forceinline__ T y_at(const T* xs, int s, int j) {
  using G = Geo<LOGP>;
  return xs[s * G::SP + G::addr(j)];
}

// Exact fallback: binary search of the m-th smallest key by re-hashing (64 passes). Used
// only when the prefilter misses (~1e-7 per sample) or a bucket overflows.
template <int LOGP, typename T>
__device__ void emit_slow_exact(const SketchParams& P, const T* xs, int s, int64_t row, uint64_t ci) {
  const int lane = threadIdx.x & 31;
  uint64_t lo = 0, hi = ~0ull;
  while (lo < hi) {
    const uint64_t mid = lo + ((hi - lo) >> 1);
    int c = 0;
    for (int j = lane; j < P.pk; j += 32) c += key_of(ci, j) <= mid;
    c = __reduce_add_sync(kFull, c);
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
      if (P.val_out) store_val<T>(P.val_out, pos, y_at<LOGP, T>(xs, s, j), P.val_f64);
    }
    base += __popc(bal);
  }
}

__device__ __forceinline__ uint64_t column_state(const SketchParams& P, int64_t row) {
  return mix64(P.s_tag + kGamma * (uint64_t)(P.col0 + row + 1));  // _hash.py:54
}

// Selection for one sample (needs no sample data): sets the kept set in rmask, bit
// (j & 31) of word (j >> 5). Returns false when the sample must take the exact slow path.
template <int LOGP>
__device__ bool select_one(const SketchParams& P, int64_t row, uint64_t* ck, uint16_t* cj, uint64_t* memk,
                           int* hist, uint32_t* rmask) {
  const int lane = threadIdx.x & 31;
  const int rows = (P.pk + 31) >> 5;  // key rows: j = 32 r + lane
  if (P.mode == kFullSet) {  // m == p: SamplingPlan shortcut, sketch.py:51-52
    for (int r = lane; r < rows; r += 32) rmask[r] = P.pk - 32 * r >= 32 ? kFull : (1u << (P.pk - 32 * r)) - 1u;
    __syncwarp();
    return true;
  }
  if (P.mode == kSlowExact) return false;
  const uint64_t ci = column_state(P, row);
  constexpr int MW = (Geo<LOGP>::P + 1023) / 1024;  // mask words: bit r of word w <-> j = 32 (32 w + r) + lane
  // pass 1: threshold bitmask
  uint32_t cm[MW];
#pragma unroll
  for (int w = 0; w < MW; ++w) cm[w] = 0;
  if (P.t_all) {
#pragma unroll
    for (int w = 0; w < MW; ++w)
      for (int r = 0; r < 32; ++r) cm[w] |= (uint32_t)(32 * (32 * w + r) + lane < P.pk) << r;
  } else {
    uint64_t kin = ci + kGamma * (uint64_t)(lane + 1);
    const uint64_t step = 32ull * kGamma;
    if (P.pk == Geo<LOGP>::P && Geo<LOGP>::P >= 32) {
#pragma unroll
      for (int w = 0; w < MW; ++w) {
#pragma unroll
        for (int r = 0; r < (Geo<LOGP>::P >= 1024 ? 32 : Geo<LOGP>::P / 32); ++r) {
          const uint32_t h = mix64_hi_pre(kin);
          kin += step;
          if (h < P.t_hi) cm[w] |= 1u << r;
        }
      }
    } else {
#pragma unroll
      for (int w = 0; w < MW; ++w) {
        const int rw = min(32, rows - 32 * w);
#pragma unroll 8
        for (int r = 0; r < rw; ++r) {
          const uint32_t h = mix64_hi_pre(kin);
          kin += step;
          cm[w] |= (uint32_t)(h < P.t_hi && 32 * (32 * w + r) + lane < P.pk) << r;
        }
      }
    }
  }
  int mine = 0;
#pragma unroll
  for (int w = 0; w < MW; ++w) mine += __popc(cm[w]);
  int off = mine;  // inclusive scan -> exclusive offset
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int t = __shfl_up_sync(kFull, off, o);
    if (lane >= o) off += t;
  }
  const int count = __shfl_sync(kFull, off, 31);
  off -= mine;
  if (count < P.m || count > P.cap) return false;
  // pass 2: candidate indices (each lane fills its slots [off, off + mine)), then full keys
  // and the bucket histogram, lane-strided over the list
  {
    int q = off;
#pragma unroll
    for (int w = 0; w < MW; ++w)
      for (uint32_t b = cm[w]; b; b &= b - 1, ++q) cj[q] = (uint16_t)(32 * (32 * w + __ffs(b) - 1) + lane);
  }
  const bool sel = count > P.m;
  // 32 key-monotone buckets over [0, t_hi * 2^32)
  const float bscale = P.t_all ? 32.0f / 4294967296.0f : 32.0f / (float)P.t_hi;
  if (sel) hist[lane] = 0;
  __syncwarp();
  for (int q = lane; q < count; q += 32) {
    const uint64_t key = key_of(ci, cj[q]);
    ck[q] = key;
    if (sel) atomicAdd(&hist[min(31, (int)((float)(uint32_t)(key >> 32) * bscale))], 1);
  }
  __syncwarp();
  uint64_t kth = ~0ull;
  if (sel) {
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
    if (hB > 32) return false;
    int nb = 0;
    for (int q0 = 0; q0 < count; q0 += 32) {
      const int q = q0 + lane;
      uint64_t key = 0;
      bool in = false;
      if (q < count) {
        key = ck[q];
        in = min(31, (int)((float)(uint32_t)(key >> 32) * bscale)) == B;
      }
      const uint32_t bal = __ballot_sync(kFull, in);
      if (in) memk[nb + __popc(bal & lanemask_lt())] = key;
      nb += __popc(bal);
    }
    __syncwarp();
    const uint64_t mk = lane < hB ? memk[lane] : ~0ull;
    int rank = 0;
    for (int o = 0; o < hB; ++o) rank += __shfl_sync(kFull, mk, o) < mk;
    const uint32_t hit = __ballot_sync(kFull, lane < hB && rank == r - 1);
    kth = __shfl_sync(kFull, mk, __ffs(hit) - 1);
  }
  // kept set as a row bitmask: bit (j & 31) of word (j >> 5)
  for (int q = lane; q < count; q += 32) {
    const int j = cj[q];
    atomicOr(&rmask[j >> 5], (uint32_t)(ck[q] <= kth) << (j & 31));
  }
  __syncwarp();
  return true;
}

// Emit one sample's kept set in ascending j: lane owns rows 32 w + lane; a prefix of the row
// counts gives each row's first slot, then the lane writes its row's kept elements in bit
// order and clears the row for the next sample.
template <int LOGP, typename T>
__device__ void emit_one(const SketchParams& P, const T* xs, int s, int64_t row, uint32_t* rmask, bool ok) {
  const int lane = threadIdx.x & 31;
  if (!ok) {
    emit_slow_exact<LOGP, T>(P, xs, s, row, column_state(P, row));
    return;
  }
  constexpr int MW = (Geo<LOGP>::P + 1023) / 1024;
  const int rows = (P.pk + 31) >> 5;
  const int64_t orow = row * P.m;
  int wbase = 0;
#pragma unroll
  for (int w = 0; w < MW; ++w) {
    const int rr = 32 * w + lane;
    uint32_t t = 0;
    if (rr < rows) {
      t = rmask[rr];
      rmask[rr] = 0;  // clean for the warp's next sample
    }
    const int cnt = __popc(t);
    int incl = cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(kFull, incl, o);
      if (lane >= o) incl += y;
    }
    int64_t pos = orow + wbase + incl - cnt;
    for (; t; t &= t - 1, ++pos) {
      const int j = 32 * rr + __ffs(t) - 1;
      P.idx_out[pos] = j;
      if (P.val_out) store_val<T>(P.val_out, pos, y_at<LOGP, T>(xs, s, j), P.val_f64);
    }
    wbase += __shfl_sync(kFull, incl, 31);
  }
  __syncwarp();
}

// ------------------------------------------------------------------------------------
template <int LOGP, typename T>
__global__ void __launch_bounds__(kThreads, 3) sketch_kernel(const SketchParams P) {
  using G = Geo<LOGP>;
  extern __shared__ __align__(16) unsigned char smem[];
  T* xs = reinterpret_cast<T*>(smem);
  constexpr int kSignWords = (G::P + 31) / 32;
  uint32_t* sgn = reinterpret_cast<uint32_t*>(smem + sizeof(T) * ((G::WORDS + 1) & ~1));
  unsigned char* wbase = reinterpret_cast<unsigned char*>(sgn) + 4 * ((kSignWords + 3) & ~3);
  const int warp = threadIdx.x >> 5;
  constexpr int kRowWords = mask_words<LOGP>();  // kept-set bitmask words
  constexpr int kSlot = LOGP < 5 ? 1 : G::P / 32;  // mask words per sample
  const size_t per_warp = warp_bytes<LOGP>(P.cap);
  unsigned char* mine = wbase + per_warp * warp;
  uint64_t* ck = reinterpret_cast<uint64_t*>(mine);
  uint64_t* memk = reinterpret_cast<uint64_t*>(mine + (size_t)P.cap * 8);
  int* hist = reinterpret_cast<int*>(mine + (size_t)P.cap * 8 + 256);
  uint32_t* rmask = reinterpret_cast<uint32_t*>(mine + (size_t)P.cap * 8 + 256 + 128);
  uint16_t* cj = reinterpret_cast<uint16_t*>(mine + (size_t)P.cap * 8 + 256 + 128 + 4 * kRowWords);
  for (int i = threadIdx.x & 31; i < kRowWords; i += 32) rmask[i] = 0;

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
  const T scale = (T)(1.0 / sqrt((double)G::P));  // transform.py:109

  // P >= 32: a warp selects all its samples of the tile while the tile's 16-byte copies
  // are in flight (the selection needs no data), then the CTA transforms and emits
  constexpr bool kEarly = LOGP >= 5;
  const bool async_load = has_x && std::is_same<T, float>::value && P.vec && !P.x_f64 && LOGP >= 2;
  const bool sampling = P.mode != kNoSample && P.mode != kGiven;
  for (int64_t tile = blockIdx.x; tile < P.num_tiles; tile += gridDim.x) {
    const int64_t row0 = tile * G::S;
    const int64_t rows_left = P.n - row0;
    __syncthreads();  // previous tile's emission is done with xs; signs visible
    if (has_x) {
      // ---- phase 1: load (zero pad p..p_pad and rows >= n) ----
      if (async_load) {
        // thread t copies 16 bytes at element f = 4 (t + k kThreads) of the tile: sample
        // s_k = f >> LOGP, column i_k = f & (P-1), compile-time offsets from k = 0
        constexpr int NV = kTileElems / 4 / kThreads;
        const int f0 = threadIdx.x * 4;
        const int s0 = f0 >> LOGP, i0 = f0 & (G::P - 1);
        const float* xb = reinterpret_cast<const float*>(P.X) + (row0 + s0) * P.ld + i0;
        const uint32_t dst0 = (uint32_t)__cvta_generic_to_shared(xs);
#pragma unroll
        for (int k = 0; k < NV; ++k) {
          const int f = f0 + k * kThreads * 4;
          const int sk = f >> LOGP, ik = f & (G::P - 1);
          const bool ok = sk < rows_left;
          const float* src = ok ? xb + (sk - s0) * P.ld + (ik - i0) : reinterpret_cast<const float*>(P.X);
          const uint32_t dst = dst0 + 4u * (uint32_t)(sk * G::SP + G::addr(ik));
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "r"(ok ? 16 : 0)
                       : "memory");
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
      } else if (P.vec && !P.x_f64) {
        constexpr int NV = kTileElems / 4 / kThreads;
        const int f0 = threadIdx.x * 4;
        const int s0 = f0 >> LOGP, i0 = f0 & (G::P - 1);
        const float* xb = reinterpret_cast<const float*>(P.X) + (row0 + s0) * P.ld + i0;
        float4 buf[NV];
#pragma unroll
        for (int k = 0; k < NV; ++k) {
          const int f = f0 + k * kThreads * 4;
          const int sk = f >> LOGP, ik = f & (G::P - 1);
          buf[k] = sk < rows_left ? __ldg(reinterpret_cast<const float4*>(xb + (sk - s0) * P.ld + (ik - i0)))
                                  : make_float4(0.f, 0.f, 0.f, 0.f);
        }
#pragma unroll
        for (int k = 0; k < NV; ++k) {
          const int f = f0 + k * kThreads * 4;
          const int sk = f >> LOGP, ik = f & (G::P - 1);
          T* d = xs + sk * G::SP + G::addr(ik);  // 4 consecutive i never cross a 32-row
          d[0] = (T)buf[k].x;
          d[1] = (T)buf[k].y;
          d[2] = (T)buf[k].z;
          d[3] = (T)buf[k].w;
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
          xs[s * G::SP + G::addr(i)] = v;
        }
      }
    }
    // ---- phase 3a: selection (one warp per sample) ----
    uint32_t okbits = 0;
    if (kEarly && sampling) {
      int k = 0;
      for (int s = warp; s < G::S && s < rows_left; s += kWarps, ++k)
        okbits |= (uint32_t)select_one<LOGP>(P, row0 + s, ck, cj, memk, hist, rmask + k * kSlot) << k;
    }
    if (has_x) {
      if (async_load) asm volatile("cp.async.wait_all;" ::: "memory");
      __syncthreads();
      // ---- phase 2: D then WHT then scale ----
      wht_all_windows<LOGP, T, 0>(xs, P.use_signs ? sgn : nullptr, scale);
      if (P.y_out) {
        for (int f = threadIdx.x; f < kTileElems; f += kThreads) {
          const int s = f >> LOGP, i = f & (G::P - 1);
          const int64_t row = row0 + s;
          if (row < P.n) P.y_out[row * G::P + i] = (double)xs[s * G::SP + G::addr(i)];
        }
      }
    }
    // ---- phase 3b: emit, one warp per sample ----
    if (sampling) {
      int k = 0;
      for (int s = warp; s < G::S && s < rows_left; s += kWarps, ++k) {
        uint32_t* rm = rmask + (kEarly ? k * kSlot : 0);
        const bool ok = kEarly ? (okbits >> k) & 1u : select_one<LOGP>(P, row0 + s, ck, cj, memk, hist, rm);
        emit_one<LOGP, T>(P, xs, s, row0 + s, rm, ok);
      }
    } else if (P.mode == kGiven) {  // gather at supplied indices (coalesced per row)
      for (int s = warp; s < G::S && s < rows_left; s += kWarps) {
        const int64_t o = (row0 + s) * P.m;
        for (int t = threadIdx.x & 31; t < P.m; t += 32)
          store_val<T>(P.val_out, o + t, y_at<LOGP, T>(xs, s, __ldg(P.idx_in + o + t)), P.val_f64);
      }
    }
  }
}

// ------------------------------------------------------------------------------------
// kGiven with fp32 rows: K1 without the selection, double-buffered. Tile k+1's cp.async
// copies are in flight while tile k is transformed and its values gathered, so the kernel
// streams at HBM rate instead of exposing each tile's load latency.
#ifndef SKC_GATHER_STAGES
#define SKC_GATHER_STAGES 2  // tile buffers per CTA: STAGES - 1 tiles load while one transforms
#endif
constexpr int kGatherStages = SKC_GATHER_STAGES;
template <int LOGP>
__global__ void __launch_bounds__(kThreads, kGatherStages > 2 ? 2 : 3) gather_kernel(const SketchParams P) {
  using G = Geo<LOGP>;
  extern __shared__ __align__(16) unsigned char smem[];
  constexpr size_t kTileBytes = sizeof(float) * ((G::WORDS + 3) & ~3);
  float* xs0 = reinterpret_cast<float*>(smem);
  constexpr int kSignWords = (G::P + 31) / 32;
  uint32_t* sgn = reinterpret_cast<uint32_t*>(smem + kGatherStages * kTileBytes);
  const int warp = threadIdx.x >> 5;
  if (P.use_signs) {  // D diagonal, _hash.py:38-43, regenerated per CTA
    for (int w = threadIdx.x; w < kSignWords; w += kThreads) {
      uint32_t bits = 0;
      for (int b = 0; b < 32 && w * 32 + b < G::P; ++b)
        bits |= (uint32_t)(mix64(P.sign_state + kGamma * (uint64_t)(w * 32 + b + 1)) >> 63) << b;
      sgn[w] = bits;
    }
  }
  const float scale = (float)(1.0 / sqrt((double)G::P));  // transform.py:109
  constexpr int NV = kTileElems / 4 / kThreads;
  const int f0 = threadIdx.x * 4;
  const int s0 = f0 >> LOGP, i0 = f0 & (G::P - 1);
  const uint32_t dst0 = (uint32_t)__cvta_generic_to_shared(smem);
  auto issue = [&](int64_t tile, int buf) {
    const int64_t row0 = tile * G::S;
    const int64_t rows_left = P.n - row0;
    const float* xb = reinterpret_cast<const float*>(P.X) + (row0 + s0) * P.ld + i0;
#pragma unroll
    for (int k = 0; k < NV; ++k) {
      const int f = f0 + k * kThreads * 4;
      const int sk = f >> LOGP, ik = f & (G::P - 1);
      const bool ok = sk < rows_left;
      const float* src = ok ? xb + (sk - s0) * P.ld + (ik - i0) : reinterpret_cast<const float*>(P.X);
      const uint32_t dst = dst0 + (uint32_t)(buf * kTileBytes) + 4u * (uint32_t)(sk * G::SP + G::addr(ik));
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "r"(ok ? 16 : 0) : "memory");
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  int64_t tile = blockIdx.x;
  // prologue: tiles it = 0 .. STAGES-2 in flight; every iteration commits one group (empty
  // past the end), so wait_group STAGES-1 always means "this iteration's tile has landed"
#pragma unroll
  for (int k = 0; k < kGatherStages - 1; ++k) {
    const int64_t t = tile + (int64_t)k * gridDim.x;
    if (t < P.num_tiles) issue(t, k);
    else asm volatile("cp.async.commit_group;" ::: "memory");
  }
  for (int it = 0; tile < P.num_tiles; tile += gridDim.x, ++it) {
    const int buf = it % kGatherStages;
    const int64_t next = tile + (int64_t)(kGatherStages - 1) * gridDim.x;
    if (next < P.num_tiles) issue(next, (it + kGatherStages - 1) % kGatherStages);
    else asm volatile("cp.async.commit_group;" ::: "memory");
    asm volatile("cp.async.wait_group %0;" ::"n"(kGatherStages - 1) : "memory");
    const int64_t row0 = tile * G::S;
    const int64_t rows_left = P.n - row0;
    // this warp's first sample's indices load during the transform (m <= 64 in registers)
    int pj0 = 0, pj1 = 0;
    if (warp < G::S && warp < rows_left && P.m <= 64) {
      const int64_t o = (row0 + warp) * P.m;
      const int lane = threadIdx.x & 31;
      if (lane < P.m) pj0 = __ldg(P.idx_in + o + lane);
      if (lane + 32 < P.m) pj1 = __ldg(P.idx_in + o + lane + 32);
    }
    __syncthreads();  // tile in buf visible to all; signs visible
    float* xs = reinterpret_cast<float*>(smem + buf * kTileBytes);
    wht_all_windows<LOGP, float, 0>(xs, P.use_signs ? sgn : nullptr, scale);
    if (P.y_out) {
      for (int f = threadIdx.x; f < kTileElems; f += kThreads) {
        const int s = f >> LOGP, i = f & (G::P - 1);
        if (s < rows_left) P.y_out[(row0 + s) * G::P + i] = (double)xs[s * G::SP + G::addr(i)];
      }
    }
    for (int s = warp; s < G::S && s < rows_left; s += kWarps) {
      const int64_t o = (row0 + s) * P.m;
      const int lane = threadIdx.x & 31;
      if (s == warp && P.m <= 64) {
        if (lane < P.m) store_val<float>(P.val_out, o + lane, y_at<LOGP, float>(xs, s, pj0), P.val_f64);
        if (lane + 32 < P.m) store_val<float>(P.val_out, o + lane + 32, y_at<LOGP, float>(xs, s, pj1), P.val_f64);
      } else {
        for (int t = lane; t < P.m; t += 32)
          store_val<float>(P.val_out, o + t, y_at<LOGP, float>(xs, s, __ldg(P.idx_in + o + t)), P.val_f64);
      }
    }
    __syncthreads();  // buf is refilled by the copies issued next iteration
  }
  (void)xs0;
}

template <int LOGP>
static int launch_gather_t(SketchParams P, cudaStream_t st) {
  using G = Geo<LOGP>;
  const size_t smem = kGatherStages * sizeof(float) * ((G::WORDS + 3) & ~3) + 4 * (((G::P + 31) / 32 + 3) & ~3);
  auto kern = gather_kernel<LOGP>;
  if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
    return check_launch("gather smem attribute");
  int occ = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, kThreads, smem);
  if (const char* e = getenv("SKC_GATHER_OCC")) occ = atoi(e) > 0 && atoi(e) < occ ? atoi(e) : occ;  // experiments
  if (occ < 1) occ = 1;
  P.num_tiles = (P.n + G::S - 1) / G::S;
  int64_t grid = (int64_t)sm_count() * occ;
  if (grid > P.num_tiles) grid = P.num_tiles;
  if (grid < 1) return SKC_OK;
  kern<<<(unsigned)grid, kThreads, smem, st>>>(P);
  return check_launch("gather_kernel");
}

static int launch_gather_logp(int logp, const SketchParams& P, cudaStream_t st) {
  switch (logp) {
    case 2: return launch_gather_t<2>(P, st);
    case 3: return launch_gather_t<3>(P, st);
    case 4: return launch_gather_t<4>(P, st);
    case 5: return launch_gather_t<5>(P, st);
    case 6: return launch_gather_t<6>(P, st);
    case 7: return launch_gather_t<7>(P, st);
    case 8: return launch_gather_t<8>(P, st);
    case 9: return launch_gather_t<9>(P, st);
    case 10: return launch_gather_t<10>(P, st);
    case 11: return launch_gather_t<11>(P, st);
    case 12: return launch_gather_t<12>(P, st);
  }
  return fail(SKC_EPARAM, "gather kernel needs 4 <= p_pad <= 4096");
}

// ------------------------------------------------------------------------------------
// Index-only sampler: the selection of K1 (phase 3) without the tile, one warp per sample,
// grid-stride over samples. With no 37 KB tile per CTA it runs at full occupancy, and K1 in
// kGiven mode then only loads, transforms and gathers (HBM-bound).
constexpr int kIdxWarps = 8;
template <int LOGP>
#ifndef SKC_IDX_MINB
#define SKC_IDX_MINB 8  // 32 registers: 8 CTAs (64 warps) per SM, no spills (measured best)
#endif
__global__ void __launch_bounds__(kIdxWarps * 32, SKC_IDX_MINB) indices_kernel(const SketchParams P) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int warp = threadIdx.x >> 5;
  constexpr int kRowWords = mask_words<LOGP>();
  unsigned char* mine = smem + warp_bytes<LOGP>(P.cap) * warp;
  uint64_t* ck = reinterpret_cast<uint64_t*>(mine);
  uint64_t* memk = reinterpret_cast<uint64_t*>(mine + (size_t)P.cap * 8);
  int* hist = reinterpret_cast<int*>(mine + (size_t)P.cap * 8 + 256);
  uint32_t* rmask = reinterpret_cast<uint32_t*>(mine + (size_t)P.cap * 8 + 256 + 128);
  uint16_t* cj = reinterpret_cast<uint16_t*>(mine + (size_t)P.cap * 8 + 256 + 128 + 4 * kRowWords);
  for (int i = threadIdx.x & 31; i < kRowWords; i += 32) rmask[i] = 0;
  __syncwarp();
  const int64_t warps = (int64_t)gridDim.x * kIdxWarps;
  for (int64_t row = blockIdx.x * (int64_t)kIdxWarps + warp; row < P.n; row += warps) {
    const bool ok = select_one<LOGP>(P, row, ck, cj, memk, hist, rmask);
    emit_one<LOGP, float>(P, nullptr, 0, row, rmask, ok);  // val_out == nullptr: indices only
  }
}

template <int LOGP>
static int launch_indices_t(SketchParams P, cudaStream_t st) {
  const size_t smem = warp_bytes<LOGP>(P.cap) * kIdxWarps;
  auto kern = indices_kernel<LOGP>;
  if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
    return check_launch("indices smem attribute");
  int occ = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, kIdxWarps * 32, smem);
  if (const char* e = getenv("SKC_IDX_OCC")) occ = atoi(e) > 0 && atoi(e) < occ ? atoi(e) : occ;  // experiments
  if (occ < 1) occ = 1;
  int64_t grid = (int64_t)sm_count() * occ;
  const int64_t need = (P.n + kIdxWarps - 1) / kIdxWarps;
  if (grid > need) grid = need;
  if (grid < 1) return SKC_OK;
  kern<<<(unsigned)grid, kIdxWarps * 32, smem, st>>>(P);
  return check_launch("indices_kernel");
}

static int launch_indices_logp(int logp, const SketchParams& P, cudaStream_t st) {
  switch (logp) {
    case 0: return launch_indices_t<0>(P, st);
    case 1: return launch_indices_t<1>(P, st);
    case 2: return launch_indices_t<2>(P, st);
    case 3: return launch_indices_t<3>(P, st);
    case 4: return launch_indices_t<4>(P, st);
    case 5: return launch_indices_t<5>(P, st);
    case 6: return launch_indices_t<6>(P, st);
    case 7: return launch_indices_t<7>(P, st);
    case 8: return launch_indices_t<8>(P, st);
    case 9: return launch_indices_t<9>(P, st);
    case 10: return launch_indices_t<10>(P, st);
    case 11: return launch_indices_t<11>(P, st);
    case 12: return launch_indices_t<12>(P, st);
  }
  return fail(SKC_EPARAM, "p_pad exceeds the largest instantiated sampler (4096)");
}

// ------------------------------------------------------------------------------------
template <int LOGP, typename T>
static int launch_sketch_t(SketchParams P, cudaStream_t st) {
  using G = Geo<LOGP>;
  const size_t sign_bytes = 4 * (((G::P + 31) / 32 + 3) & ~3);
  const size_t smem = sizeof(T) * ((G::WORDS + 1) & ~1) + sign_bytes + warp_bytes<LOGP>(P.cap) * kWarps;
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

// Host: prefilter threshold and candidate capacity for a plan of (pk, m)
static void plan_select(int32_t pk, int32_t m, SketchParams& P) {
  P.t_all = 0;
  P.t_hi = 0;
  if (m == pk) {
    P.mode = kFullSet;
    P.cap = 32;
    return;
  }
  // expected candidates: count < m (P ~ 3e-5 at m = 51) takes the exact slow path, ~64x a
  // row's hashing; measured: 4 sqrt(m) + 6 beats 5 sqrt(m) + 8 by 2% of the index kernel
  const double mu = m + 4.0 * sqrt((double)m) + 6.0;
  if (mu >= 0.25 * pk) {
    P.t_all = 1;  // every coordinate is a candidate
    P.cap = (pk + 31) & ~31;
  } else {
    P.t_hi = (uint32_t)floor(mu / pk * 4294967296.0);  // < 2^30 since mu < pk/4
    const double cap = mu + 6.0 * sqrt(mu) + 32.0;
    P.cap = ((int)cap + 31) & ~31;
  }
  P.mode = kSelect;
  if (P.cap > 1024) {
    P.mode = kSlowExact;
    P.cap = 32;
  }
}

// gather.cu: the TMA-staged gather (-1 when the shape is not eligible)
int gather_tma_launch(const void* X, int32_t x_dtype, int64_t ld, int64_t n, int32_t p, int32_t p_pad,
                      int32_t use_signs, uint64_t sign_seed, int32_t m, int32_t compute_dtype, const int32_t* idx_in,
                      void* val_out, int32_t val_dtype, cudaStream_t st);

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
  if (kind == SKC_KIND_NONE && X != nullptr) return fail(SKC_EPARAM, "internal: kind none uses sketch_identity");
  // Default: indices first (index-only sampler at full occupancy), then K1 gathers values at
  // them. SKC_SKETCH_FUSED=1 selects the single fused kernel instead.
  static const bool fused = getenv("SKC_SKETCH_FUSED") != nullptr;
  if (X == nullptr || idx_out == nullptr || fused) {
    if (X == nullptr && idx_out != nullptr && !fused) return launch_indices_logp(logp, P, st);
    if (compute_dtype == SKC_F64) return launch_sketch_logp<double>(logp, P, st);
    return launch_sketch_logp<float>(logp, P, st);
  }
  int rc = launch_indices_logp(logp, P, st);
  if (rc) return rc;
  SketchParams G = P;
  G.mode = kGiven;
  G.idx_in = idx_out;
  G.idx_out = nullptr;
  G.cap = 0;  // no selection scratch
  if (val_out == nullptr) return SKC_OK;
  rc = gather_tma_launch(X, x_dtype, ld, n, p, p_pad, P.use_signs, sign_seed, m, compute_dtype, idx_out, val_out,
                         val_dtype, st);
  if (rc != -1) return rc;
  if (compute_dtype == SKC_F64) return launch_sketch_logp<double>(logp, G, st);
  if (G.vec && !G.x_f64 && logp >= 2) return launch_gather_logp(logp, G, st);
  return launch_sketch_logp<float>(logp, G, st);
}

// kind == none: values are the raw coordinates (transform.py:141-146); the sampler runs
// without a transform and a gather kernel reads the values.
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

// ------------------------------------------------------------------------------------
// Philox sampler (north_star's counter-based alternative to the reference hash). Column g
// (global) draws m of p coordinates without replacement by Floyd's algorithm:
//   for s in 0..m-1: j = p - m + s; t = floor(r_s * (j + 1) / 2^32);
//                    insert t unless already present, else insert j,
// with r_s = component s % 4 of Philox4x32-10(counter {s / 4, g_lo, g_hi, "PHLX"},
// key mix64(master ^ "PHLX")). The set is returned in ascending order. One lane per column;
// the lane's p-bit set lives in shared memory as [word][lane], which is bank-conflict-free
// for any word indices. ~45 warp-instructions per column at p=1024, m=51.
constexpr int kPhxThreads = 128;

constexpr int kPhxStageMaxM = 160;  // staged, coalesced output up to here (80 KB); direct stores above

__global__ void __launch_bounds__(kPhxThreads) philox_indices_kernel(uint64_t key, int64_t col0, int64_t n, int32_t p,
                                                                    int32_t m, int32_t* __restrict__ idx_out) {
  extern __shared__ uint32_t bm[];  // [W][kPhxThreads] sets, then [kPhxThreads][S] staged rows
  const int W = (p + 31) >> 5;
  const int S = m | 1;  // odd stride: conflict-free both when lanes write and when a row is read
  const bool staged = m <= kPhxStageMaxM;
  uint32_t* stage = bm + (size_t)W * kPhxThreads;
  const int t = threadIdx.x, lane = t & 31, wbase = t & ~31;
  const uint32_t k0 = (uint32_t)key, k1 = (uint32_t)(key >> 32);
  for (int64_t base = blockIdx.x * (int64_t)kPhxThreads; base < n; base += (int64_t)gridDim.x * kPhxThreads) {
    const int64_t row = base + t;
    if (row < n) {
      for (int w = 0; w < W; ++w) bm[w * kPhxThreads + t] = 0u;
      const uint64_t g = (uint64_t)(col0 + row);
      for (int s0 = 0; s0 < m; s0 += 4) {
        const Philox4 r4 = philox4x32_10(
            Philox4{(uint32_t)(s0 >> 2), (uint32_t)g, (uint32_t)(g >> 32), (uint32_t)kTagPhilox}, k0, k1);
        const uint32_t rr[4] = {r4.x, r4.y, r4.z, r4.w};
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int s = s0 + q;
          if (s < m) {
            const uint32_t j = (uint32_t)(p - m + s);
            const uint32_t c = __umulhi(rr[q], j + 1u);
            const uint32_t hit = (bm[(c >> 5) * kPhxThreads + t] >> (c & 31)) & 1u;
            const uint32_t x = hit ? j : c;
            bm[(x >> 5) * kPhxThreads + t] |= 1u << (x & 31);
          }
        }
      }
      // ascending emit with a uniform trip count (m); the word advance is short
      int w = 0;
      uint32_t b = bm[t];
      int32_t* mine = idx_out + row * m;
      for (int k = 0; k < m; ++k) {
        while (b == 0u) b = bm[++w * kPhxThreads + t];
        const uint32_t j = 32u * w + __ffs(b) - 1;
        if (staged) stage[t * S + k] = j;
        else mine[k] = (int32_t)j;
        b &= b - 1u;
      }
    }
    if (staged) {
      __syncwarp();
      // the warp's 32 rows are contiguous in idx_out: coalesced stores
      const int64_t r0 = base + wbase;
      const int64_t left = n - r0;
      const int rows = left < 32 ? (int)left : 32;
      int32_t* out = idx_out + r0 * m;
      for (int r = 0; r < rows; ++r)
        for (int q = lane; q < m; q += 32) out[r * m + q] = (int32_t)stage[(wbase + r) * S + q];
      __syncwarp();
    }
  }
}

int philox_indices_launch(uint64_t master_seed, int64_t col0, int64_t n, int32_t p, int32_t m, int32_t* idx_out,
                          cudaStream_t st) {
  if (n <= 0) return SKC_OK;
  const size_t smem =
      ((size_t)((p + 31) / 32) * kPhxThreads + (m <= kPhxStageMaxM ? (size_t)kPhxThreads * (m | 1) : 0)) * 4;
  if (cudaFuncSetAttribute(philox_indices_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
    return check_launch("philox smem attribute");
  int occ = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, philox_indices_kernel, kPhxThreads, smem);
  int64_t grid = (int64_t)sm_count() * (occ < 1 ? 1 : occ);
  const int64_t need = (n + kPhxThreads - 1) / kPhxThreads;
  if (grid > need) grid = need;
  philox_indices_kernel<<<(unsigned)grid, kPhxThreads, smem, st>>>(mix64(master_seed ^ kTagPhilox), col0, n, p, m,
                                                                   idx_out);
  return check_launch("philox_indices_kernel");
}

// Values at supplied sorted indices (oracle mode with reference-supplied indices, or the
// Philox sampler's): load + D + WHT + gather, no selection.
int sketch_given_launch(const void* X, int32_t x_dtype, int64_t ld, int64_t n, int32_t p, int32_t p_pad, int32_t kind,
                        uint64_t sign_seed, int32_t m, int32_t compute_dtype, const int32_t* idx_in, void* val_out,
                        int32_t val_dtype, cudaStream_t st) {
  if (n <= 0 || val_out == nullptr) return SKC_OK;
  if (kind == SKC_KIND_NONE) {
    const int64_t blocks = (n * (int64_t)m + 255) / 256;
    gather_identity_kernel<<<(unsigned)blocks, 256, 0, st>>>(X, x_dtype == SKC_F64, ld, n, p, m, idx_in, val_out,
                                                             val_dtype == SKC_F64, nullptr, p_pad);
    return check_launch("gather_identity_kernel");
  }
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
  P.val_out = val_out;
  P.val_f64 = val_dtype == SKC_F64;
  P.mode = kGiven;
  P.idx_in = idx_in;
  P.cap = 0;
  int logp = 0;
  while ((1 << logp) < p_pad) ++logp;
  const uintptr_t xa = reinterpret_cast<uintptr_t>(X);
  P.vec = p == p_pad && p_pad >= 4 && (ld % 4) == 0 && (xa % 16) == 0;
  const int rc = gather_tma_launch(X, x_dtype, ld, n, p, p_pad, P.use_signs, sign_seed, m, compute_dtype, idx_in,
                                   val_out, val_dtype, st);
  if (rc != -1) return rc;
  if (compute_dtype == SKC_F64) return launch_sketch_logp<double>(logp, P, st);
  if (P.vec && !P.x_f64 && logp >= 2) return launch_gather_logp(logp, P, st);
  return launch_sketch_logp<float>(logp, P, st);
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
