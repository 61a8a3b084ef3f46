// K1b: precondition + gather at supplied indices, TMA-staged and warp-specialised (sm_100a).
//
// The values half of sketch_stream (sketch.py:211-220: precondition_columns, then
// take_along_axis at the plan's indices), for fp32 rows and both compute types:
//   compute f64: the reference's fp64 arithmetic in its butterfly order (transform.py:92-110),
//                so the values are bit-identical to sketchpipe's;
//   compute f32: the fast path (packed FADD2 butterflies).
//
// CTA = NCW consumer warps + 1 producer warp, one CTA per SM, persistent over tiles.
//   producer  one lane streams tiles of S_T samples (rows) into an NST-deep ring of
//             shared-memory stages with cp.async.bulk.tensor (TMA). The tensor map views X
//             as [n][p/32][32] fp32 with 128-byte swizzle: 16-byte chunk c of 128-byte row r
//             lands at chunk c ^ (r & 7), so the window-0 reads below are conflict-free.
//             Rows past n are zero-filled by the TMA unit. full/empty mbarriers per stage.
//   team      the consumers form teams: one warp per 1024 elements (1024/p samples) for
//             p <= 1024, p/1024 warps per sample above (named barriers).
//   window 0  thread u of a team owns the 32 consecutive elements of 128-byte row u: eight
//             16-byte LDS from the stage, the D signs, conversion to the compute type,
//             butterfly stages h = 1..16 in registers, then 16-byte stores into the team's
//             private work buffer (padded rows, conflict-free). The stage is released.
//   window k  the next 5 index bits per thread (stages h = 32.., in order), in place in
//             the work buffer: element i at s*SP + j + PAD*(j >> 5), SP and PAD chosen by a
//             bank simulation (tools/gather_banks.py) so every access is conflict-free for
//             the BASELINE shapes (p = 256 .. 4096).
//   gather    the team's (sample, t) entries, prefetched before the stage wait, read their
//             transformed value, scale by fl(1/sqrt(p)) (only the kept values: the reference
//             scales every entry, an elementwise product, so the result is identical) and
//             store contiguously: a team's rows are adjacent in val_out, so the stores of a
//             warp cover one contiguous range.
// Algorithmic HBM bytes per sample: 4p (row) + 4m (indices) + m * sizeof(value).
#include <cuda.h>
#include <cudaTypedefs.h>
#include <math.h>
#include <stdlib.h>

#include <mutex>
#include <type_traits>

#include "common.cuh"

namespace skc {
namespace gtma {

constexpr uint32_t kFull = 0xFFFFFFFFu;

template <int LOGP, typename T>
struct Lay {
  static constexpr int P = 1 << LOGP;
  static constexpr int TT = P / 32 > 32 ? P / 32 : 32;  // threads per team
  static constexpr int TW = TT / 32;                    // warps per team
  static constexpr int Q = LOGP <= 10 ? 1024 / P : 1;   // samples per team
  static constexpr int PAD = sizeof(T) == 4 ? 4 : 2;    // elements of padding per 32
  static constexpr int SP0 = (P / 32) * (32 + PAD);
  // sample stride (elements): the base layout, except where the bank simulation found a
  // conflict across the samples of one warp (p = 256/512 floats, p = 256 doubles)
  static constexpr int SP = sizeof(T) == 4 ? (LOGP == 8 ? 296 : LOGP == 9 ? 592 : SP0) : (LOGP == 8 ? 280 : SP0);
  static constexpr int TEAM_ELEMS = Q * SP;
  static constexpr int NWIN = (LOGP + 4) / 5;
  static __host__ __device__ constexpr int bk(int k) { return 5 * k < LOGP - 5 ? 5 * k : LOGP - 5; }
  // work-buffer offset of team-local element i (linear over disjoint bit sets of i)
  static __host__ __device__ constexpr int addr(int i) {
    return (i >> LOGP) * SP + (i & (P - 1)) + PAD * ((i & (P - 1)) >> 5);
  }
  static __device__ __forceinline__ int u_part(int k, int u) {
    const int b = bk(k);
    return (u & ((1 << b) - 1)) | ((u >> b) << (b + 5));
  }
};

struct Params {
  int64_t n;
  int32_t m;
  const int32_t* idx_in;
  void* val_out;
  int32_t val_f64;
  uint64_t sign_state;
  int32_t use_signs;
  int64_t num_tiles;
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint32_t a, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(a), "r"(count));
}
__device__ __forceinline__ void mbar_arrive(uint32_t a) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(a) : "memory");
}
__device__ __forceinline__ void mbar_arrive_tx(uint32_t a, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(a), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t a, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n\tWAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1, %2;\n\t"
      "@!P1 bra WAIT_%=;\n\t}\n" ::"r"(a),
      "r"(parity), "r"(1000000)
      : "memory");
}
__device__ __forceinline__ void tma_load_3d(uint32_t dst, const CUtensorMap* map, uint32_t bar, int c0, int c1, int c2,
                                            uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%3, %4, %5}], [%2], %6;" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(bar), "r"(c0), "r"(c1), "r"(c2), "l"(policy)
      : "memory");
}
template <int TW>
__device__ __forceinline__ void team_sync(int team) {
  if constexpr (TW == 1) {
    __syncwarp();
  } else {
    asm volatile("bar.sync %0, %1;" ::"r"(1 + team), "r"(TW * 32) : "memory");
  }
}

// packed fp32 pairs (FADD2 / FMUL2): each lane is an IEEE round-to-nearest add, so the
// results equal the scalar order exactly
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

// butterfly stages on bits [b0, b1) of a thread's 32 register elements (h = 1 << (b - bk)
// in register-index space), in the reference order
template <typename T, int B0, int B1>
__device__ __forceinline__ void stages(T (&v)[32]) {
  using A = Arith<T>;
  if constexpr (std::is_same<T, float>::value) {
    uint64_t w[16];
#pragma unroll
    for (int k = 0; k < 16; ++k) w[k] = pack2(v[2 * k], v[2 * k + 1]);
#pragma unroll
    for (int b = B0; b < B1; ++b) {
      const int h = 1 << b;
      if (h == 1) {
#pragma unroll
        for (int k = 0; k < 16; ++k) {
          float a, c;
          unpack2(w[k], a, c);
          w[k] = pack2(fadd(a, c), fsub(a, c));
        }
      } else {
        const int hp = h >> 1;
#pragma unroll
        for (int k = 0; k < 16; ++k) {
          if (((2 * k) & h) == 0) {
            const uint64_t x = w[k], y = w[k + hp];
            w[k] = add2(x, y);
            w[k + hp] = sub2(x, y);
          }
        }
      }
    }
#pragma unroll
    for (int k = 0; k < 16; ++k) unpack2(w[k], v[2 * k], v[2 * k + 1]);
  } else {
#pragma unroll
    for (int b = B0; b < B1; ++b) {
      const int h = 1 << b;
#pragma unroll
      for (int e = 0; e < 32; ++e) {
        if ((e & h) == 0) {
          const T a = v[e], c = v[e + h];
          v[e] = A::add(a, c);
          v[e + h] = A::sub(a, c);
        }
      }
    }
  }
}

// window 0: stage (swizzled fp32 row r) -> signs -> h = 1..16 -> work buffer (contiguous 32)
template <int LOGP, typename T>
__device__ __forceinline__ void window0(const unsigned char* stage, uint32_t r, uint32_t sbits, T* dst) {
  float f[32];
  const unsigned char* row = stage + (size_t)r * 128;
#pragma unroll
  for (int c = 0; c < 8; ++c) {
    const float4 t = *reinterpret_cast<const float4*>(row + ((c ^ (r & 7)) << 4));
    f[4 * c] = t.x;
    f[4 * c + 1] = t.y;
    f[4 * c + 2] = t.z;
    f[4 * c + 3] = t.w;
  }
  T v[32];
#pragma unroll
  for (int e = 0; e < 32; ++e)
    v[e] = (T)__int_as_float(__float_as_int(f[e]) ^ (int)(((sbits >> e) & 1u) << 31));  // D (_hash.py:38-43)
  stages<T, 0, 5>(v);
  using V16 = typename std::conditional<sizeof(T) == 4, float4, double2>::type;
  constexpr int PER = 16 / sizeof(T);
#pragma unroll
  for (int c = 0; c < 32 / PER; ++c) {
    V16 t;
    T* tp = reinterpret_cast<T*>(&t);
#pragma unroll
    for (int q = 0; q < PER; ++q) tp[q] = v[c * PER + q];
    reinterpret_cast<V16*>(dst)[c] = t;
  }
}

// window k >= 1 in place in the work buffer
template <int LOGP, typename T, int K>
__device__ __forceinline__ void window_k(T* work, int u) {
  using L = Lay<LOGP, T>;
  constexpr int bk = L::bk(K);
  T* base = work + L::addr(L::u_part(K, u));
  T v[32];
#pragma unroll
  for (int e = 0; e < 32; ++e) v[e] = base[L::addr(e << bk)];
  stages<T, 5 * K - bk, 5>(v);
#pragma unroll
  for (int e = 0; e < 32; ++e) base[L::addr(e << bk)] = v[e];
}

template <int LOGP, typename T, int K>
__device__ __forceinline__ void windows_from(T* work, int u, int team) {
  using L = Lay<LOGP, T>;
  if constexpr (K < L::NWIN) {
    team_sync<L::TW>(team);
    window_k<LOGP, T, K>(work, u);
    windows_from<LOGP, T, K + 1>(work, u, team);
  }
}

template <int LOGP, typename T, int NCW, int NST>
__global__ void __launch_bounds__((NCW + 1) * 32, 1)
    gather_tma_kernel(const __grid_constant__ CUtensorMap tmap, const Params P) {
  using L = Lay<LOGP, T>;
  constexpr int TEAMS = NCW / L::TW;
  constexpr int S_T = TEAMS * L::Q;                 // samples per stage tile
  constexpr uint32_t STAGE_BYTES = S_T * L::P * 4;  // fp32 rows
  constexpr int SIGN_WORDS = L::P / 32;
  extern __shared__ unsigned char smem_raw[];
  const uint32_t raw = smem_u32(smem_raw);
  unsigned char* sm = smem_raw + (((raw + 1023u) & ~1023u) - raw);  // 1024-aligned (128B swizzle)
  unsigned char* stages_p = sm;
  T* work_all = reinterpret_cast<T*>(sm + NST * STAGE_BYTES);
  uint32_t* sgn = reinterpret_cast<uint32_t*>(work_all + TEAMS * L::TEAM_ELEMS);
  uint64_t* bars = reinterpret_cast<uint64_t*>(sgn + ((SIGN_WORDS + 1) & ~1));  // full[NST], empty[NST]
  const uint32_t full0 = smem_u32(bars), empty0 = full0 + 8 * NST;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    for (int s = 0; s < NST; ++s) {
      mbar_init(full0 + 8 * s, 1);
      mbar_init(empty0 + 8 * s, NCW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  for (int w = threadIdx.x; w < SIGN_WORDS; w += blockDim.x) {  // D diagonal, regenerated per CTA
    uint32_t bits = 0;
    if (P.use_signs)
      for (int b = 0; b < 32; ++b)
        bits |= (uint32_t)(mix64(P.sign_state + kGamma * (uint64_t)(w * 32 + b + 1)) >> 63) << b;
    sgn[w] = bits;
  }
  __syncthreads();

  if (warp == NCW) {  // producer: TMA ring
    if (lane == 0) {
      uint64_t policy;
      asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(policy));
      int it = 0;
      for (int64_t tile = blockIdx.x; tile < P.num_tiles; tile += gridDim.x, ++it) {
        const int st = it % NST;
        if (it >= NST) mbar_wait(empty0 + 8 * st, ((it / NST) - 1) & 1);
        mbar_arrive_tx(full0 + 8 * st, STAGE_BYTES);
        tma_load_3d(smem_u32(stages_p + (size_t)st * STAGE_BYTES), &tmap, full0 + 8 * st, 0, 0, (int)(tile * S_T),
                    policy);
      }
    }
    return;
  }

  const int team = warp / L::TW;
  const int tu = threadIdx.x - team * L::TT;  // thread within the team
  T* work = work_all + team * L::TEAM_ELEMS;
  const T scale = (T)(1.0 / sqrt((double)L::P));  // transform.py:109, fl(1/sqrt(p_pad))
  const int m = P.m;
  const uint32_t swords = (uint32_t)(tu % SIGN_WORDS);
  const uint32_t sbits = sgn[swords];
  int it = 0;
  for (int64_t tile = blockIdx.x; tile < P.num_tiles; tile += gridDim.x, ++it) {
    const int st = it % NST;
    const int64_t row0 = tile * S_T + (int64_t)team * L::Q;  // the team's first sample
    const int64_t left = P.n - row0;
    const int qv = left >= L::Q ? L::Q : (left > 0 ? (int)left : 0);  // valid samples of the team
    const int F = qv * m;                                             // gather entries
    const int32_t* ib = P.idx_in + row0 * m;
    // the first two entries per thread load while the tile is in flight
    const int j0 = tu < F ? __ldg(ib + tu) : 0;
    const int j1 = tu + L::TT < F ? __ldg(ib + tu + L::TT) : 0;
    mbar_wait(full0 + 8 * st, (it / NST) & 1);
    if (qv > 0)
      window0<LOGP, T>(stages_p + (size_t)st * STAGE_BYTES, (uint32_t)(team * L::TT + tu), sbits,
                       work + L::addr(32 * tu));
    __syncwarp();
    if (lane == 0) mbar_arrive(empty0 + 8 * st);  // the stage may be refilled
    if (qv > 0) {
      windows_from<LOGP, T, 1>(work, tu, team);
      team_sync<L::TW>(team);
      auto val_at = [&](int f, int j) -> T {
        const int s = L::Q == 1 ? 0 : f / m;
        return Arith<T>::mul(work[s * L::SP + j + L::PAD * (j >> 5)], scale);
      };
      const int64_t o = row0 * m;
      if (P.val_f64) {
        double* out = reinterpret_cast<double*>(P.val_out) + o;
        if (tu < F) out[tu] = (double)val_at(tu, j0);
        if (tu + L::TT < F) out[tu + L::TT] = (double)val_at(tu + L::TT, j1);
        for (int f = tu + 2 * L::TT; f < F; f += L::TT) out[f] = (double)val_at(f, __ldg(ib + f));
      } else {
        float* out = reinterpret_cast<float*>(P.val_out) + o;
        if (tu < F) out[tu] = (float)val_at(tu, j0);
        if (tu + L::TT < F) out[tu + L::TT] = (float)val_at(tu + L::TT, j1);
        for (int f = tu + 2 * L::TT; f < F; f += L::TT) out[f] = (float)val_at(f, __ldg(ib + f));
      }
    }
    team_sync<L::TW>(team);  // the work buffer is rewritten by the next tile
  }
}

// ------------------------------------------------------------------------------------
// host side
template <typename T>
struct Cfg;
// consumer warps and stages per type (A/B: tools/variant_build.sh NAME "-DSKC_GT64_NCW=12 ...")
#ifndef SKC_GT32_NCW
#define SKC_GT32_NCW 16
#endif
#ifndef SKC_GT32_NST
#define SKC_GT32_NST 2
#endif
#ifndef SKC_GT64_NCW
#define SKC_GT64_NCW 8
#endif
#ifndef SKC_GT64_NST
#define SKC_GT64_NST 3
#endif
template <int A, int B>
struct CfgV {
  static constexpr int NCW = A, NST = B;
};
template <>
struct Cfg<float> : CfgV<SKC_GT32_NCW, SKC_GT32_NST> {};
template <>
struct Cfg<double> : CfgV<SKC_GT64_NCW, SKC_GT64_NST> {};

template <int LOGP, typename T>
static size_t smem_bytes() {
  using L = Lay<LOGP, T>;
  constexpr int NCW = Cfg<T>::NCW, NST = Cfg<T>::NST;
  constexpr int TEAMS = NCW / L::TW;
  return 1024 + (size_t)NST * TEAMS * L::Q * L::P * 4 + (size_t)TEAMS * L::TEAM_ELEMS * sizeof(T) +
         4 * (size_t)(((L::P / 32) + 1) & ~1) + 16 * NST;
}

static PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  return fn;
}

template <int LOGP, typename T>
static int launch_t(const float* X, int64_t ld, const Params& P0, cudaStream_t st) {
  using L = Lay<LOGP, T>;
  constexpr int NCW = Cfg<T>::NCW, NST = Cfg<T>::NST;
  constexpr int TEAMS = NCW / L::TW;
  constexpr int S_T = TEAMS * L::Q;
  Params P = P0;
  P.num_tiles = (P.n + S_T - 1) / S_T;
  auto enc = encode_fn();
  if (enc == nullptr) return -1;
  CUtensorMap map;
  const cuuint64_t gdim[3] = {32, (cuuint64_t)(L::P / 32), (cuuint64_t)P.n};
  const cuuint64_t gstride[2] = {128, (cuuint64_t)ld * 4};
  const cuuint32_t box[3] = {32, (cuuint32_t)(L::P / 32), (cuuint32_t)S_T};
  const cuuint32_t estr[3] = {1, 1, 1};
  if (enc(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<float*>(X), gdim, gstride, box, estr,
          CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return -1;
  const size_t smem = smem_bytes<LOGP, T>();
  auto kern = gather_tma_kernel<LOGP, T, NCW, NST>;
  if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
    return check_launch("gather_tma smem attribute");
  int64_t grid = sm_count();
  if (grid > P.num_tiles) grid = P.num_tiles;
  if (grid < 1) return SKC_OK;
  kern<<<(unsigned)grid, (NCW + 1) * 32, smem, st>>>(map, P);
  return check_launch("gather_tma_kernel");
}

template <typename T>
static int launch_logp(int logp, const float* X, int64_t ld, const Params& P, cudaStream_t st) {
  switch (logp) {
    case 5: return launch_t<5, T>(X, ld, P, st);
    case 6: return launch_t<6, T>(X, ld, P, st);
    case 7: return launch_t<7, T>(X, ld, P, st);
    case 8: return launch_t<8, T>(X, ld, P, st);
    case 9: return launch_t<9, T>(X, ld, P, st);
    case 10: return launch_t<10, T>(X, ld, P, st);
    case 11: return launch_t<11, T>(X, ld, P, st);
    case 12: return launch_t<12, T>(X, ld, P, st);
  }
  return -1;
}

}  // namespace gtma

// Returns SKC_OK / an error code, or -1 when the shape is not eligible (the caller then
// uses the cp.async kernels of sketch.cu). Eligible: fp32 rows, p == p_pad in [32, 4096],
// 16-byte aligned base and row stride, n < 2^31. SKC_GATHER=old disables it (A/B runs).
bool gather_tma_eligible(const void* X, int32_t x_dtype, int64_t ld, int64_t n, int32_t p, int32_t p_pad) {
  static const bool off = [] {
    const char* e = getenv("SKC_GATHER");
    return e != nullptr && e[0] == 'o';
  }();
  return !(off || X == nullptr || x_dtype != SKC_F32 || p != p_pad || p_pad < 32 || p_pad > 4096 || n <= 0 ||
           n >= ((int64_t)1 << 31) || (reinterpret_cast<uintptr_t>(X) % 16) != 0 || ((ld * 4) % 16) != 0 || ld < p);
}

int gather_tma_launch(const void* X, int32_t x_dtype, int64_t ld, int64_t n, int32_t p, int32_t p_pad,
                      int32_t use_signs, uint64_t sign_seed, int32_t m, int32_t compute_dtype, const int32_t* idx_in,
                      void* val_out, int32_t val_dtype, cudaStream_t st) {
  if (!gather_tma_eligible(X, x_dtype, ld, n, p, p_pad)) return -1;
  int logp = 0;
  while ((1 << logp) < p_pad) ++logp;
  gtma::Params P{};
  P.n = n;
  P.m = m;
  P.idx_in = idx_in;
  P.val_out = val_out;
  P.val_f64 = val_dtype == SKC_F64;
  P.sign_state = mix64(sign_seed ^ kTagSign);
  P.use_signs = use_signs;
  const float* Xf = reinterpret_cast<const float*>(X);
  if (compute_dtype == SKC_F64) return gtma::launch_logp<double>(logp, Xf, ld, P, st);
  return gtma::launch_logp<float>(logp, Xf, ld, P, st);
}

}  // namespace skc
