// K5t: sparsified K-means assignment with a tensor-core filter and exact fp64 verification.
// Reference: _SparseOps.assign, cluster.py:181-187: d2 = [values | ones] @ [-2 mu ; mu*mu] + colsq,
// labels = first argmin over k, d2min = max(d2[label], 0).
//
// The product [values | ones] @ [-2 mu ; mu*mu] is GEMM-shaped: (points x 2p) @ (2p x K). K5t
// computes it densely on the 5th-generation tensor cores over zero-filled tiles, in bf16 with
// fp32 accumulation in TMEM, as a FILTER; the exact fp64 value in the reference's operation
// order is then computed only for the candidates the filter cannot rule out.
//
//  prepare  (once per sketch) the sketch as compact u32 entries (coordinate | bf16(value) << 16)
//           laid out [tile pair][entry group of 4][256 rows] (16-byte loads, coalesced per
//           warp), plus colsq per point in numpy's pairwise order (row_sqnorms_launch).
//  table    (per iteration) B = [-2 mu ; mu*mu] in bf16, per 32-coordinate chunk one image
//           in the UMMA K-major core-matrix layout, so one bulk copy moves a chunk.
//  filter   CTA = 256 points (two M=128 tiles sharing every B chunk). Eight fill warps build
//           the A operand (lane = point row; 16-byte stores of the row's values and of ones
//           at its support), a producer lane bulk-copies B, one thread issues
//           tcgen05.mma kind::f16 (bf16 x bf16 -> fp32, M=128, N = K rounded up to 16) into
//           TMEM (two accumulator buffers), and four epilogue warps turn each row into a
//           candidate set: with dt = D + colsq, every centre with dt - E <= min(dt + E).
//  bound    |dt - d| <= E = 1.1 eps (2 max(dt,0) + 8 colsq) / (1 - 2 eps), where
//           eps = 1.001 * 2^-8 (bf16 inputs) + (2m + 2p/16 + 64) 2^-22 (fp32 accumulation)
//           + (2m+1) 2^-53 (fp64 reference rounding) + 2^-20: the absolute terms
//           T = sum |2 v mu| + sum mu^2 satisfy T <= 2d + 8 colsq (Cauchy-Schwarz:
//           sqrt(P) <= sqrt(d) + sqrt(colsq)), and d <= (dt + 8 eps colsq) / (1 - 2 eps).
//           So the exact argmin is always a candidate.
//  verify   lane = point: the exact fp64 value (km_assign_kernel's arithmetic) for each of
//           its candidates, first minimum (lowest k on ties). Points with more than kCmax
//           candidates or a non-finite filter value go to a list that the fp32 filter K5f
//           (tight bound) resolves. Labels, d2min, the changed count and the farthest point
//           are bit-identical to K5.
#include <cuda_bf16.h>
#include <math.h>

#include "common.cuh"

namespace skc {

int row_sqnorms_launch(const void* val, int val_f64, int64_t n, int32_t m, double* out, cudaStream_t st);
int assign_filter_list_launch(const int32_t* idx, const void* val, int val_f64, int64_t n, int32_t m,
                              const double* mu, int32_t p_pad, int32_t K, const int32_t* prev, int32_t* labels,
                              double* d2min, const int64_t* list, const int32_t* list_n, const double* tx,
                              const double* ty, float* t32, int64_t* bch, double* bmx, int64_t* barg, int G,
                              cudaStream_t st);
int assign_reduce_launch(const int64_t* bch, const double* bmx, const int64_t* barg, int G, int64_t* out,
                         double* d2max, cudaStream_t st);
int tables2_launch(const double* mu, int32_t p_pad, int32_t K, double* tx, double* ty, cudaStream_t st);

namespace {
constexpr int kRows = 128;  // M of one MMA = rows of one tile
constexpr int kTiles = 2;   // tiles per CTA pass: 256 points share every B chunk
constexpr int kPts = kRows * kTiles;
#ifndef SKC_KT_CHUNK
#define SKC_KT_CHUNK 32
#endif
constexpr int kChunk = SKC_KT_CHUNK;  // coordinates per stage
constexpr int kKC = 2 * kChunk;       // K elements per stage: values part, then ones part
constexpr int kRowShift = 16 + (kChunk == 32 ? 5 : kChunk == 64 ? 6 : 4);  // list entry: value | x | row
static_assert(kChunk == 16 || kChunk == 32 || kChunk == 64, "chunk of 16, 32 or 64 coordinates");
constexpr int kSBO = kKC * 16;        // bytes between 8-row core-matrix groups
constexpr int kTileA = kRows * kKC * 2;
#ifndef SKC_KT_STAGES
#define SKC_KT_STAGES 4
#endif
constexpr int kNst = SKC_KT_STAGES;
constexpr int kNmax = 128;  // two tiles x two TMEM buffers x 128 columns = 512
#ifndef SKC_KT_FILLW
#define SKC_KT_FILLW 8
#endif
constexpr int kFillWarps = SKC_KT_FILLW;        // fill warps (8: two entries per thread per chunk)
constexpr int kFillT = kFillWarps * 32;
constexpr int kPF = kPts * 2 / kFillT;          // entries per fill thread per chunk kept in registers
constexpr int kProdWarp = kFillWarps;
constexpr int kMmaWarp = kFillWarps + 1;
constexpr int kEpi0 = kFillWarps + 2;
constexpr int kWarps = kEpi0 + 4;
constexpr int kCmax = 8;  // candidates kept per point; more go to the K5f list
constexpr uint32_t kSentinel = 0xFFFFu;
constexpr uint8_t kOverflow = 0xFF;
constexpr int kVerifyThreads = 256;

__device__ __forceinline__ uint64_t sdesc(uint32_t saddr) {  // SWIZZLE_NONE, LBO 128 B, SBO kSBO, version 1
  return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)(128 >> 4) << 16) | ((uint64_t)(kSBO >> 4) << 32) |
         (1ull << 46);
}
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
__device__ __forceinline__ void sts128(uint32_t a, uint32_t x, uint32_t y, uint32_t z, uint32_t w) {
  asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(a), "r"(x), "r"(y), "r"(z), "r"(w) : "memory");
}
__device__ __forceinline__ void mma_bf16(uint32_t tmem, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem),
      "l"(a), "l"(b), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void mma_commit(uint32_t bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void tmem_ld16(uint32_t addr, float* f) {
  uint32_t v[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]),
        "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
      : "r"(addr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int j = 0; j < 16; ++j) f[j] = __uint_as_float(v[j]);
}
}  // namespace

// ------------------------------------------------------------------------------ prepare
// one thread per (tile pair, entry group g, row r): four entries of point tp*256 + r
// exact values transposed per tile pair, vT[tp][t][r] (fp64): the verify pass's loads coalesce
template <typename V>
__global__ void km_tc_values_kernel(const V* __restrict__ val, int64_t n, int m, int64_t ntp, double* __restrict__ vT) {
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= ntp * m * kPts) return;
  const int r = (int)(e % kPts);
  const int64_t tt = e / kPts;
  const int t = (int)(tt % m);
  const int64_t i = (tt / m) * kPts + r;
  vT[e] = i < n ? (double)__ldg(val + i * m + t) : 0.0;
}

template <typename V>
__global__ void km_tc_entries_kernel(const int32_t* __restrict__ idx, const V* __restrict__ val, int64_t n, int m,
                                     int G, int64_t ntp, uint4* __restrict__ ent) {
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= ntp * G * kPts) return;
  const int r = (int)(e % kPts);
  const int64_t tg = e / kPts;
  const int g = (int)(tg % G);
  const int64_t tp = tg / G;
  const int64_t i = tp * kPts + r;
  uint32_t w[4];
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    const int t = 4 * g + u;
    w[u] = kSentinel;
    if (i < n && t < m) {
      const uint32_t j = (uint32_t)__ldg(idx + i * m + t);
      const uint32_t b = __bfloat16_as_ushort(__double2bfloat16((double)__ldg(val + i * m + t)));
      w[u] = j | (b << 16);
    }
  }
  ent[e] = make_uint4(w[0], w[1], w[2], w[3]);
}

// per tile pair and 32-coordinate chunk, the list of its entries as u32 (bf16 value | x << 16 |
// row << kRowShift, x = coordinate - chunk start), so each stage's A operand is a zero fill plus one
// coalesced pass over a short list. offs[tp][c] (nch + 1 per tile pair) index into the tile
// pair's 256 m entries; the order inside a list is irrelevant (positions are distinct).
template <typename V>
__global__ void __launch_bounds__(kPts) km_tc_bucket_kernel(const int32_t* __restrict__ idx,
                                                            const V* __restrict__ val, int64_t n, int m, int nch,
                                                            int64_t ntp, uint32_t* __restrict__ lists,
                                                            uint32_t* __restrict__ offs) {
  extern __shared__ uint32_t bk[];  // cnt[nch], pos[nch]
  uint32_t* cnt = bk;
  uint32_t* pos = bk + nch;
  const int r = threadIdx.x;
  for (int64_t tp = blockIdx.x; tp < ntp; tp += gridDim.x) {
    for (int c = r; c < nch; c += kPts) cnt[c] = 0;
    __syncthreads();
    const int64_t i = tp * kPts + r;
    if (i < n)
      for (int t = 0; t < m; ++t) atomicAdd(&cnt[__ldg(idx + i * m + t) / kChunk], 1u);
    __syncthreads();
    if (r < 32) {  // exclusive scan by one warp
      uint32_t run = 0;
      for (int c0 = 0; c0 < nch; c0 += 32) {
        const int c = c0 + r;
        const uint32_t k = c < nch ? cnt[c] : 0;
        uint32_t x = k;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, x, o);
          if (r >= o) x += y;
        }
        if (c < nch) pos[c] = run + x - k, offs[tp * (nch + 1) + c] = run + x - k;
        run += __shfl_sync(0xFFFFFFFFu, x, 31);
      }
      if (r == 0) offs[tp * (nch + 1) + nch] = run;
    }
    __syncthreads();
    uint32_t* L = lists + (size_t)tp * kPts * m;
    if (i < n)
      for (int t = 0; t < m; ++t) {
        const uint32_t j = (uint32_t)__ldg(idx + i * m + t);
        const uint32_t b = __bfloat16_as_ushort(__double2bfloat16((double)__ldg(val + i * m + t)));
        L[atomicAdd(&pos[j / kChunk], 1u)] = b | ((j % kChunk) << 16) | ((uint32_t)r << kRowShift);
      }
    __syncthreads();
  }
}

// ------------------------------------------------------------------------------ table
// B image of chunk c: element (centre x, k) at half [x>>3][k>>3][x&7][k&7], k < kChunk: -2 mu,
// k >= kChunk: mu*mu, at coordinate c*kChunk + (k mod kChunk); centres x >= K are zero
__global__ void km_tc_table_kernel(const double* __restrict__ mu, int32_t p_pad, int K, int Npad,
                                   __nv_bfloat16* __restrict__ img) {
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t per = (int64_t)Npad * kKC;
  if (e >= (int64_t)(p_pad / kChunk) * per) return;
  const int64_t c = e / per;
  const int rem = (int)(e - c * per);
  const int x = rem / kKC, k = rem % kKC;
  double v = 0.0;
  if (x < K) {
    const double u = mu[(c * kChunk + (k % kChunk)) * (int64_t)K + x];
    v = k < kChunk ? -2.0 * u : u * u;
  }
  img[c * per + (x >> 3) * (kKC * 8) + (k >> 3) * 64 + (x & 7) * 8 + (k & 7)] = __double2bfloat16(v);
}

// ------------------------------------------------------------------------------ filter
struct KtParams {
  const uint32_t* lists;  // km_tc_bucket_kernel
  const uint32_t* offs;
  int m;
  const double* colsq;
  const __nv_bfloat16* img;
  int64_t n, ntp;
  int G, nch, K, Npad;
  float eps;       // E = eps (2 max(dt,0) + 8 colsq), the 1.1 / (1 - 2 eps) folded in
  uint8_t* cand;   // [n][kCmax]
  uint8_t* ncand;  // [n]: count, or kOverflow
  int64_t* list;   // overflow points
  int32_t* list_n;
};

__global__ void __launch_bounds__(kWarps * 32, 1) km_tc_filter_kernel(const __grid_constant__ KtParams P) {
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ __align__(8) uint64_t bars[2 * kNst + 4];
  __shared__ uint32_t tmem_base;
  __shared__ uint32_t prev_off[kNst][kPF][kFillT];  // fill: offsets this thread wrote in each stage
  __shared__ int dirty[kNst];                   // chunk sequence number of a stage's last overflow
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t bbytes = (uint32_t)P.Npad * kKC * 2;
  const uint32_t stage_bytes = kTiles * kTileA + bbytes;
  const uint32_t base_sh = (uint32_t)__cvta_generic_to_shared(smem);
  const uint32_t bar_sh = (uint32_t)__cvta_generic_to_shared(bars);
  auto full_bar = [&](int s) { return bar_sh + 8u * s; };
  auto empty_bar = [&](int s) { return bar_sh + 8u * (kNst + s); };
  auto accf_bar = [&](int b) { return bar_sh + 8u * (2 * kNst + b); };
  auto acce_bar = [&](int b) { return bar_sh + 8u * (2 * kNst + 2 + b); };
  if (threadIdx.x == 0) {
    for (int s = 0; s < kNst; ++s) mbar_init(full_bar(s), kFillWarps + 1), mbar_init(empty_bar(s), 1);
    for (int b = 0; b < 2; ++b) mbar_init(accf_bar(b), 1), mbar_init(acce_bar(b), 4);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == kMmaWarp) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
        (uint32_t)__cvta_generic_to_shared(&tmem_base)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (warp < kFillWarps) {  // every A operand starts zero; the fill then only clears what it wrote
    for (uint32_t q = threadIdx.x; q < (uint32_t)kNst * stage_bytes / 16; q += kFillT)
      if ((16u * q) % stage_bytes < (uint32_t)(kTiles * kTileA)) sts128(base_sh + 16u * q, 0u, 0u, 0u, 0u);
    for (int s = 0; s < kNst; ++s)
      for (int u = 0; u < kPF; ++u) prev_off[s][u][threadIdx.x] = 0xFFFFFFFFu;
    if (threadIdx.x < kNst) dirty[threadIdx.x] = -1 - kNst;
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tmem_base;
  const int nch = P.nch;

  if (warp < kFillWarps) {
    // ------------------------------------------------------------ fill: zero + scatter per stage
    const int ft = threadIdx.x;  // 0 .. kFillT-1
    int64_t gc = 0;
    for (int64_t tp = blockIdx.x; tp < P.ntp; tp += gridDim.x) {
      const uint32_t* L = P.lists + (size_t)tp * kPts * P.m;
      const uint32_t* of = P.offs + (size_t)tp * (nch + 1);
      // chunk c's first kPF entries of this thread, loaded two chunks ahead into one of three
      // register sets (fixed roles: a register move would wait for its load)
      struct Set {
        uint32_t e[kPF];
        uint32_t o0, o1;  // the chunk's list range
      };
      Set e0, e1, e2;
      auto fetch = [&](int c, Set& f) {
        f.o0 = c < nch ? __ldg(of + c) : 0u;
        f.o1 = c < nch ? __ldg(of + c + 1) : 0u;
#pragma unroll
        for (int u = 0; u < kPF; ++u) {
          const uint32_t q = f.o0 + (uint32_t)(ft + u * kFillT);
          f.e[u] = q < f.o1 ? __ldg(L + q) : 0xFFFFFFFFu;
        }
      };
      auto put = [&](uint32_t sa, uint32_t w) {  // returns the entry's offset inside the stage
        const uint32_t r = w >> kRowShift, x = (w >> 16) & (kChunk - 1u);
        const uint32_t a0 = (r >> 7) * kTileA + ((r & 127u) >> 3) * kSBO + (r & 7u) * 16u + (x >> 3) * 128u + (x & 7u) * 2u;
        asm volatile("st.shared.u16 [%0], %1;" ::"r"(sa + a0), "h"((uint16_t)(w & 0xFFFFu)) : "memory");
        asm volatile("st.shared.u16 [%0], %1;" ::"r"(sa + a0 + 128u * (kChunk / 8)), "h"((uint16_t)0x3F80u) : "memory");
        return a0;
      };
      auto body = [&](int c, const Set& cur, Set& f) {
        const uint32_t(&e)[kPF] = cur.e;
        fetch(c + 2, f);
        const int s = (int)(gc % kNst);
        mbar_wait(empty_bar(s), (uint32_t)(((gc / kNst) & 1) ^ 1));
        const uint32_t sa = base_sh + (uint32_t)s * stage_bytes;
#ifndef SKC_KT_NOFILL  // timing experiment: MMA pipeline without the A fill
        // the stage is all zero except where its previous chunk wrote: clear exactly those
        // (or everything, if that chunk had entries beyond the kPF per thread kept here)
        if (dirty[s] == (int)gc - kNst) {
#pragma unroll
          for (int q = 0; q < kTiles * kTileA / 16 / kFillT; ++q) sts128(sa + 16u * (ft + q * kFillT), 0u, 0u, 0u, 0u);
        } else {
#pragma unroll
          for (int u = 0; u < kPF; ++u) {
            const uint32_t a0 = prev_off[s][u][ft];
            if (a0 != 0xFFFFFFFFu) {
              asm volatile("st.shared.u16 [%0], %1;" ::"r"(sa + a0), "h"((uint16_t)0) : "memory");
              asm volatile("st.shared.u16 [%0], %1;" ::"r"(sa + a0 + 128u * (kChunk / 8)), "h"((uint16_t)0) : "memory");
            }
          }
        }
        asm volatile("bar.sync 1, %0;" ::"n"(kFillT) : "memory");
#pragma unroll
        for (int u = 0; u < kPF; ++u) prev_off[s][u][ft] = e[u] != 0xFFFFFFFFu ? put(sa, e[u]) : 0xFFFFFFFFu;
        for (uint32_t q = cur.o0 + (uint32_t)(ft + kPF * kFillT); q < cur.o1; q += kFillT) {
          put(sa, __ldg(L + q));
          dirty[s] = (int)gc;
        }
#else
        (void)e;
        (void)put;
#endif
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();
        if (lane == 0) mbar_arrive(full_bar(s));
        ++gc;
      };
      fetch(0, e0);
      fetch(1, e1);
      for (int c = 0; c < nch; c += 3) {
        body(c, e0, e2);
        if (c + 1 < nch) body(c + 1, e1, e0);
        if (c + 2 < nch) body(c + 2, e2, e1);
      }
    }
  } else if (warp == kProdWarp) {
    // ------------------------------------------------------------ producer: B chunk copies
    if (lane == 0) {
      int64_t gc = 0;
      const char* img = reinterpret_cast<const char*>(P.img);
      for (int64_t tp = blockIdx.x; tp < P.ntp; tp += gridDim.x) {
        for (int c = 0; c < nch; ++c, ++gc) {
          const int s = (int)(gc % kNst);
          mbar_wait(empty_bar(s), (uint32_t)(((gc / kNst) & 1) ^ 1));
          mbar_arrive_tx(full_bar(s), bbytes);
          const uint32_t dst = base_sh + (uint32_t)s * stage_bytes + kTiles * kTileA;
          asm volatile(
              "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
              "l"(img + (size_t)c * bbytes), "r"(bbytes), "r"(full_bar(s))
              : "memory");
        }
      }
    }
    __syncwarp();
  } else if (warp == kMmaWarp) {
    // ------------------------------------------------------------ MMA issuer
    if (lane == 0) {
      // bf16 x bf16 -> fp32, K-major A and B, N = Npad, M = 128
      const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(P.Npad >> 3) << 17) |
                             ((uint32_t)(kRows >> 4) << 24);
      int64_t gc = 0, tl = 0;
      for (int64_t tp = blockIdx.x; tp < P.ntp; tp += gridDim.x, ++tl) {
        const int b = (int)(tl & 1);
        mbar_wait(acce_bar(b), (uint32_t)(((tl >> 1) & 1) ^ 1));
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        for (int c = 0; c < nch; ++c, ++gc) {
          const int s = (int)(gc % kNst);
          mbar_wait(full_bar(s), (uint32_t)((gc / kNst) & 1));
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          const uint32_t st = base_sh + (uint32_t)s * stage_bytes, sb = st + kTiles * kTileA;
#pragma unroll
          for (int t = 0; t < kTiles; ++t)
#pragma unroll
            for (int ks = 0; ks < kKC / 16; ++ks)
              mma_bf16(tmem + (uint32_t)(b * 256 + t * 128), sdesc(st + t * kTileA + 256u * ks), sdesc(sb + 256u * ks),
                       idesc, (c > 0 || ks > 0) ? 1u : 0u);
          mma_commit(empty_bar(s));
        }
        mma_commit(accf_bar(b));
      }
    }
    __syncwarp();
  } else {
    // ------------------------------------------------------------ epilogue: TMEM -> candidates
    const int q = warp & 3;  // TMEM lane quarter of this warp
    const int K = P.K, nb16 = P.Npad / 16;
    int64_t tl = 0;
    for (int64_t tp = blockIdx.x; tp < P.ntp; tp += gridDim.x, ++tl) {
      const int b = (int)(tl & 1);
      mbar_wait(accf_bar(b), (uint32_t)((tl >> 1) & 1));
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
#ifndef SKC_KT_NOEPI  // timing experiment: no TMEM drain
#pragma unroll 1
      for (int t = 0; t < kTiles; ++t) {
        const int64_t i = tp * kPts + t * kRows + 32 * q + lane;
        const bool live = i < P.n;
        const float cf = live ? (float)__ldg(P.colsq + i) : 0.f;
        const float e8 = 8.f * cf;
        const uint32_t ta = tmem + ((uint32_t)(32 * q) << 16) + (uint32_t)(b * 256 + t * 128);
        float ub = __int_as_float(0x7F800000);
        // the bound needs colsq in [2^-90, 2^100] (no fp32 under/overflow of the terms that matter)
        bool bad = !(cf >= 0x1p-90f && cf <= 0x1p100f);
#pragma unroll 1
        for (int cb = 0; cb < nb16; ++cb) {
          float f[16];
          tmem_ld16(ta + 16u * cb, f);
#pragma unroll
          for (int j = 0; j < 16; ++j) {
            if (cb * 16 + j < K) {
              const float dt = f[j] + cf;
              bad |= !isfinite(dt);
              ub = fminf(ub, dt + P.eps * fmaf(2.f, fmaxf(dt, 0.f), e8));
            }
          }
        }
        int cnt = 0;
#pragma unroll 1
        for (int cb = 0; cb < nb16; ++cb) {
          float f[16];
          tmem_ld16(ta + 16u * cb, f);
#pragma unroll
          for (int j = 0; j < 16; ++j) {
            const int k = cb * 16 + j;
            if (k < K) {
              const float dt = f[j] + cf;
              if (dt - P.eps * fmaf(2.f, fmaxf(dt, 0.f), e8) <= ub) {
                if (live && cnt < kCmax) P.cand[i * kCmax + cnt] = (uint8_t)k;
                ++cnt;
              }
            }
          }
        }
        if (live) {
          const bool over = bad || cnt > kCmax || cnt == 0;
          P.ncand[i] = over ? kOverflow : (uint8_t)cnt;
          if (over) P.list[atomicAdd(P.list_n, 1)] = i;
        }
      }
#endif
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      __syncwarp();
      if (lane == 0) mbar_arrive(acce_bar(b));
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == kMmaWarp) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

// ------------------------------------------------------------------------------ verify
// block = one tile pair. Its (point, candidate) pairs are flattened (a block scan of the
// candidate counts) so that threads take pairs, not points: a point's 2-3 near-tie candidates
// do not serialise its warp. Each pair gets the exact fp64 d in km_assign_kernel's order (sum_t
// v*(-2 mu), then sum_t mu^2, then + colsq) from the prepared coalesced entries and values; then
// each point takes the first minimum (lowest k on ties). Per-block changed count and (max d2min,
// first index).
__global__ void __launch_bounds__(kVerifyThreads) km_tc_verify_kernel(
    const uint4* __restrict__ ent, const double* __restrict__ vT, int G, int64_t ntp, int64_t n, int m,
    const double* __restrict__ tabx, const double* __restrict__ taby, int K, const double* __restrict__ colsq,
    const uint8_t* __restrict__ cand,
    const uint8_t* __restrict__ ncand, const int32_t* __restrict__ prev, int32_t* __restrict__ labels,
    double* __restrict__ d2min, int64_t* __restrict__ blk_changed, double* __restrict__ blk_max,
    int64_t* __restrict__ blk_arg) {
  static_assert(kVerifyThreads == kPts, "one thread per point of a tile pair");
  __shared__ uint8_t pk[kPts * kCmax], pr[kPts * kCmax];
  __shared__ double sd[kPts * kCmax];
  __shared__ int wsum[kPts / 32];
  int64_t changed = 0;
  double bmax = -1.0;
  int64_t barg = -1;
  const int r = threadIdx.x, lane = r & 31, wp = r >> 5;
  for (int64_t tp = blockIdx.x; tp < ntp; tp += gridDim.x) {
    const int64_t i = tp * kPts + r;
    int nc = i < n ? ncand[i] : 0;
    if (nc == kOverflow) nc = 0;  // resolved by the K5f list pass
    // block exclusive scan of nc
    int x = nc;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xFFFFFFFFu, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) wsum[wp] = x;
    __syncthreads();
    int base = 0, total = 0;
#pragma unroll
    for (int w = 0; w < kPts / 32; ++w) {
      base += w < wp ? wsum[w] : 0;
      total += wsum[w];
    }
    const int start = base + x - nc;
    for (int c = 0; c < nc; ++c) pk[start + c] = cand[i * kCmax + c], pr[start + c] = (uint8_t)r;
    __syncthreads();
    for (int q = r; q < total; q += kPts) {
      const int rr = pr[q], k = pk[q];
      const uint4* ep = ent + (size_t)tp * G * kPts + rr;
      const double* vp = vT + (size_t)tp * m * kPts + rr;
      const double* tkx = tabx + k;
      const double* tky = taby + k;
      double acc = 0.0;
      for (int g = 0; g < G; ++g) {
        const uint4 w = __ldg(ep + (size_t)g * kPts);
        const uint32_t ww[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int t = 4 * g + u;
          if (t < m) acc = dadd(acc, dmul(__ldg(vp + (size_t)t * kPts), __ldg(tkx + (ww[u] & 0xFFFFu) * (size_t)K)));
        }
      }
      for (int g = 0; g < G; ++g) {
        const uint4 w = __ldg(ep + (size_t)g * kPts);
        const uint32_t ww[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
        for (int u = 0; u < 4; ++u)
          if (4 * g + u < m) acc = dadd(acc, __ldg(tky + (ww[u] & 0xFFFFu) * (size_t)K));
      }
      sd[q] = dadd(acc, __ldg(colsq + tp * kPts + rr));
    }
    __syncthreads();
    if (nc > 0) {
      double best = 0.0;
      int bk = -1;
      for (int c = 0; c < nc; ++c) {
        const double d = sd[start + c];
        const int k = pk[start + c];
        if (bk < 0 || d < best || (d == best && k < bk)) best = d, bk = k;
      }
      const double dm = best > 0.0 ? best : 0.0;  // np.clip(.., 0, None)
      labels[i] = bk;
      d2min[i] = dm;
      if (prev != nullptr) changed += prev[i] != bk;
      if (dm > bmax || (dm == bmax && (barg < 0 || i < barg))) bmax = dm, barg = i;
    }
    __syncthreads();  // pk / pr / sd / wsum are reused by the next tile pair
  }
  __shared__ int64_t s_ch[kVerifyThreads / 32], s_arg[kVerifyThreads / 32];
  __shared__ double s_mx[kVerifyThreads / 32];
  const int warp = wp;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const int64_t oc = __shfl_xor_sync(0xFFFFFFFFu, changed, o), oa = __shfl_xor_sync(0xFFFFFFFFu, barg, o);
    const double om = __shfl_xor_sync(0xFFFFFFFFu, bmax, o);
    changed += oc;
    if (oa >= 0 && (om > bmax || (om == bmax && (barg < 0 || oa < barg)))) bmax = om, barg = oa;
  }
  if (lane == 0) s_ch[warp] = changed, s_mx[warp] = bmax, s_arg[warp] = barg;
  __syncthreads();
  if (threadIdx.x == 0) {
    int64_t c = 0, a = -1;
    double mx = -1.0;
    for (int w = 0; w < kVerifyThreads / 32; ++w) {
      c += s_ch[w];
      if (s_arg[w] >= 0 && (s_mx[w] > mx || (s_mx[w] == mx && (a < 0 || s_arg[w] < a)))) mx = s_mx[w], a = s_arg[w];
    }
    blk_changed[blockIdx.x] = c;
    blk_max[blockIdx.x] = mx;
    blk_arg[blockIdx.x] = a;
  }
}

// ------------------------------------------------------------------------------ host
bool kmtc_supported(int32_t p_pad, int32_t K, int32_t m) {
  return p_pad % kChunk == 0 && p_pad <= 65535 && K >= 1 && K <= kNmax && m >= 1;
}

static int64_t kt_ntp(int64_t n) { return (n + kPts - 1) / kPts; }
static int kt_groups(int32_t m) { return (m + 3) / 4; }

// per-sketch: [colsq: n doubles][entries][transposed fp64 values][chunk lists][list offsets]
static size_t prep_colsq_bytes(int64_t n) { return ((size_t)n * 8 + 255) & ~(size_t)255; }
static size_t prep_ent_bytes(int64_t n, int32_t m) { return (size_t)kt_ntp(n) * kt_groups(m) * kPts * 16; }
static size_t prep_vt_bytes(int64_t n, int32_t m) { return (size_t)kt_ntp(n) * m * kPts * 8; }
static size_t prep_list_bytes(int64_t n, int32_t m) { return ((size_t)kt_ntp(n) * m * kPts * 4 + 255) & ~(size_t)255; }
size_t kmtc_prep_ws(int64_t n, int32_t m, int32_t p_pad) {
  return prep_colsq_bytes(n) + prep_ent_bytes(n, m) + prep_vt_bytes(n, m) + prep_list_bytes(n, m) +
         (size_t)kt_ntp(n) * (p_pad / kChunk + 1) * 4 + 256;
}
struct KtPrep {
  double* colsq;
  uint4* ent;
  double* vT;
  uint32_t* lists;
  uint32_t* offs;
};
static KtPrep kt_prep(const void* prep, int64_t n, int32_t m) {
  char* b = static_cast<char*>(const_cast<void*>(prep));
  KtPrep R;
  R.colsq = reinterpret_cast<double*>(b);
  b += prep_colsq_bytes(n);
  R.ent = reinterpret_cast<uint4*>(b);
  b += prep_ent_bytes(n, m);
  R.vT = reinterpret_cast<double*>(b);
  b += prep_vt_bytes(n, m);
  R.lists = reinterpret_cast<uint32_t*>(b);
  b += prep_list_bytes(n, m);
  R.offs = reinterpret_cast<uint32_t*>(b);
  return R;
}

int kmtc_prepare_launch(const int32_t* idx, const void* val, int val_f64, int64_t n, int32_t m, int32_t p_pad,
                        void* prep, cudaStream_t st) {
  const KtPrep R = kt_prep(prep, n, m);
  double* colsq = R.colsq;
  uint4* ent = R.ent;
  double* vT = R.vT;
  int rc = row_sqnorms_launch(val, val_f64, n, m, colsq, st);
  if (rc) return rc;
  const int G = kt_groups(m);
  const int64_t ntp = kt_ntp(n), tot = ntp * G * kPts;
  if (tot == 0) return SKC_OK;
  const unsigned blocks = (unsigned)((tot + 255) / 256);
  if (val_f64)
    km_tc_entries_kernel<double><<<blocks, 256, 0, st>>>(idx, static_cast<const double*>(val), n, m, G, ntp, ent);
  else
    km_tc_entries_kernel<float><<<blocks, 256, 0, st>>>(idx, static_cast<const float*>(val), n, m, G, ntp, ent);
  if ((rc = check_launch("km_tc_entries_kernel"))) return rc;
  const unsigned vblocks = (unsigned)((ntp * m * kPts + 255) / 256);
  if (val_f64)
    km_tc_values_kernel<double><<<vblocks, 256, 0, st>>>(static_cast<const double*>(val), n, m, ntp, vT);
  else
    km_tc_values_kernel<float><<<vblocks, 256, 0, st>>>(static_cast<const float*>(val), n, m, ntp, vT);
  if ((rc = check_launch("km_tc_values_kernel"))) return rc;
  const int nch = p_pad / kChunk;
  const size_t bsm = (size_t)2 * nch * 4;
  int64_t bgrid = ntp < 8LL * sm_count() ? ntp : 8LL * sm_count();
  if (val_f64) {
    cudaFuncSetAttribute(km_tc_bucket_kernel<double>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bsm);
    km_tc_bucket_kernel<double><<<(unsigned)bgrid, kPts, bsm, st>>>(idx, static_cast<const double*>(val), n, m, nch,
                                                                   ntp, R.lists, R.offs);
  } else {
    cudaFuncSetAttribute(km_tc_bucket_kernel<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bsm);
    km_tc_bucket_kernel<float><<<(unsigned)bgrid, kPts, bsm, st>>>(idx, static_cast<const float*>(val), n, m, nch,
                                                                  ntp, R.lists, R.offs);
  }
  return check_launch("km_tc_bucket_kernel");
}

// one resident wave of the grid-stride verify blocks (each loops over tile pairs): a second,
// partial wave would leave most SMs idle while it finishes
static int verify_grid(int64_t n) {
  static int occ = 0;
  if (occ == 0) {
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, km_tc_verify_kernel, kVerifyThreads, 0);
    if (occ < 1) occ = 1;
  }
  int64_t g = kt_ntp(n);
  const int64_t cap = (int64_t)occ * sm_count();
  if (g > cap) g = cap;
  return (int)(g < 1 ? 1 : g);
}
static int list_grid() { return 4 * sm_count(); }
static int kt_npad(int32_t K) { return (K + 15) & ~15; }

// per-iteration: [tab: -2 mu and mu*mu planes, p*K each][t32 p*K4][img][cand n*8][ncand n][list n][list_n][block partials]
struct KtWs {
  size_t tab, t32, img, cand, ncand, list, list_n, bch, bmx, barg, total;
};
static KtWs kt_ws(int64_t n, int32_t p_pad, int32_t K) {
  KtWs L{};
  size_t o = 0;
  auto take = [&](size_t bytes) {
    const size_t r = o;
    o += (bytes + 255) & ~(size_t)255;
    return r;
  };
  const int Gb = verify_grid(n) + list_grid();
  L.tab = take((size_t)p_pad * K * 16);
  L.t32 = take((size_t)p_pad * ((K + 3) & ~3) * 4);
  L.img = take((size_t)(p_pad / kChunk) * kt_npad(K) * kKC * 2);
  L.cand = take((size_t)n * kCmax);
  L.ncand = take((size_t)n);
  L.list = take((size_t)n * 8);
  L.list_n = take(4);
  L.bch = take((size_t)Gb * 8);
  L.bmx = take((size_t)Gb * 8);
  L.barg = take((size_t)Gb * 8);
  L.total = o;
  return L;
}
size_t kmtc_assign_ws(int64_t n, int32_t p_pad, int32_t K) { return kt_ws(n, p_pad, K).total; }

int kmtc_assign_launch(const int32_t* idx, const void* val, int val_f64, int64_t n, int32_t m, const double* mu,
                       int32_t p_pad, int32_t K, const int32_t* prev, int32_t* labels, double* d2min, int64_t* out,
                       double* d2max, const void* prep, void* ws, cudaStream_t st) {
  const KtWs L = kt_ws(n, p_pad, K);
  char* w = static_cast<char*>(ws);
  double* tx = reinterpret_cast<double*>(w + L.tab);
  double* ty = tx + (size_t)p_pad * K;
  float* t32 = reinterpret_cast<float*>(w + L.t32);
  __nv_bfloat16* img = reinterpret_cast<__nv_bfloat16*>(w + L.img);
  uint8_t* cand = reinterpret_cast<uint8_t*>(w + L.cand);
  uint8_t* ncand = reinterpret_cast<uint8_t*>(w + L.ncand);
  int64_t* list = reinterpret_cast<int64_t*>(w + L.list);
  int32_t* list_n = reinterpret_cast<int32_t*>(w + L.list_n);
  int64_t* bch = reinterpret_cast<int64_t*>(w + L.bch);
  double* bmx = reinterpret_cast<double*>(w + L.bmx);
  int64_t* barg = reinterpret_cast<int64_t*>(w + L.barg);
  const KtPrep R = kt_prep(prep, n, m);
  const double* colsq = R.colsq;
  const uint4* ent = R.ent;
  const double* vT = R.vT;
  int rc;
  if ((rc = tables2_launch(mu, p_pad, K, tx, ty, st))) return rc;
  const int Npad = kt_npad(K);
  const int64_t img_elems = (int64_t)(p_pad / kChunk) * Npad * kKC;
  km_tc_table_kernel<<<(unsigned)((img_elems + 255) / 256), 256, 0, st>>>(mu, p_pad, K, Npad, img);
  if ((rc = check_launch("km_tc_table_kernel"))) return rc;
  cudaMemsetAsync(list_n, 0, 4, st);
  const int Gv = verify_grid(n), Gl = list_grid();
  if (n > 0) {
    KtParams H{};
    H.lists = R.lists;
    H.offs = R.offs;
    H.m = m;
    H.colsq = colsq;
    H.img = img;
    H.n = n;
    H.ntp = kt_ntp(n);
    H.G = kt_groups(m);
    H.nch = p_pad / kChunk;
    H.K = K;
    H.Npad = Npad;
    const double eps = 1.001 * 0x1p-8 + (2.0 * m + 2.0 * p_pad / 16.0 + 64.0) * 0x1p-22 + (2.0 * m + 1.0) * 0x1p-53 +
                       0x1p-20;
    H.eps = (float)(1.1 * eps / (1.0 - 2.0 * eps));
#ifdef SKC_KT_EPS_SCALE  // experiment only (unsafe): how the candidate count depends on the bound
    H.eps *= (float)SKC_KT_EPS_SCALE;
#endif
    H.cand = cand;
    H.ncand = ncand;
    H.list = list;
    H.list_n = list_n;
    const size_t smem = (size_t)kNst * (kTiles * kTileA + (size_t)Npad * kKC * 2);
    cudaFuncSetAttribute(km_tc_filter_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    int64_t grid = sm_count();
    if (grid > H.ntp) grid = H.ntp;
    km_tc_filter_kernel<<<(unsigned)grid, kWarps * 32, smem, st>>>(H);
    if ((rc = check_launch("km_tc_filter_kernel"))) return rc;
    km_tc_verify_kernel<<<Gv, kVerifyThreads, 0, st>>>(ent, vT, H.G, H.ntp, n, m, tx, ty, K, colsq, cand, ncand, prev,
                                                        labels, d2min, bch, bmx, barg);
    if ((rc = check_launch("km_tc_verify_kernel"))) return rc;
    if ((rc = assign_filter_list_launch(idx, val, val_f64, n, m, mu, p_pad, K, prev, labels, d2min, list, list_n, tx, ty,
                                        t32, bch + Gv, bmx + Gv, barg + Gv, Gl, st)))
      return rc;
  }
  return assign_reduce_launch(bch, bmx, barg, n > 0 ? Gv + Gl : 0, out, d2max, st);
}

}  // namespace skc
