// K3t: the raw covariance W^T W on the 5th-generation tensor cores, for large m/p
// (north_star: "a tcgen05/TMEM GEMM over zero-filled tiles when m/p is large"; the sparse
// scatter K3 / K3g covers small m/p). Reference: estimators.py:59-61 (W @ W.T).
//
// K3b (bucket): one warp per chunk of 32 rows sorts the chunk's elements by 128-coordinate
// block and writes, per element, an 8-byte entry: its offset inside a 128-coordinate operand
// tile (core-matrix layout below) and the fp16 hi/lo split of x = w * 2^e (|x| <= 2^15,
// e from max |w|): hi = fp16(x), lo = fp16(x - hi), ~22 bits together. Blocks are padded to
// an even entry count.
// K3t: a unit is a 128 x 256 output strip, coordinates [A0, A0+128) x [B0, B0+256) with
// A0 = 128 I, B0 = 256 J2, for every (I, J2) touching the upper triangle. CTA (unit,
// replica) walks the replica's chunks. Four fill groups of four warps each own one of four
// operand stages and every fourth chunk: zero the stage (16-byte stores), then store the
// chunk's entries of blocks I, 2 J2, 2 J2 + 1 (contiguous in the bucketed chunk) as fp16 into
// K-major, unswizzled tiles. One thread issues per 16-row K-step three tcgen05.mma kind::f16
// M=128 N=256 (hi*hi + hi*lo + lo*hi, fp32 accumulation in TMEM). Each window of rows
// accumulates into one of two 256-column TMEM buffers; four epilogue warps add the finished
// buffer into a per-CTA fp64 partial (L2-resident, transposed so the stores coalesce) while
// the MMAs fill the other. A reduce kernel sums the replicas in fixed order and scales by
// 2^-2e exactly. Deterministic for a given launch shape.
#include <cuda_fp16.h>
#include <math.h>
#include <stdlib.h>

#include "common.cuh"

namespace skc {

namespace {
constexpr int kKC = 32;       // rows per chunk = 2 K-steps of 16
constexpr int kStages = 4;    // operand stages = fill groups
constexpr int kGroupWarps = 4;
constexpr int kFillWarps = kStages * kGroupWarps;  // warps 0..15
constexpr int kEpi0 = 16;                          // warps 16..19: epilogue (warp % 4 = TMEM lane quarter)
constexpr int kMmaWarp = 20;
constexpr int kWarps = 21;
constexpr int kA = 128, kB = 256;
constexpr int kTileA = kA * kKC * 2;  // bytes per limb tile
constexpr int kTileB = kB * kKC * 2;
constexpr int kStageBytes = 2 * kTileB + 2 * kTileA;  // B hi, B lo, A hi, A lo: 48 KB
constexpr int kSmemBytes = kStages * kStageBytes + 256;
constexpr int kSegRows = 1 << 18;  // rows bucketed per K3b/K3t launch pair (bounds the entry buffer)
constexpr uint32_t kPad = 0xFFFFu;  // entry offset of a padding entry
// instruction descriptor: fp16 x fp16 -> fp32, K-major A and B, N = 256, M = 128
constexpr uint32_t kIdesc = (1u << 4) | ((uint32_t)(kB >> 3) << 17) | ((uint32_t)(kA >> 4) << 24);

// Operand tiles: element (coordinate c, row k) at half offset [c>>3][k>>3][c&7][k&7]: a core
// matrix (8 coordinates x 8 rows) is 128 contiguous bytes; a 128-coordinate block is 4096
// halves, so B's second block follows its first.
// Shared-memory descriptor, SWIZZLE_NONE: LBO = 128 B (next core matrix along K),
// SBO = 512 B (next 8 coordinates), version 1.
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr) {
  return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)(128 >> 4) << 16) | ((uint64_t)(512 >> 4) << 32) | (1ull << 46);
}
__device__ __forceinline__ void mbar_init(uint32_t a, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(a), "r"(count));
}
__device__ __forceinline__ void mbar_arrive(uint32_t a) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(a) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t a, uint32_t parity) {
  // try_wait with a suspend-time hint: a waiting warp sleeps instead of spinning on issue slots
  asm volatile(
      "{\n\t.reg .pred P1;\n\tWAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1, %2;\n\t"
      "@!P1 bra WAIT_%=;\n\t}\n" ::"r"(a),
      "r"(parity), "r"(1000000)
      : "memory");
}
__device__ __forceinline__ void sts16(uint32_t a, uint32_t v) {
  asm volatile("st.shared.u16 [%0], %1;" ::"r"(a), "h"((uint16_t)v) : "memory");
}
__device__ __forceinline__ void sts128z(uint32_t a) {
  asm volatile("st.shared.v4.u32 [%0], {%1, %1, %1, %1};" ::"r"(a), "r"(0) : "memory");
}
__device__ __forceinline__ void mma_f16(uint32_t tmem, uint64_t a, uint64_t b, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem),
      "l"(a), "l"(b), "r"(kIdesc), "r"(acc));
}
__device__ __forceinline__ void mma_commit(uint32_t bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar) : "memory");
}

// unit u -> (I, J2): block row I owns the units J2 = floor(I/2) .. nb2 - 1
__device__ __forceinline__ void unit_of(int u, int nb, int nb2, int* I, int* J2) {
  int i = 0;
  while (i < nb) {
    const int c = nb2 - (i >> 1);
    if (u < c) break;
    u -= c;
    ++i;
  }
  *I = i;
  *J2 = (i >> 1) + u;
}
__host__ __device__ __forceinline__ int units_total(int nb) {
  int t = 0;
  for (int i = 0; i < nb; ++i) t += nb / 2 - (i >> 1);
  return t;
}
__device__ __forceinline__ double value_scale(const double* stats) {
  int E = 0;
  frexp(stats[1] > 0.0 && stats[1] <= 1.0e300 ? stats[1] : 1.0, &E);  // x = w * 2^(15 - E): |x| <= 2^15
  return ldexp(1.0, 15 - E);  // applied in fp64, so any exponent range scales exactly
}
}  // namespace

// ---------------------------------------------------------------------------- K3b
// ent: [chunk][stride] entries (offset | hi << 16 | lo << 32), boff: [chunk][nb + 1] entry
// offsets of the 128-coordinate blocks inside the chunk (each block padded to even length)
template <typename V>
__global__ void __launch_bounds__(256) cov_bucket_kernel(const int32_t* __restrict__ idx, const V* __restrict__ val,
                                                        int64_t n, int m, int nb, const double* __restrict__ stats,
                                                        uint64_t* __restrict__ ent, uint32_t* __restrict__ boff,
                                                        int64_t stride) {
  extern __shared__ uint32_t bsm[];  // per warp: cnt[nb], cur[nb]
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t c = (int64_t)blockIdx.x * 8 + warp;
  const int64_t nch = (n + kKC - 1) / kKC;
  if (c >= nch) return;
  uint32_t* cnt = bsm + warp * 2 * nb;
  uint32_t* cur = cnt + nb;
  for (int b = lane; b < nb; b += 32) cnt[b] = 0;
  __syncwarp();
  const int rows = (int)min((int64_t)kKC, n - c * kKC);
  const int32_t* ic = idx + c * kKC * (int64_t)m;
  const V* vc = val + c * kKC * (int64_t)m;
  for (int e = lane; e < rows * m; e += 32) atomicAdd(&cnt[__ldg(ic + e) >> 7], 1u);
  __syncwarp();
  // exclusive scan of the even-padded counts (nb <= 64: two bins per lane)
  uint32_t run = 0;
  uint64_t* ec = ent + c * stride;
  for (int b0 = 0; b0 < nb; b0 += 32) {
    const int b = b0 + lane;
    const uint32_t k = b < nb ? cnt[b] : 0, pk = (k + 1) & ~1u;
    uint32_t x = pk;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, x, o);
      if (lane >= o) x += y;
    }
    const uint32_t start = run + x - pk;
    if (b < nb) {
      cur[b] = start;
      boff[c * (nb + 1) + b] = start;
      if (k & 1) ec[start + k] = kPad;
    }
    run += __shfl_sync(0xFFFFFFFFu, x, 31);
  }
  if (lane == 0) boff[c * (nb + 1) + nb] = run;
  __syncwarp();
  const double xs = value_scale(stats);
  for (int k = 0; k < rows; ++k)
    for (int t = lane; t < m; t += 32) {
      const int j = __ldg(ic + k * m + t);
      const float x = (float)((double)__ldg(vc + k * m + t) * xs);
      const __half h = __float2half_rn(x);
      const uint32_t lo = __half_as_ushort(__float2half_rn(x - __half2float(h)));
      const int cc = j & 127;
      const uint32_t off = (uint32_t)((cc >> 3) * 256 + (cc & 7) * 8 + (k >> 3) * 64 + (k & 7));
      const uint32_t pos = atomicAdd(&cur[j >> 7], 1u);
      ec[pos] = (uint64_t)off | ((uint64_t)__half_as_ushort(h) << 16) | ((uint64_t)lo << 32);
    }
}

// ---------------------------------------------------------------------------- K3t
struct TcParams {
  const uint64_t* ent;
  const uint32_t* boff;
  int64_t stride;   // entries per chunk
  int64_t nch;      // chunks in this segment; replica r owns [nch r / R, nch (r+1) / R)
  int32_t p_pad;
  double* part;     // [replica][unit][256][128] fp64 partials (transposed strip)
  int nunits, replicas, cpw;
};

__global__ void __launch_bounds__(kWarps * 32, 1) cov_tc_kernel(const __grid_constant__ TcParams P) {
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ __align__(8) uint64_t bars[2 * kStages + 4];
  __shared__ uint32_t tmem_base;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nb = P.p_pad / kA, nb2 = P.p_pad / kB;
  const int unit = blockIdx.x % P.nunits, rep = blockIdx.x / P.nunits;
  int I, J2;
  unit_of(unit, nb, nb2, &I, &J2);
  const bool diag = I == 2 * J2 || I == 2 * J2 + 1;  // A's coordinates lie inside B's: A is a sub-tile of B
  const int64_t c0 = P.nch * rep / P.replicas, c1 = P.nch * (rep + 1) / P.replicas;
  const int64_t nchunks = c1 - c0;

  const uint32_t base_sh = (uint32_t)__cvta_generic_to_shared(smem);
  const uint32_t bar_sh = (uint32_t)__cvta_generic_to_shared(bars);
  auto full_bar = [&](int s) { return bar_sh + 8u * s; };
  auto empty_bar = [&](int s) { return bar_sh + 8u * (kStages + s); };
  auto accf_bar = [&](int b) { return bar_sh + 8u * (2 * kStages + b); };
  auto acce_bar = [&](int b) { return bar_sh + 8u * (2 * kStages + 2 + b); };

  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) mbar_init(full_bar(s), kGroupWarps), mbar_init(empty_bar(s), 1);
    for (int b = 0; b < 2; ++b) mbar_init(accf_bar(b), 1), mbar_init(acce_bar(b), 4);
  }
  if (warp == kMmaWarp) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
        (uint32_t)__cvta_generic_to_shared(&tmem_base)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tmem_base;

  if (warp < kFillWarps) {
    // ---------------------------------------------------------------- fill groups
    // group g (warps 4g .. 4g+3) owns stage g and chunks c0 + g + 4i; the next chunk's block
    // offsets are loaded one iteration ahead
    const int g = warp / kGroupWarps, lg = (warp % kGroupWarps) * 32 + lane;
    const uint32_t bh = base_sh + (uint32_t)g * kStageBytes, bl = bh + kTileB, ah = bh + 2 * kTileB,
                   al = ah + kTileA;
    auto offsets = [&](int64_t c, uint32_t* o) {  // o: B start, B mid, B end, A start, A end
      if (c >= c1) return;
      const uint32_t* bo = P.boff + c * (nb + 1);
      o[0] = __ldg(bo + 2 * J2), o[1] = __ldg(bo + 2 * J2 + 1), o[2] = __ldg(bo + 2 * J2 + 2);
      o[3] = __ldg(bo + I), o[4] = __ldg(bo + I + 1);
    };
    uint32_t oc[5] = {0, 0, 0, 0, 0}, on[5] = {0, 0, 0, 0, 0};
    offsets(c0 + g, oc);
    for (int64_t i = 0;; ++i) {
      const int64_t c = c0 + g + (int64_t)kStages * i;
      if (c >= c1) break;
      offsets(c + kStages, on);
      mbar_wait(empty_bar(g), (uint32_t)((i & 1) ^ 1));
      for (int q = lg; q < kStageBytes / 16; q += kGroupWarps * 32) sts128z(bh + 16u * q);
      asm volatile("bar.sync %0, %1;" ::"r"(1 + g), "n"(kGroupWarps * 32) : "memory");
      const uint64_t* ec = P.ent + c * P.stride;
      const int nbt = (int)(oc[2] - oc[0]), nat = diag ? 0 : (int)(oc[4] - oc[3]);
      constexpr int kU = 8;  // entries per lane in flight
      for (int q0 = lg; q0 < nbt + nat; q0 += kU * kGroupWarps * 32) {
        uint64_t v[kU];
#pragma unroll
        for (int u = 0; u < kU; ++u) {
          const int q = q0 + u * kGroupWarps * 32;
          v[u] = kPad;
          if (q < nbt + nat) v[u] = __ldg(ec + (q < nbt ? oc[0] + q : oc[3] + (q - nbt)));
        }
#pragma unroll
        for (int u = 0; u < kU; ++u) {
          const int q = q0 + u * kGroupWarps * 32;
          const uint32_t off = (uint32_t)v[u] & 0xFFFFu;
          if (off == kPad) continue;
          const bool inb = q < nbt;
          const uint32_t o2 = 2u * (off + (inb && oc[0] + q >= oc[1] ? 4096u : 0u));
          sts16((inb ? bh : ah) + o2, (uint32_t)(v[u] >> 16));
          sts16((inb ? bl : al) + o2, (uint32_t)(v[u] >> 32));
        }
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncwarp();
      if (lane == 0) mbar_arrive(full_bar(g));
#pragma unroll
      for (int t = 0; t < 5; ++t) oc[t] = on[t];
    }
  } else if (warp == kMmaWarp) {
    // ---------------------------------------------------------------- MMA issuer
    if (lane == 0) {
      for (int64_t c = 0; c < nchunks; ++c) {
        const int64_t w = c / P.cpw;
        const int b = (int)(w & 1);
        const bool first = c % P.cpw == 0;
        if (first) mbar_wait(acce_bar(b), (uint32_t)(((w >> 1) & 1) ^ 1));
        const int s = (int)(c % kStages);
        mbar_wait(full_bar(s), (uint32_t)((c / kStages) & 1));
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t st = base_sh + (uint32_t)s * kStageBytes;
        const uint32_t bh = st, bl = st + kTileB;
        const uint32_t ah = diag ? bh + (uint32_t)(I - 2 * J2) * kTileA : st + 2 * kTileB;
        const uint32_t al = diag ? bl + (uint32_t)(I - 2 * J2) * kTileA : st + 2 * kTileB + kTileA;
        const uint32_t d = tmem + (uint32_t)b * kB;
#pragma unroll
        for (int ks = 0; ks < kKC / 16; ++ks) {
          const uint32_t o = (uint32_t)ks * 256;  // two core matrices along K
          mma_f16(d, sdesc(ah + o), sdesc(bh + o), (first && ks == 0) ? 0u : 1u);
          mma_f16(d, sdesc(ah + o), sdesc(bl + o), 1u);
          mma_f16(d, sdesc(al + o), sdesc(bh + o), 1u);
        }
        mma_commit(empty_bar(s));
        if (c % P.cpw == P.cpw - 1 || c == nchunks - 1) mma_commit(accf_bar(b));
      }
    }
    __syncwarp();
  } else {
    // ---------------------------------------------------------------- epilogue warps
    const int q = (warp - kEpi0) & 3;  // TMEM lanes 32q .. 32q + 31 = strip rows (warp % 4 == q)
    const int i = 32 * q + lane;
    double* part = P.part + ((size_t)rep * P.nunits + unit) * (size_t)(kA * kB);
    const int64_t nwin = (nchunks + P.cpw - 1) / P.cpw;
    for (int64_t w = 0; w < nwin; ++w) {
      const int b = (int)(w & 1);
      mbar_wait(accf_bar(b), (uint32_t)((w >> 1) & 1));
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
#pragma unroll 1
      for (int c0c = 0; c0c < kB; c0c += 16) {
        uint32_t v[16];
        const uint32_t addr = tmem + ((uint32_t)(32 * q) << 16) + (uint32_t)(b * kB + c0c);
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
            : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
              "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
            : "r"(addr));
        double* pp = part + (size_t)c0c * kA + i;
        double o[16];  // all partial loads in flight before the first store
#pragma unroll
        for (int j = 0; j < 16; ++j) o[j] = pp[(size_t)j * kA];
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
        for (int j = 0; j < 16; ++j) pp[(size_t)j * kA] = dadd(o[j], (double)__uint_as_float(v[j]));
      }
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      __syncwarp();
      if (lane == 0) mbar_arrive(acce_bar(b));
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == kMmaWarp) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

// tri[a, b] += 2^-2e * sum over replicas of the strip partials, a <= b
__global__ void cov_tc_reduce_kernel(const double* __restrict__ part, int nunits, int replicas, int32_t p_pad,
                                     const double* __restrict__ stats, double* __restrict__ tri) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x, a = blockIdx.y;
  if (b >= p_pad || b < a) return;
  int E = 0;
  frexp(stats[1] > 0.0 && stats[1] <= 1.0e300 ? stats[1] : 1.0, &E);
  const double inv = ldexp(1.0, 2 * (E - 15));
  const int nb2 = p_pad / kB, I = a / kA, J2 = b / kB;
  int u = 0;
  for (int i = 0; i < I; ++i) u += nb2 - (i >> 1);
  u += J2 - (I >> 1);
  double s = 0.0;
  for (int r = 0; r < replicas; ++r)
    s = dadd(s, part[((size_t)r * nunits + u) * (size_t)(kA * kB) + (size_t)(b - J2 * kB) * kA + (a - I * kA)]);
  double* t = tri + ((int64_t)a * p_pad - (int64_t)a * (a - 1) / 2) + (b - a);
  *t = dadd(*t, dmul(s, inv));
}

static int tc_replicas(int nunits, int64_t n) {
  int r = sm_count() / nunits;
  if (r < 1) r = 1;
  const int64_t maxr = (n + 32 * kKC - 1) / (32 * kKC);  // at least ~32 chunks per replica
  if (r > maxr) r = (int)(maxr < 1 ? 1 : maxr);
  return r;
}
static int64_t seg_stride(int32_t m, int nb) { return ((int64_t)kKC * m + nb + 1) & ~(int64_t)1; }

bool covtc_supported(int32_t p_pad) { return p_pad >= kB && p_pad % kB == 0 && p_pad <= 8192; }

// workspace: [partials][entries of one segment][block offsets of one segment]
size_t covtc_ws(int64_t n, int32_t m, int32_t p_pad) {
  const int nb = p_pad / kA, nu = units_total(nb);
  const int64_t seg = n < kSegRows ? n : kSegRows, sch = (seg + kKC - 1) / kKC;
  return (size_t)nu * tc_replicas(nu, seg) * kA * kB * sizeof(double) + (size_t)sch * seg_stride(m, nb) * 8 +
         (size_t)sch * (nb + 1) * 4 + 64;
}

int covtc_launch(const int32_t* idx, const void* val, int val_f64, int64_t n, int32_t m, int32_t p_pad,
                 const double* stats, double* tri, void* ws, cudaStream_t st) {
  if (n == 0) return SKC_OK;
  const int nb = p_pad / kA;
  TcParams H{};
  H.p_pad = p_pad;
  H.nunits = units_total(nb);
  const int64_t seg = n < kSegRows ? n : kSegRows, sch = (seg + kKC - 1) / kKC;
  H.replicas = tc_replicas(H.nunits, seg);
  H.cpw = 32;  // window of 1024 rows per fp32 TMEM accumulation
  if (const char* e = getenv("SKC_COVTC_WINDOW")) H.cpw = atoi(e) > 0 ? atoi(e) : H.cpw;
  H.part = reinterpret_cast<double*>(ws);
  const size_t part_bytes = (size_t)H.nunits * H.replicas * kA * kB * sizeof(double);
  H.stride = seg_stride(m, nb);
  uint64_t* ent = reinterpret_cast<uint64_t*>(static_cast<char*>(ws) + part_bytes);
  uint32_t* boff = reinterpret_cast<uint32_t*>(ent + sch * H.stride);
  H.ent = ent;
  H.boff = boff;
  cudaMemsetAsync(ws, 0, part_bytes, st);
  cudaFuncSetAttribute(cov_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemBytes);
  const size_t bsmem = (size_t)8 * 2 * nb * sizeof(uint32_t);
  cudaFuncSetAttribute(cov_bucket_kernel<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bsmem);
  cudaFuncSetAttribute(cov_bucket_kernel<double>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bsmem);
  int rc;
  for (int64_t r0 = 0; r0 < n; r0 += kSegRows) {
    const int64_t rows = n - r0 < kSegRows ? n - r0 : kSegRows, nch = (rows + kKC - 1) / kKC;
    const unsigned bgrid = (unsigned)((nch + 7) / 8);
    if (val_f64)
      cov_bucket_kernel<double><<<bgrid, 256, bsmem, st>>>(idx + r0 * m, static_cast<const double*>(val) + r0 * m,
                                                          rows, m, nb, stats, ent, boff, H.stride);
    else
      cov_bucket_kernel<float><<<bgrid, 256, bsmem, st>>>(idx + r0 * m, static_cast<const float*>(val) + r0 * m,
                                                         rows, m, nb, stats, ent, boff, H.stride);
    if ((rc = check_launch("cov_bucket_kernel"))) return rc;
    H.nch = nch;
    cov_tc_kernel<<<H.nunits * H.replicas, kWarps * 32, kSmemBytes, st>>>(H);
    if ((rc = check_launch("cov_tc_kernel"))) return rc;
  }
  cov_tc_reduce_kernel<<<dim3((p_pad + 255) / 256, p_pad), 256, 0, st>>>(H.part, H.nunits, H.replicas, p_pad, stats,
                                                                         tri);
  return check_launch("cov_tc_reduce_kernel");
}

}  // namespace skc
