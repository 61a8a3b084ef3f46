// Check of the hand-built UMMA path the tensor-core covariance kernel uses: fp16 K-major
// no-swizzle operand tiles in the core-matrix layout [c>>3][k>>3][c&7][k&7], instruction and
// shared-memory descriptors, tcgen05.mma kind::f16 M=128 N=256 K=16 into TMEM, commit to an
// mbarrier, tcgen05.ld 32x32b.x32 back. Then a timed loop of 3 MMAs per K-step (the kernel's
// hi*hi + hi*lo + lo*hi) for the per-SM rate.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mb_umma mb_umma.cu
#include <cuda_fp16.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#include <cmath>
#include <vector>

constexpr int M = 128, N = 256, KC = 32;  // chunk of 32 rows = 2 K-steps
__host__ __device__ inline int off_elem(int c, int k) {  // element offset in a [C][KC] tile
  return (c >> 3) * (KC / 8) * 64 + (k >> 3) * 64 + (c & 7) * 8 + (k & 7);
}
__device__ inline uint64_t sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | (1ull << 46);
}
constexpr uint32_t kIdesc = (1u << 4) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);

__device__ inline void mma(uint32_t tmem, uint64_t a, uint64_t b, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem),
      "l"(a), "l"(b), "r"(kIdesc), "r"(acc));
}

__global__ void umma_check(const __half* A, const __half* B, float* D, int reps) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __half* sa = reinterpret_cast<__half*>(sm);
  __half* sb = sa + M * KC;
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  for (int i = threadIdx.x; i < M * KC; i += blockDim.x) sa[i] = A[i];
  for (int i = threadIdx.x; i < N * KC; i += blockDim.x) sb[i] = B[i];
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  const uint32_t bar_a = (uint32_t)__cvta_generic_to_shared(&bar);
  if (threadIdx.x == 0) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar_a));
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(
        (uint32_t)__cvta_generic_to_shared(&tbase)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tbase;
  const uint32_t a0 = (uint32_t)__cvta_generic_to_shared(sa), b0 = (uint32_t)__cvta_generic_to_shared(sb);
  long long t0 = 0, t1 = 0;
  if (threadIdx.x == 0) {
    t0 = clock64();
    for (int r = 0; r < reps; ++r)
      for (int s = 0; s < KC / 16; ++s)
        for (int l = 0; l < (reps > 1 ? 3 : 1); ++l)
          mma(tmem, sdesc(a0 + s * 256, 128, (KC / 8) * 128), sdesc(b0 + s * 256, 128, (KC / 8) * 128),
              (r | s | l) != 0);
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar_a));
  }
  // wait for phase 0
  asm volatile(
      "{\n\t.reg .pred P1;\n\tWAIT:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n\t"
      "@!P1 bra WAIT;\n\t}\n" ::"r"(bar_a));
  if (threadIdx.x == 0) {
    t1 = clock64();
    if (reps > 1) printf("%d x %d MMAs (128x256x16 f16): %lld cycles, %.1f cycles/MMA\n", reps, 3 * KC / 16,
                         t1 - t0, (double)(t1 - t0) / (reps * 3 * KC / 16));
  }
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int c0 = 0; c0 < N; c0 += 32) {
    uint32_t v[32];
    const uint32_t addr = tmem + ((uint32_t)(warp * 32) << 16) + c0;
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,"
        "%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
          "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),
          "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]),
          "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
        : "r"(addr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    for (int j = 0; j < 32; ++j) D[(warp * 32 + lane) * N + c0 + j] = __uint_as_float(v[j]);
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tmem));
}

int main() {
  std::vector<float> a(M * KC), b(N * KC);
  std::vector<__half> ha(M * KC), hb(N * KC);
  srand(1);
  for (int c = 0; c < M; ++c)
    for (int k = 0; k < KC; ++k) {
      const float x = (rand() % 2001 - 1000) / 256.0f;
      a[c * KC + k] = __half2float(__float2half(x));
      ha[off_elem(c, k)] = __float2half(x);
    }
  for (int c = 0; c < N; ++c)
    for (int k = 0; k < KC; ++k) {
      const float x = (rand() % 2001 - 1000) / 256.0f;
      b[c * KC + k] = __half2float(__float2half(x));
      hb[off_elem(c, k)] = __float2half(x);
    }
  __half *dA, *dB;
  float* dD;
  cudaMalloc(&dA, M * KC * 2);
  cudaMalloc(&dB, N * KC * 2);
  cudaMalloc(&dD, M * N * 4);
  cudaMemcpy(dA, ha.data(), M * KC * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, hb.data(), N * KC * 2, cudaMemcpyHostToDevice);
  const int smem = (M + N) * KC * 2;
  cudaFuncSetAttribute(umma_check, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  umma_check<<<1, 128, smem>>>(dA, dB, dD, 1);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    printf("error %s\n", cudaGetErrorString(e));
    return 1;
  }
  std::vector<float> d(M * N);
  cudaMemcpy(d.data(), dD, M * N * 4, cudaMemcpyDeviceToHost);
  double maxerr = 0, maxref = 0;
  for (int i = 0; i < M; ++i)
    for (int j = 0; j < N; ++j) {
      double s = 0;
      for (int k = 0; k < KC; ++k) s += (double)a[i * KC + k] * b[j * KC + k];
      maxerr = fmax(maxerr, fabs(s - d[i * N + j]));
      maxref = fmax(maxref, fabs(s));
    }
  printf("umma check: max |err| %.3e of max |ref| %.3e -> %s\n", maxerr, maxref, maxerr <= 1e-5 * maxref ? "OK" : "FAIL");
  umma_check<<<1, 128, smem>>>(dA, dB, dD, 2000);
  e = cudaDeviceSynchronize();
  if (e != cudaSuccess) printf("error %s\n", cudaGetErrorString(e));
  return maxerr <= 1e-5 * maxref ? 0 : 1;
}
