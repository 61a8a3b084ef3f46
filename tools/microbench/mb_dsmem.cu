// Shared-memory atomic throughput: CTA-local ATOMS vs distributed shared memory atomics
// across a thread-block cluster (atom.shared::cluster after mapa). 1 CTA per SM, 32 warps,
// ~200 KB of int32 words per CTA, random word and (for DSMEM) random CTA rank per update;
// every update uses its returned old value (as the covariance kernel's carry test does).
// Also reports how many clusters of each size can be co-resident.
// build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o mb_dsmem mb_dsmem.cu
#include <cooperative_groups.h>
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s @%d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

constexpr int kWords = 50 * 1024;  // 200 KB

__device__ __forceinline__ uint32_t xs(uint32_t& s) { s ^= s << 13; s ^= s >> 17; s ^= s << 5; return s; }

// mode 0: local atom.shared (cta); mode 1: cluster atom to own rank; mode 2: cluster atom to random rank
__global__ void __launch_bounds__(1024, 1) k_atom(uint32_t* sink, int iters, int mode, int csize) {
  extern __shared__ uint32_t w[];
  for (int i = threadIdx.x; i < kWords; i += blockDim.x) w[i] = 0x80000000u;
  cooperative_groups::this_cluster().sync();
  const uint32_t base = (uint32_t)__cvta_generic_to_shared(w);
  uint32_t rank;
  asm("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
  uint32_t s = 0x9E3779B9u ^ (blockIdx.x * 1024 + threadIdx.x) * 2654435761u;
  uint32_t acc = 0;
  for (int it = 0; it < iters; ++it) {
    const uint32_t r = xs(s);
    const uint32_t off = base + 4 * (r % kWords);
    uint32_t old;
    if (mode == 0) {
      asm volatile("atom.shared.add.u32 %0, [%1], %2;" : "=r"(old) : "r"(off), "r"(r & 0xFFFF) : "memory");
    } else {
      const uint32_t tgt = mode == 1 ? rank : (r >> 24) % csize;
      uint32_t ra;
      asm("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(off), "r"(tgt));
      asm volatile("atom.shared::cluster.add.u32 %0, [%1], %2;" : "=r"(old) : "r"(ra), "r"(r & 0xFFFF) : "memory");
    }
    if (old + (r & 0xFFFF) < old) acc += 1;  // carry test on the returned value
  }
  cooperative_groups::this_cluster().sync();
  if (acc == 0x12345) sink[0] = acc;
}

int main() {
  int sms;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  const size_t smem = kWords * 4;
  CK(cudaFuncSetAttribute(k_atom, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  CK(cudaFuncSetAttribute(k_atom, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  uint32_t* sink;
  CK(cudaMalloc(&sink, 16));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int iters = 4096;
  struct Cfg { int mode, csize; const char* name; } cfgs[] = {
      {0, 1, "local atom.shared"},          {1, 2, "cluster atom, own rank (C=2)"},
      {2, 2, "cluster atom, random rank C=2"}, {2, 4, "cluster atom, random rank C=4"},
      {2, 8, "cluster atom, random rank C=8"}, {2, 10, "cluster atom, random rank C=10"},
      {2, 12, "cluster atom, random rank C=12"}, {2, 16, "cluster atom, random rank C=16"}};
  for (auto c : cfgs) {
    cudaLaunchConfig_t lc = {};
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = c.csize;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    lc.attrs = at;
    lc.numAttrs = 1;
    lc.blockDim = dim3(1024);
    lc.dynamicSmemBytes = smem;
    lc.gridDim = dim3(c.csize);
    int ncl = 0;
    cudaError_t oe = cudaOccupancyMaxActiveClusters(&ncl, k_atom, &lc);
    if (oe != cudaSuccess || ncl == 0) {
      printf("%-34s cluster size %2d: not launchable (%s)\n", c.name, c.csize, cudaGetErrorString(oe));
      cudaGetLastError();
      continue;
    }
    lc.gridDim = dim3(ncl * c.csize);
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(e0);
      CK(cudaLaunchKernelEx(&lc, k_atom, sink, iters, c.mode, c.csize));
      cudaEventRecord(e1);
      CK(cudaEventSynchronize(e1));
    }
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double ups = (double)ncl * c.csize * 1024 * iters / (ms * 1e-3);
    printf("%-34s clusters %3d (%3d SMs busy): %.3e updates/s = %.2f /busy-SM/cycle @1.965GHz\n", c.name, ncl,
           ncl * c.csize, ups, ups / (ncl * c.csize) / 1.965e9);
  }
  return 0;
}
