// Microbenchmarks that decide the covariance / hashing design on B200.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mb mb.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#define CK(x) do{cudaError_t e=(x); if(e!=cudaSuccess){printf("CUDA %s @%d\n",cudaGetErrorString(e),__LINE__); return 1;}}while(0)

__device__ __forceinline__ uint32_t hsh(uint32_t x){ x ^= x>>16; x*=0x7feb352dU; x^=x>>15; x*=0x846ca68bU; x^=x>>16; return x; }
constexpr int NE = 48*1024; // entries per smem band (192 KB fp32)

template<int MODE>
__global__ void __launch_bounds__(256) smem_scatter(float* out, int iters, uint32_t seed){
  extern __shared__ float acc[];
  for(int i=threadIdx.x;i<NE;i+=blockDim.x) acc[i]=0;
  __syncthreads();
  uint32_t s = hsh(seed ^ (blockIdx.x*256+threadIdx.x));
  float v = 1.0f;
  for(int it=0; it<iters; ++it){
    s = s*1664525u + 1013904223u;
    uint32_t a = (s>>8) % NE;
    if(MODE==0) atomicAdd(&acc[a], v);                 // CAS loop
    else if(MODE==1) atomicAdd((int*)&acc[a], 1);      // native ATOMS.ADD
    else { acc[a] += v; }                               // racy RMW (throughput ceiling)
  }
  __syncthreads();
  float t=0; for(int i=threadIdx.x;i<NE;i+=blockDim.x) t+=acc[i];
  atomicAdd(out, t);
}

template<typename T>
__global__ void gmem_red(T* acc, int nacc, int iters, uint32_t seed){
  uint32_t s = hsh(seed ^ (blockIdx.x*blockDim.x+threadIdx.x));
  for(int it=0; it<iters; ++it){ s = s*1664525u + 1013904223u; atomicAdd(&acc[(s>>4)%nacc], (T)1); }
}

__device__ __forceinline__ uint64_t mix64(uint64_t z){
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL; z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL; return z ^ (z >> 31);
}
__global__ void hashk(uint32_t* out, int iters, uint32_t thr){
  uint64_t k = 0x9E3779B97F4A7C15ULL * (blockIdx.x*blockDim.x+threadIdx.x+1);
  uint32_t cnt=0;
  for(int it=0; it<iters; ++it){ k += 32ULL*0x9E3779B97F4A7C15ULL; uint64_t z = mix64(k); cnt += (uint32_t)(z>>32) < thr; }
  out[blockIdx.x*blockDim.x+threadIdx.x]=cnt;
}
template<typename T>
__global__ void addk(T* out, int iters){
  T a[8]; for(int i=0;i<8;i++) a[i]=(T)(threadIdx.x+i);
  for(int it=0; it<iters; ++it){
#pragma unroll
    for(int i=0;i<8;i+=2){ T x=a[i], y=a[i+1]; a[i]=x+y; a[i+1]=x-y; }
#pragma unroll
    for(int i=0;i<4;i++){ T x=a[i], y=a[i+4]; a[i]=x+y; a[i+4]=x-y; }
  }
  T t=0; for(int i=0;i<8;i++) t+=a[i]; out[blockIdx.x*blockDim.x+threadIdx.x]=t;
}

int main(){
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0,e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  float* outf; CK(cudaMalloc(&outf, 1<<24));
  float ms;
  // smem scatter
  const char* names[3]={"smem f32 atomicAdd (CAS)","smem i32 atomicAdd (ATOMS.ADD)","smem f32 racy RMW"};
  for(int mode=0; mode<3; ++mode){
    int iters=4096; int grid=sms*1; size_t sm=NE*4;
    auto f = mode==0? smem_scatter<0> : mode==1? smem_scatter<1> : smem_scatter<2>;
    CK(cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
    f<<<grid,256,sm>>>(outf, iters, 1); CK(cudaDeviceSynchronize());
    cudaEventRecord(e0); f<<<grid,256,sm>>>(outf, iters, 2); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms,e0,e1);
    double ups = (double)grid*256*iters/(ms*1e-3);
    printf("%-36s %.3e updates/s  (%.2f /SM/cycle @1.9GHz)\n", names[mode], ups, ups/sms/1.9e9);
  }
  // global red
  for(int sz : {1<<19, 1<<21, 1<<24}){
    float* af; double* ad; CK(cudaMalloc(&af, sz*4)); CK(cudaMalloc(&ad, sz*8));
    int iters=1024, grid=sms*8;
    gmem_red<float><<<grid,256>>>(af, sz, iters, 1); CK(cudaDeviceSynchronize());
    cudaEventRecord(e0); gmem_red<float><<<grid,256>>>(af, sz, iters, 2); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms,e0,e1); printf("global REDG.F32 into %8d entries: %.3e updates/s\n", sz, (double)grid*256*iters/(ms*1e-3));
    cudaEventRecord(e0); gmem_red<double><<<grid,256>>>(ad, sz, iters, 2); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms,e0,e1); printf("global REDG.F64 into %8d entries: %.3e updates/s\n", sz, (double)grid*256*iters/(ms*1e-3));
    cudaFree(af); cudaFree(ad);
  }
  { int iters=1<<14, grid=sms*8; uint32_t* o; CK(cudaMalloc(&o, grid*256*4));
    hashk<<<grid,256>>>(o, iters, 1u<<28); CK(cudaDeviceSynchronize());
    cudaEventRecord(e0); hashk<<<grid,256>>>(o, iters, 1u<<28); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms,e0,e1); printf("splitmix64 keys+threshold: %.3e keys/s\n", (double)grid*256*iters/(ms*1e-3)); }
  { int iters=1<<14, grid=sms*8; double* o; CK(cudaMalloc(&o, grid*256*8));
    addk<float><<<grid,256>>>((float*)o, iters); CK(cudaDeviceSynchronize());
    cudaEventRecord(e0); addk<float><<<grid,256>>>((float*)o, iters); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms,e0,e1); printf("fp32 butterfly add/sub: %.3e ops/s\n", (double)grid*256*iters*16/(ms*1e-3));
    cudaEventRecord(e0); addk<double><<<grid,256>>>(o, iters); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms,e0,e1); printf("fp64 butterfly add/sub: %.3e ops/s\n", (double)grid*256*iters*16/(ms*1e-3)); }
  return 0;
}
