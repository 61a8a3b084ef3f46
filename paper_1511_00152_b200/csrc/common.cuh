// Shared device helpers for the sm_100a sketch kernels.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <string>

#include "../../include/sketchcu.h"

namespace skc {

constexpr uint64_t kGamma = 0x9E3779B97F4A7C15ULL;  // _hash.py:11
constexpr uint64_t kMix1 = 0xBF58476D1CE4E5B9ULL;   // _hash.py:12
constexpr uint64_t kMix2 = 0x94D049BB133111EBULL;   // _hash.py:13
constexpr uint64_t kTagSign = 0x53494748ULL;        // _hash.py:16
constexpr uint64_t kTagSample = 0x53414D50ULL;      // _hash.py:17
constexpr uint64_t kTagPhilox = 0x50484C58ULL;      // "PHLX": Philox sampler key derivation

// splitmix64 finalizer (_hash.py:20-26). 64-bit ops lower to 32-bit IMAD/SHF/LOP3.
__host__ __device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * kMix1;
  z = (z ^ (z >> 27)) * kMix2;
  return z ^ (z >> 31);
}

// Philox4x32-10 (Salmon et al., SC'11): counter (4 x u32) and key (2 x u32) -> 4 x u32.
struct Philox4 {
  uint32_t x, y, z, w;
};
__host__ __device__ __forceinline__ Philox4 philox4x32_10(Philox4 c, uint32_t k0, uint32_t k1) {
  constexpr uint32_t kM0 = 0xD2511F53u, kM1 = 0xCD9E8D57u, kW0 = 0x9E3779B9u, kW1 = 0xBB67AE85u;
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    const uint64_t p0 = (uint64_t)kM0 * c.x, p1 = (uint64_t)kM1 * c.z;
    c = Philox4{(uint32_t)(p1 >> 32) ^ c.y ^ k0, (uint32_t)p1, (uint32_t)(p0 >> 32) ^ c.w ^ k1, (uint32_t)p0};
    k0 += kW0;
    k1 += kW1;
  }
  return c;
}

__device__ __forceinline__ uint32_t lanemask_lt() {
  uint32_t r;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(r));
  return r;
}

// fp64 add/mul with explicit round-to-nearest: never contracted into FMA, which keeps
// the reference's separate-rounding order (transform.py:104-109, cluster.py:183).
__device__ __forceinline__ double dadd(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double dsub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double dmul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ float fadd(float a, float b) { return __fadd_rn(a, b); }
__device__ __forceinline__ float fsub(float a, float b) { return __fsub_rn(a, b); }
__device__ __forceinline__ float fmul(float a, float b) { return __fmul_rn(a, b); }

template <typename T> struct Arith;
template <> struct Arith<float> {
  static __device__ __forceinline__ float add(float a, float b) { return fadd(a, b); }
  static __device__ __forceinline__ float sub(float a, float b) { return fsub(a, b); }
  static __device__ __forceinline__ float mul(float a, float b) { return fmul(a, b); }
  static __device__ __forceinline__ float flip(float a, uint32_t neg) {
    return __int_as_float(__float_as_int(a) ^ (int)(neg << 31));
  }
};
template <> struct Arith<double> {
  static __device__ __forceinline__ double add(double a, double b) { return dadd(a, b); }
  static __device__ __forceinline__ double sub(double a, double b) { return dsub(a, b); }
  static __device__ __forceinline__ double mul(double a, double b) { return dmul(a, b); }
  static __device__ __forceinline__ double flip(double a, uint32_t neg) {
    return __longlong_as_double(__double_as_longlong(a) ^ ((long long)neg << 63));
  }
};

template <typename T> __device__ __forceinline__ T load_val(const void* p, int64_t i);
template <> __device__ __forceinline__ float load_val<float>(const void* p, int64_t i) {
  return __ldg(reinterpret_cast<const float*>(p) + i);
}
template <> __device__ __forceinline__ double load_val<double>(const void* p, int64_t i) {
  return __ldg(reinterpret_cast<const double*>(p) + i);
}

// ---- host-side error plumbing -------------------------------------------------
void set_error(const std::string& msg);
int fail(int code, const std::string& msg);
int check_launch(const char* what);
int sm_count();

}  // namespace skc
