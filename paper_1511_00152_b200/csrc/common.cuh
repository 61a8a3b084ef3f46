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

// splitmix64 finalizer (_hash.py:20-26). 64-bit ops lower to 32-bit IMAD/SHF/LOP3.
__host__ __device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * kMix1;
  z = (z ^ (z >> 27)) * kMix2;
  return z ^ (z >> 31);
}

__device__ __forceinline__ uint32_t lanemask_lt() {
  uint32_t r;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(r));
  return r;
}

// fp64 add/mul with explicit round-to-nearest: never contracted into FMA, which keeps
// the reference's separate-rounding order (transform.py:165-170, cluster.py:183).
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
