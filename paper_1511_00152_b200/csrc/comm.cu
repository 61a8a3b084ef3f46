// Collectives of the sample-sharded path: ONE fp64 SUM allreduce per pass of the
// packed moments [acc | stats | triangle], and ONE per Lloyd iteration of the packed K-means
// exchange [sums | counts | sizes | changed | objective | per-rank (max d2min, its global row)].
// The reference has no distributed layer; its spec allows "parallel partial sums
// then deterministic ordered combine", which these sums implement.
//
// NCCL is loaded at run time (dlopen "libnccl.so.2"): a process that already loaded NCCL (e.g.
// through torch) shares that copy, and the library has no link-time NCCL dependency. A C
// consumer creates communicators with skc_nccl_get_unique_id / skc_nccl_comm_init_rank or
// passes its own ncclComm_t. NCCL failures return SKC_ENCCL.
#include <dlfcn.h>
#include <string.h>

#include <mutex>
#include <string>

#include "common.cuh"

namespace skc {
namespace {

typedef int (*GetUniqueIdFn)(void*);
typedef int (*CommInitRankFn)(void**, int, const void*, int);  // ncclUniqueId passed by value: 128 bytes
typedef int (*CommDestroyFn)(void*);
typedef int (*AllReduceFn)(const void*, void*, size_t, int, int, void*, cudaStream_t);
typedef const char* (*ErrStrFn)(int);

struct Nccl {
  void* h = nullptr;
  GetUniqueIdFn get_id = nullptr;
  void* init_rank = nullptr;
  CommDestroyFn destroy = nullptr;
  AllReduceFn allreduce = nullptr;
  ErrStrFn errstr = nullptr;
  std::string why;
};

constexpr int kNcclSum = 0;      // ncclSum (nccl.h)
constexpr int kNcclFloat64 = 8;  // ncclFloat64 (nccl.h)

Nccl& nccl() {
  static Nccl N;
  static std::once_flag once;
  std::call_once(once, [] {
    const char* names[] = {"libnccl.so.2", "libnccl.so"};
    for (const char* nm : names) {
      N.h = dlopen(nm, RTLD_NOW | RTLD_GLOBAL);
      if (N.h) break;
    }
    if (!N.h) {
      N.why = std::string("libnccl.so.2 not loadable: ") + (dlerror() ? dlerror() : "?");
      return;
    }
    N.get_id = reinterpret_cast<GetUniqueIdFn>(dlsym(N.h, "ncclGetUniqueId"));
    N.init_rank = dlsym(N.h, "ncclCommInitRank");
    N.destroy = reinterpret_cast<CommDestroyFn>(dlsym(N.h, "ncclCommDestroy"));
    N.allreduce = reinterpret_cast<AllReduceFn>(dlsym(N.h, "ncclAllReduce"));
    N.errstr = reinterpret_cast<ErrStrFn>(dlsym(N.h, "ncclGetErrorString"));
    if (!N.get_id || !N.init_rank || !N.destroy || !N.allreduce) N.why = "libnccl.so.2 lacks a required symbol";
  });
  return N;
}

int nccl_fail(int rc, const char* what) {
  Nccl& N = nccl();
  return fail(SKC_ENCCL, std::string(what) + ": " + (N.errstr ? N.errstr(rc) : "nccl error") + " (" +
                             std::to_string(rc) + ")");
}

struct UniqueId {
  char internal[128];
};
typedef int (*CommInitRankByValue)(void**, int, UniqueId, int);

// K-means exchange layout (fp64): [sums p*K | counts p*K | sizes K | changed | objective |
// per rank r: (max d2min, global row of its first argmax)]
__global__ void kmeans_pack_kernel(const double* __restrict__ sums, const int64_t* __restrict__ counts,
                                   const int64_t* __restrict__ sizes, const int64_t* __restrict__ out,
                                   const double* __restrict__ d2max, const double* __restrict__ obj, int64_t pk, int K,
                                   int rank, int world, int64_t col0, double* __restrict__ buf) {
  const int64_t total = 2 * pk + K + 2 + 2 * (int64_t)world;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    double v = 0.0;
    if (i < pk) v = sums[i];
    else if (i < 2 * pk) v = (double)counts[i - pk];  // exact below 2^53
    else if (i < 2 * pk + K) v = (double)sizes[i - 2 * pk];
    else if (i == 2 * pk + K) v = (double)out[0];
    else if (i == 2 * pk + K + 1) v = *obj;
    else {
      const int64_t s = i - (2 * pk + K + 2);
      if (s / 2 == rank) v = (s & 1) ? (out[1] >= 0 ? (double)(col0 + out[1]) : -1.0) : *d2max;
    }
    buf[i] = v;
  }
}

__global__ void kmeans_unpack_kernel(const double* __restrict__ buf, int64_t pk, int K, double* __restrict__ sums,
                                     int64_t* __restrict__ counts, int64_t* __restrict__ sizes) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < 2 * pk + K; i += (int64_t)gridDim.x * blockDim.x) {
    if (i < pk) sums[i] = buf[i];
    else if (i < 2 * pk) counts[i - pk] = (int64_t)buf[i];
    else sizes[i - 2 * pk] = (int64_t)buf[i];
  }
}

}  // namespace
}  // namespace skc

using namespace skc;

extern "C" {

int skc_nccl_get_unique_id(void* id_out) {
  Nccl& N = nccl();
  if (!N.why.empty()) return fail(SKC_ENCCL, N.why);
  if (id_out == nullptr) return fail(SKC_EPARAM, "id_out is NULL");
  const int rc = N.get_id(id_out);
  return rc ? nccl_fail(rc, "ncclGetUniqueId") : SKC_OK;
}

int skc_nccl_comm_init_rank(void** comm_out, int32_t nranks, const void* id, int32_t rank) {
  Nccl& N = nccl();
  if (!N.why.empty()) return fail(SKC_ENCCL, N.why);
  if (comm_out == nullptr || id == nullptr) return fail(SKC_EPARAM, "comm_out and id are required");
  if (nranks < 1 || rank < 0 || rank >= nranks) return fail(SKC_EPARAM, "need 0 <= rank < nranks");
  UniqueId u;
  memcpy(u.internal, id, sizeof(u.internal));
  const int rc = reinterpret_cast<CommInitRankByValue>(N.init_rank)(comm_out, nranks, u, rank);
  return rc ? nccl_fail(rc, "ncclCommInitRank") : SKC_OK;
}

int skc_nccl_comm_destroy(void* comm) {
  Nccl& N = nccl();
  if (!N.why.empty()) return fail(SKC_ENCCL, N.why);
  if (comm == nullptr) return SKC_OK;
  const int rc = N.destroy(comm);
  return rc ? nccl_fail(rc, "ncclCommDestroy") : SKC_OK;
}

int skc_allreduce_sum_f64(double* buf, size_t count, void* comm, void* stream) {
  Nccl& N = nccl();
  if (!N.why.empty()) return fail(SKC_ENCCL, N.why);
  if (comm == nullptr) return fail(SKC_EPARAM, "comm (ncclComm_t) is NULL");
  if (count == 0) return SKC_OK;
  if (buf == nullptr) return fail(SKC_EPARAM, "buf is NULL");
  const int rc = N.allreduce(buf, buf, count, kNcclFloat64, kNcclSum, comm, static_cast<cudaStream_t>(stream));
  return rc ? nccl_fail(rc, "ncclAllReduce") : SKC_OK;
}

size_t skc_moments_packed_len(int32_t p_pad, int32_t covariance) {
  return (size_t)p_pad + 3 + (covariance ? (size_t)p_pad * (p_pad + 1) / 2 : 0);
}

size_t skc_kmeans_exchange_len(int32_t p_pad, int32_t K, int32_t world) {
  return 2 * (size_t)p_pad * K + K + 2 + 2 * (size_t)world;
}

int skc_kmeans_pack_exchange(const double* sums, const int64_t* counts, const int64_t* sizes, const int64_t* out,
                             const double* d2max, const double* objective, int32_t p_pad, int32_t K, int32_t rank,
                             int32_t world, int64_t col0, double* buf, void* stream) {
  if (p_pad < 1 || K < 1 || world < 1 || rank < 0 || rank >= world) return fail(SKC_EPARAM, "bad (p_pad, K, rank)");
  const int64_t total = (int64_t)skc_kmeans_exchange_len(p_pad, K, world);
  kmeans_pack_kernel<<<(unsigned)((total + 255) / 256 < 1024 ? (total + 255) / 256 : 1024), 256, 0,
                       static_cast<cudaStream_t>(stream)>>>(sums, counts, sizes, out, d2max, objective,
                                                           (int64_t)p_pad * K, K, rank, world, col0, buf);
  return check_launch("kmeans_pack_kernel");
}

int skc_kmeans_unpack_exchange(const double* buf, int32_t p_pad, int32_t K, double* sums, int64_t* counts,
                               int64_t* sizes, void* stream) {
  if (p_pad < 1 || K < 1) return fail(SKC_EPARAM, "bad (p_pad, K)");
  const int64_t total = 2 * (int64_t)p_pad * K + K;
  kmeans_unpack_kernel<<<(unsigned)((total + 255) / 256 < 1024 ? (total + 255) / 256 : 1024), 256, 0,
                         static_cast<cudaStream_t>(stream)>>>(buf, (int64_t)p_pad * K, K, sums, counts, sizes);
  return check_launch("kmeans_unpack_kernel");
}

}  // extern "C"
