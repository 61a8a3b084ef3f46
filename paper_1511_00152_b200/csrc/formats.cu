// SKCH1 record packing (io.py:84-136 of the reference): per sample, m u32 indices then m
// f64 values, packed back to back (12 m bytes, 4-byte aligned fields). The device sketch
// keeps int32 indices and fp64 or fp32 values in separate arrays; these kernels build and
// split the file's record stream on the GPU so a chunk crosses PCIe in one copy.
#include "common.cuh"

namespace skc {

// one thread per 32-bit output word: word w of record r is idx[r][w] for w < m, else the
// low / high half of val[r][(w - m) / 2] widened to f64
template <typename V>
__global__ void pack_records_kernel(const int32_t* __restrict__ idx, const V* __restrict__ val, int64_t n, int32_t m,
                                    uint32_t* __restrict__ out) {
  const int64_t per = 3 * (int64_t)m;
  const int64_t total = n * per;
  for (int64_t w = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; w < total; w += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = w / per;
    const int c = (int)(w - r * per);
    uint32_t x;
    if (c < m) {
      x = (uint32_t)idx[r * m + c];
    } else {
      const int t = (c - m) >> 1;
      const uint64_t b = (uint64_t)__double_as_longlong((double)val[r * m + t]);
      x = ((c - m) & 1) ? (uint32_t)(b >> 32) : (uint32_t)b;
    }
    out[w] = x;
  }
}

// inverse: one thread per (record, slot) of the m pairs
__global__ void unpack_records_kernel(const uint32_t* __restrict__ in, int64_t n, int32_t m, int32_t* __restrict__ idx,
                                      double* __restrict__ val) {
  const int64_t total = n * (int64_t)m;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = e / m;
    const int t = (int)(e - r * m);
    const uint32_t* rec = in + r * 3 * (int64_t)m;
    idx[e] = (int32_t)rec[t];
    const uint64_t b = (uint64_t)rec[m + 2 * t] | ((uint64_t)rec[m + 2 * t + 1] << 32);
    val[e] = __longlong_as_double((long long)b);
  }
}

static unsigned grid_for(int64_t work) {
  int64_t g = (work + 255) / 256;
  const int64_t cap = 8 * (int64_t)sm_count();
  if (g > cap) g = cap;
  return (unsigned)(g < 1 ? 1 : g);
}

int pack_records_launch(const int32_t* idx, const void* val, int val_f64, int64_t n, int32_t m, uint32_t* out,
                        cudaStream_t st) {
  if (n == 0) return SKC_OK;
  const unsigned g = grid_for(n * 3 * (int64_t)m);
  if (val_f64)
    pack_records_kernel<double><<<g, 256, 0, st>>>(idx, (const double*)val, n, m, out);
  else
    pack_records_kernel<float><<<g, 256, 0, st>>>(idx, (const float*)val, n, m, out);
  return check_launch("pack_records_kernel");
}

int unpack_records_launch(const uint32_t* in, int64_t n, int32_t m, int32_t* idx, double* val, cudaStream_t st) {
  if (n == 0) return SKC_OK;
  unpack_records_kernel<<<grid_for(n * (int64_t)m), 256, 0, st>>>(in, n, m, idx, val);
  return check_launch("unpack_records_kernel");
}

}  // namespace skc
