// sgh_util.cu -- harness utilities of libsgh: seeded fill and order-independent
// digest.  Not part of the method; used to create
// synthetic inputs on the device (the C5 set is 41 GB) and to compare results
// without copying them back.  Written independently of oracle/.
#include <cuda_runtime.h>

#include <cstdint>

#include "sgh_common.cuh"

namespace sgh {

__device__ __forceinline__ uint64_t splitmix_finalise(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

uint64_t host_splitmix_finalise(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}


constexpr int kUtilThreads = 256;
constexpr int kUtilPerCta = kUtilThreads * 16;  // elements per CTA chunk

__device__ __forceinline__ int find_item(const int64_t *prefix, int n, int64_t q) {
  int lo = 0, hi = n - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (prefix[mid] <= q) lo = mid; else hi = mid - 1;
  }
  return lo;
}

__global__ void __launch_bounds__(kUtilThreads) k_fill(const FillItem *items, const int64_t *prefix, int nitems,
                                                        const FillItem single) {
  const int it = items ? find_item(prefix, nitems, blockIdx.x) : 0;
  const FillItem f = items ? items[it] : single;
  const int64_t c0 = (int64_t)(blockIdx.x - (items ? prefix[it] : 0)) * kUtilPerCta;
  const int64_t c1 = min(f.n, c0 + kUtilPerCta);
  for (int64_t k = c0 + threadIdx.x; k < c1; k += kUtilThreads) {
    const uint64_t i = (uint64_t)(f.index_offset + k);
    const double u = (double)(splitmix_finalise(f.key + i) >> 11) * 0x1.0p-53;
    f.ptr[k] = 2.0 * u - 1.0;
  }
}

__global__ void __launch_bounds__(kUtilThreads) k_digest(const FillItem *items, const int64_t *prefix, int nitems,
                                                          const FillItem single, unsigned long long *out) {
  const int it = items ? find_item(prefix, nitems, blockIdx.x) : 0;
  const FillItem f = items ? items[it] : single;
  const int64_t c0 = (int64_t)(blockIdx.x - (items ? prefix[it] : 0)) * kUtilPerCta;
  const int64_t c1 = min(f.n, c0 + kUtilPerCta);
  uint64_t h = 0;
  for (int64_t k = c0 + threadIdx.x; k < c1; k += kUtilThreads) {
    const uint64_t bits = (uint64_t)__double_as_longlong(f.ptr[k]);
    const uint64_t i = (uint64_t)(f.index_offset + k);
    h += splitmix_finalise(bits ^ (i * 0x9E3779B97F4A7C15ull));
  }
  for (int off = 16; off > 0; off >>= 1) h += __shfl_xor_sync(0xffffffffu, h, off);
  __shared__ uint64_t red[kUtilThreads / 32];
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = h;
  __syncthreads();
  if (threadIdx.x == 0) {
    uint64_t s = 0;
    for (int w = 0; w < kUtilThreads / 32; ++w) s += red[w];
    atomicAdd(&out[it], (unsigned long long)s);  // wrap-around sum: order independent
  }
}

// chunk count of an item
int64_t util_chunks(int64_t n) { return (n + kUtilPerCta - 1) / kUtilPerCta; }

cudaError_t launch_fill(const FillItem *d_items, const int64_t *d_prefix, int nitems, const FillItem &single,
                        int64_t total_chunks, cudaStream_t st) {
  if (total_chunks <= 0) return cudaSuccess;
  k_fill<<<(unsigned)total_chunks, kUtilThreads, 0, st>>>(d_items, d_prefix, nitems, single);
  return cudaGetLastError();
}

cudaError_t launch_digest(const FillItem *d_items, const int64_t *d_prefix, int nitems, const FillItem &single,
                          int64_t total_chunks, unsigned long long *d_out, cudaStream_t st) {
  if (total_chunks <= 0) return cudaSuccess;
  k_digest<<<(unsigned)total_chunks, kUtilThreads, 0, st>>>(d_items, d_prefix, nitems, single, d_out);
  return cudaGetLastError();
}

}  // namespace sgh
