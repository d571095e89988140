// sgh_ablation.cu -- SURVEY 8(f) 4 ablation: the paper's BFS data layout
// ("BFS layouts": the points of a 1-D pole ordered by a breadth-
// first traversal of the binary hierarchy, Fig. fig:hierDehier -- root first,
// then level 2 left to right, ..., the finest level last) on B200.
// Report only; the product path keeps the row-major layout.
//
// Position p (0-based) of a level-l pole in BFS order holds hierarchical level
// lam = floor(log2(p + 1)) + 1, index j = p + 1 - 2^{lam-1} on that level, i.e.
// the natural 1-based point i = (2 j + 1) 2^{l - lam}.  Its predecessors
// i -+ 2^{l - lam} sit at the BFS positions of the natural indices
// 2 j 2^{l-lam} and (2 j + 2) 2^{l-lam} (absent on the boundary 0 / 2^l).
//
// Hierarchization is the one-pass stencil of the values entering the pass
// (SURVEY 8(a)), done out of place: out[p] = (in[p] - 0.5 in[pL]) - 0.5 in[pR],
// every point independent (one kernel).  Dehierarchization is the recursion
// coarse -> fine, in place, one launch per level (a level reads only coarser,
// already nodal levels).  Both with the oracle's rounding (two IEEE
// operations per term), so the results are bitwise those of Alg. 1.
#include <cuda_runtime.h>

#include <cstdint>

#include "../../include/sgh.h"
#include "sgh_common.cuh"
#include "sgh_plan.hpp"

namespace sgh {

// BFS position of natural 1-based index x (1 <= x < 2^l) of a level-l pole
__device__ __forceinline__ int64_t bfs_pos(int64_t x, int l) {
  const int t = __ffsll((long long)x) - 1;        // tz(x)
  const int lam = l - t;
  const int64_t j = ((x >> t) - 1) >> 1;
  return (int64_t(1) << (lam - 1)) - 1 + j;
}

// natural 1-based index of BFS position p
__device__ __forceinline__ int64_t bfs_nat(int64_t p, int l) {
  const int lam = 64 - __clzll((long long)(p + 1));    // floor(log2(p + 1)) + 1
  const int64_t j = p + 1 - (int64_t(1) << (lam - 1));
  return (2 * j + 1) << (l - lam);
}

__global__ void k_bfs_permute(const double *__restrict__ src, double *__restrict__ dst, int l, int to_bfs) {
  const int64_t n = (int64_t(1) << l) - 1;
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < n; p += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = bfs_nat(p, l);              // natural point at BFS position p
    if (to_bfs) dst[p] = src[i - 1];
    else dst[i - 1] = src[p];
  }
}

__global__ void k_bfs_hier(const double *__restrict__ in, double *__restrict__ out, int l) {
  const int64_t n = (int64_t(1) << l) - 1;
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < n; p += (int64_t)gridDim.x * blockDim.x) {
    const int lam = 64 - __clzll((long long)(p + 1));
    const int64_t j = p + 1 - (int64_t(1) << (lam - 1));
    const int64_t s = int64_t(1) << (l - lam);
    const int64_t i = (2 * j + 1) * s;
    double x = in[p];
    if (i - s >= 1) x = __dsub_rn(x, __dmul_rn(0.5, __ldg(&in[bfs_pos(i - s, l)])));
    if (i + s <= n) x = __dsub_rn(x, __dmul_rn(0.5, __ldg(&in[bfs_pos(i + s, l)])));
    out[p] = x;
  }
}

// one level lam (its 2^{lam-1} points are contiguous at 2^{lam-1} - 1 ...)
__global__ void k_bfs_dehier_level(double *__restrict__ g, int l, int lam) {
  const int64_t n = (int64_t(1) << l) - 1;
  const int64_t cnt = int64_t(1) << (lam - 1);
  const int64_t s = int64_t(1) << (l - lam);
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < cnt; j += (int64_t)gridDim.x * blockDim.x) {
    const int64_t p = cnt - 1 + j;
    const int64_t i = (2 * j + 1) * s;
    double x = g[p];
    if (i - s >= 1) x = __dadd_rn(x, __dmul_rn(0.5, g[bfs_pos(i - s, l)]));
    if (i + s <= n) x = __dadd_rn(x, __dmul_rn(0.5, g[bfs_pos(i + s, l)]));
    g[p] = x;
  }
}

static unsigned grid_for(int64_t n) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t want = (n + 255) / 256;
  const int64_t cap = int64_t(sms) * 8;
  return (unsigned)(want < cap ? (want > 0 ? want : 1) : cap);
}

}  // namespace sgh

using namespace sgh;

extern "C" {

sgh_status sgh_ablation_bfs_permute_1d(const double *src, double *dst, int32_t l, int32_t to_bfs, void *stream) {
  if (!src || !dst || src == dst) return invalid("src / dst NULL or aliased");
  if (l < 1 || l > SGH_MAX_LEVEL) return invalid("level out of range");
  const int64_t n = (int64_t(1) << l) - 1;
  k_bfs_permute<<<grid_for(n), 256, 0, static_cast<cudaStream_t>(stream)>>>(src, dst, l, to_bfs ? 1 : 0);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(e, "k_bfs_permute");
  count_launch();
  return SGH_OK;
}

sgh_status sgh_ablation_bfs_hierarchize_1d(const double *in, double *out, int32_t l, void *stream) {
  if (!in || !out || in == out) return invalid("in / out NULL or aliased (the BFS hierarchization is out of place)");
  if (l < 1 || l > SGH_MAX_LEVEL) return invalid("level out of range");
  const int64_t n = (int64_t(1) << l) - 1;
  k_bfs_hier<<<grid_for(n), 256, 0, static_cast<cudaStream_t>(stream)>>>(in, out, l);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(e, "k_bfs_hier");
  count_launch();
  return SGH_OK;
}

sgh_status sgh_ablation_bfs_dehierarchize_1d(double *grid, int32_t l, void *stream) {
  if (!grid) return invalid("grid is NULL");
  if (l < 1 || l > SGH_MAX_LEVEL) return invalid("level out of range");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  for (int lam = 2; lam <= l; ++lam) {            // coarse -> fine (reading R9)
    k_bfs_dehier_level<<<grid_for(int64_t(1) << (lam - 1)), 256, 0, s>>>(grid, l, lam);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_fail(e, "k_bfs_dehier_level");
    count_launch();
  }
  return SGH_OK;
}

}  // extern "C"
