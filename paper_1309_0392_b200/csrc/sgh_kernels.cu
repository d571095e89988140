// sgh_kernels.cu -- the per-axis hierarchization kernels of libsgh (sm_100a).
//
// Method (Alg. 1): along one axis, every pole point i on level
// lam = l - tz(i) receives   x_i <- (x_i - 0.5 x_{i-s}) - 0.5 x_{i+s},  s = 2^{tz(i)},
// skipping a predecessor that lies on the zero boundary.  Because
// Alg. 1 walks the levels finest-first and every predecessor is strictly
// coarser, the in-place sweep equals this one-pass stencil evaluated on the
// values ENTERING the sweep (checked bitwise in tests), so a tile
// may compute all its points from a staged copy in any order.
// Dehierarchization is the inverse recursion, levels 2..l (coarse to
// fine), x_i <- (x_i + 0.5 x_{i-s}) + 0.5 x_{i+s} with already-nodal
// predecessors: a level-synchronous sweep in shared memory / registers.
//
// Kernel kinds (sgh_common.cuh):
//   FLAT_SLABS / FLAT_BLOCKS  views whose slab o is contiguous (PS == S, OS == n S) and S < 64:
//                             the tile is one contiguous range of global memory.
//   STRIDED                   32 adjacent columns x (2^t + 1) pole rows, warps read rows coalesced.
//   REG<L>                    one thread per column holding the whole pole (n <= 31) in registers.
// All kernels are persistent: a CTA walks tiles q = blockIdx.x, +gridDim.x, ...
// over a task table (batched) or a single task (one grid).
#include <cuda_runtime.h>

#include <cstdint>

#include "sgh_common.cuh"
#include "sgh_plan.hpp"

namespace sgh {

struct Src {
  const Task *tasks;      // device task table, or nullptr -> use `single`
  const int64_t *prefix;  // device exclusive prefix of task tiles, ntasks+1 entries
  int32_t ntasks;
  int64_t total_tiles;
  Task single;
};

// Task index owning tile q.  `idx` is the cursor from the previous tile of this
// CTA (tiles only increase), so the scan is amortised O(1).
__device__ __forceinline__ int advance_task(const Src &src, int idx, int64_t q) {
  while (idx + 1 < src.ntasks && __ldg(&src.prefix[idx + 1]) <= q) ++idx;
  return idx;
}

__device__ __forceinline__ int first_task(const Src &src, int64_t q) {
  int lo = 0, hi = src.ntasks - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (__ldg(&src.prefix[mid]) <= q) lo = mid; else hi = mid - 1;
  }
  return lo;
}

// Walk this CTA's tiles; body(task, local tile index).
template <class F>
__device__ __forceinline__ void for_each_tile(const Src &src, F &&body) {
  if (src.tasks == nullptr) {
    for (int64_t q = blockIdx.x; q < src.total_tiles; q += gridDim.x) body(src.single, q);
    return;
  }
  int idx = -1;
  for (int64_t q = blockIdx.x; q < src.total_tiles; q += gridDim.x) {
    idx = (idx < 0) ? first_task(src, q) : advance_task(src, idx, q);
    const Task &t = src.tasks[idx];
    body(t, q - __ldg(&src.prefix[idx]));
  }
}

// ----------------------------------------------------------------- FLAT_SLABS
// Tile = R consecutive slabs (o0 .. o0+R-1), each n*S contiguous doubles.
template <bool INV>
__global__ void __launch_bounds__(kThreads) k_flat_slabs(const __grid_constant__ Src src) {
  extern __shared__ double sm[];  // R*n*S doubles (<= kFlatT)
  for_each_tile(src, [&](const Task &T, int64_t q) {
    const int l = T.l;
    const int n = (1 << l) - 1;
    const int S = (int)T.S;
    const int nS = n * S;
    const int64_t o0 = q * T.R;
    const int ns = (int)min((int64_t)T.R, T.O - o0);
    const int len = ns * nS;
    const FDiv fS = T.fS, fNS = T.fNS;
    double *__restrict__ g = T.grid + T.base + o0 * T.OS;
#pragma unroll 4
    for (int e = threadIdx.x; e < len; e += kThreads) sm[e] = g[e];
    __syncthreads();
    if (!INV) {
      for (int e = threadIdx.x; e < len; e += kThreads) {
        const uint32_t slab = fdiv((uint32_t)e, fNS);
        const uint32_t p = (uint32_t)e - slab * (uint32_t)nS;
        const int i = (int)fdiv(p, fS) + 1;           // 1-based pole index
        const int s = i & -i;                          // 2^{tz(i)}
        const int sS = s * S;
        double x = sm[e];
        if (i - s >= 1) x = x - 0.5 * sm[e - sS];      // left predecessor
        if (i + s <= n) x = x - 0.5 * sm[e + sS];      // right predecessor
        g[e] = x;
      }
    } else {
      for (int lam = 2; lam <= l; ++lam) {             // coarse -> fine (reading R9)
        const int s = 1 << (l - lam);
        const int rows = 1 << (lam - 1);
        const int cnt = ns * rows * S;
        const int sS = s * S;
        for (int k = threadIdx.x; k < cnt; k += kThreads) {
          const uint32_t qq = fdiv((uint32_t)k, fS);
          const int r = k - (int)qq * S;
          const int slab = (int)(qq >> (lam - 1));
          const int j = (int)qq & (rows - 1);
          const int i = s * (2 * j + 1);
          const int e = slab * nS + (i - 1) * S + r;
          double x = sm[e];
          if (i - s >= 1) x = x + 0.5 * sm[e - sS];
          if (i + s <= n) x = x + 0.5 * sm[e + sS];
          sm[e] = x;
        }
        __syncthreads();
      }
#pragma unroll 4
      for (int e = threadIdx.x; e < len; e += kThreads) g[e] = sm[e];
    }
    __syncthreads();
  });
}

// ---------------------------------------------------------------- FLAT_BLOCKS
// Tile = rows [b 2^t, (b+1) 2^t] (local rb = 0..2^t) of slab o; rows are S
// contiguous doubles and consecutive rows are adjacent (PS == S).  Only the
// fine rows rb = 1..2^t-1 are written; rb = 0 and rb = 2^t are coarse-lattice
// points owned by another phase (read-only halo here).
template <bool INV>
__global__ void __launch_bounds__(kThreads) k_flat_blocks(const __grid_constant__ Src src) {
  extern __shared__ double sm[];  // (2^t + 1) * S doubles
  for_each_tile(src, [&](const Task &T, int64_t q) {
    const int t = T.t;
    const int B = 1 << t;
    const int nb_log = T.l - t;
    const int64_t o = q >> nb_log;
    const int b = (int)(q & ((1 << nb_log) - 1));
    const int S = (int)T.S;
    const int n = (1 << T.l) - 1;
    const int i0 = b * B;                                  // pole index of local row 0
    const int rb_lo = (b == 0) ? 1 : 0;                    // row 0 of block 0 is the boundary
    const int rb_hi = (b == (1 << nb_log) - 1) ? B - 1 : B;  // row 2^l is the boundary
    const FDiv fS = T.fS;
    // global offset of local element e = rb*S + r is  row0 + e
    const int64_t row0 = T.base + o * T.OS + (int64_t)(i0 - 1) * S;
    double *__restrict__ g = T.grid;
    {
      const int e0 = rb_lo * S, e1 = (rb_hi + 1) * S;
#pragma unroll 4
      for (int e = e0 + threadIdx.x; e < e1; e += kThreads) sm[e] = g[row0 + e];
    }
    __syncthreads();
    if (!INV) {
      const int e1 = B * S;
      for (int e = S + threadIdx.x; e < e1; e += kThreads) {
        const int rb = (int)fdiv((uint32_t)e, fS);
        const int i = i0 + rb;
        const int s = rb & -rb;                            // tz(i) = tz(rb) < t
        const int sS = s * S;
        double x = sm[e];
        if (i - s >= 1) x = x - 0.5 * sm[e - sS];
        if (i + s <= n) x = x - 0.5 * sm[e + sS];
        g[row0 + e] = x;
      }
    } else {
      for (int s = B >> 1; s >= 1; s >>= 1) {              // block-local levels, coarse -> fine
        const int cnt = (B / (2 * s)) * S;
        const int sS = s * S;
        for (int k = threadIdx.x; k < cnt; k += kThreads) {
          const int jj = (int)fdiv((uint32_t)k, fS);
          const int r = k - jj * S;
          const int rb = s * (2 * jj + 1);
          const int e = rb * S + r;
          const int i = i0 + rb;
          double x = sm[e];
          if (i - s >= 1) x = x + 0.5 * sm[e - sS];
          if (i + s <= n) x = x + 0.5 * sm[e + sS];
          sm[e] = x;
        }
        __syncthreads();
      }
      const int e1 = B * S;
#pragma unroll 4
      for (int e = S + threadIdx.x; e < e1; e += kThreads) g[row0 + e] = sm[e];
    }
    __syncthreads();
  });
}

// ------------------------------------------------------------------- STRIDED
// Tile = (o, block b, column group cb): rows rb = 0..2^t (pole index b 2^t + rb),
// columns c0 .. c0+31.  Warp w moves rows w, w+8, ...; lane = column, so every
// row segment is one coalesced 256-byte access.  t == l means the whole pole.
template <bool INV>
__global__ void __launch_bounds__(kThreads) k_strided(const __grid_constant__ Src src) {
  extern __shared__ double sm_raw[];  // (2^t + 1) rows of kStridedW doubles
  auto sm = reinterpret_cast<double (*)[kStridedW]>(sm_raw);
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  constexpr int kWarps = kThreads / 32;
  for_each_tile(src, [&](const Task &T, int64_t q) {
    const int t = T.t;
    const int B = 1 << t;
    const int nb_log = T.l - t;
    const int64_t cb = q % T.ncb;
    const int64_t rest = q / T.ncb;
    const int b = (int)(rest & ((1 << nb_log) - 1));
    const int64_t o = rest >> nb_log;
    const int64_t c0 = cb * kStridedW;
    const bool active = (c0 + lane) < T.S;
    const int n = (1 << T.l) - 1;
    const int i0 = b * B;
    const int rb_lo = (i0 == 0) ? 1 : 0;
    const int rb_hi = min(B, n - i0);
    const int64_t PS = T.PS;
    double *__restrict__ g = T.grid + T.base + o * T.OS + c0 + lane - PS;  // + i*PS -> element (o,i,c0+lane)
#pragma unroll 4
    for (int rb = rb_lo + warp; rb <= rb_hi; rb += kWarps)
      if (active) sm[rb][lane] = g[(int64_t)(i0 + rb) * PS];
    __syncthreads();
    const int rhi = (t == T.l) ? n : B - 1;
    if (!INV) {
      for (int rb = 1 + warp; rb <= rhi; rb += kWarps) {
        const int i = i0 + rb;
        const int s = rb & -rb;
        double x = sm[rb][lane];
        if (i - s >= 1) x = x - 0.5 * sm[rb - s][lane];
        if (i + s <= n) x = x - 0.5 * sm[rb + s][lane];
        if (active) g[(int64_t)i * PS] = x;
      }
    } else {
      const int s_top = (t == T.l) ? (B >> 2) : (B >> 1);
      for (int s = s_top; s >= 1; s >>= 1) {
        const int cnt = B / (2 * s);
        for (int j = warp; j < cnt; j += kWarps) {
          const int rb = s * (2 * j + 1);
          const int i = i0 + rb;
          double x = sm[rb][lane];
          if (i - s >= 1) x = x + 0.5 * sm[rb - s][lane];
          if (i + s <= n) x = x + 0.5 * sm[rb + s][lane];
          sm[rb][lane] = x;
        }
        __syncthreads();
      }
#pragma unroll 4
      for (int rb = 1 + warp; rb <= rhi; rb += kWarps)
        if (active) g[(int64_t)(i0 + rb) * PS] = sm[rb][lane];
    }
    __syncthreads();
  });
}

// ----------------------------------------------------------------------- REG
// One thread per column (o, r); the whole pole of n = 2^L - 1 points lives in
// registers; the level structure is resolved at compile time.
template <int L, bool INV>
__global__ void __launch_bounds__(kThreads) k_reg(const __grid_constant__ Src src) {
  constexpr int n = (1 << L) - 1;
  for_each_tile(src, [&](const Task &T, int64_t q) {
    const int64_t gcol = q * kThreads + threadIdx.x;
    if (gcol >= T.O * T.S) return;
    const int64_t o = gcol / T.S;
    const int64_t r = gcol - o * T.S;
    double *__restrict__ p = T.grid + T.base + o * T.OS + r;
    const int64_t PS = T.PS;
    double v[n];
#pragma unroll
    for (int i = 0; i < n; ++i) v[i] = p[i * PS];
    if (!INV) {
      // v keeps the values entering the sweep; results go straight to memory
#pragma unroll
      for (int i = 1; i <= n; ++i) {
        const int s = i & -i;
        double x = v[i - 1];
        if (i - s >= 1) x = x - 0.5 * v[i - s - 1];
        if (i + s <= n) x = x - 0.5 * v[i + s - 1];
        p[(i - 1) * PS] = x;
      }
    } else {
#pragma unroll
      for (int lam = 2; lam <= L; ++lam) {
        const int s = 1 << (L - lam);
#pragma unroll
        for (int i = s; i <= n; i += 2 * s) {
          double x = v[i - 1];
          if (i - s >= 1) x = x + 0.5 * v[i - s - 1];
          if (i + s <= n) x = x + 0.5 * v[i + s - 1];
          v[i - 1] = x;
        }
      }
#pragma unroll
      for (int i = 0; i < n; ++i) p[i * PS] = v[i];
    }
  });
}

// ------------------------------------------------------------ host launchers
using KernelFn = void (*)(Src);

static KernelFn kernel_for(int kind, int l, bool inv) {
  switch (kind) {
    case KIND_FLAT_SLABS: return inv ? k_flat_slabs<true> : k_flat_slabs<false>;
    case KIND_FLAT_BLOCKS: return inv ? k_flat_blocks<true> : k_flat_blocks<false>;
    case KIND_STRIDED: return inv ? k_strided<true> : k_strided<false>;
    case KIND_REG:
      switch (l) {
        case 2: return inv ? k_reg<2, true> : k_reg<2, false>;
        case 3: return inv ? k_reg<3, true> : k_reg<3, false>;
        case 4: return inv ? k_reg<4, true> : k_reg<4, false>;
        case 5: return inv ? k_reg<5, true> : k_reg<5, false>;
        default: return nullptr;
      }
    default: return nullptr;
  }
}

// dynamic shared memory a task needs
size_t task_smem(const Task &t) {
  const int64_t n = (int64_t(1) << t.l) - 1;
  switch (t.kind) {
    case KIND_FLAT_SLABS: return size_t(t.R) * size_t(n * t.S) * 8;
    case KIND_FLAT_BLOCKS: return size_t((int64_t(1) << t.t) + 1) * size_t(t.S) * 8;
    case KIND_STRIDED: return size_t((int64_t(1) << t.t) + 1) * kStridedW * 8;
    default: return 0;
  }
}

// resident CTAs on the whole device for a kernel instance and smem size (cached)
static int resident_ctas(KernelFn fn, size_t smem) {
  int dev = 0;
  cudaGetDevice(&dev);
  struct Entry { KernelFn fn; int dev; size_t smem; int ctas; };
  static Entry cache[256];
  static int ncache = 0;
  for (int i = 0; i < ncache; ++i)
    if (cache[i].fn == fn && cache[i].dev == dev && cache[i].smem == smem) return cache[i].ctas;
  int ctas = 1;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&ctas, fn, kThreads, smem) != cudaSuccess || ctas < 1) ctas = 1;
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int total = ctas * sms;
  if (ncache < 256) cache[ncache++] = Entry{fn, dev, smem, total};
  return total;
}

// Launch one task (single grid).  Returns the CUDA error of the launch.
cudaError_t launch_single(const Task &task, bool inv, cudaStream_t stream) {
  KernelFn fn = kernel_for(task.kind, task.l, inv);
  if (!fn) return cudaErrorInvalidValue;
  Src src{};
  src.tasks = nullptr;
  src.prefix = nullptr;
  src.ntasks = 1;
  src.total_tiles = task.tiles;
  src.single = task;
  const size_t smem = task_smem(task);
  const int64_t cap = resident_ctas(fn, smem);
  const int64_t grid = task.tiles < cap ? task.tiles : cap;
  if (grid <= 0) return cudaSuccess;
  ProfToken tok = prof_begin(stream);
  fn<<<(unsigned)grid, kThreads, smem, stream>>>(src);
  cudaError_t e = cudaGetLastError();
  prof_end(tok, task.kind, task.l, inv, 16.0 * task_points(task), stream);
  return e;
}

// Launch a group of tasks of one kernel instance from a device task table;
// smem = max task_smem over the group.
cudaError_t launch_table(int kind, int l, bool inv, const Task *d_tasks, const int64_t *d_prefix,
                         int32_t ntasks, int64_t total_tiles, size_t smem, double points, cudaStream_t stream) {
  KernelFn fn = kernel_for(kind, l, inv);
  if (!fn) return cudaErrorInvalidValue;
  Src src{};
  src.tasks = d_tasks;
  src.prefix = d_prefix;
  src.ntasks = ntasks;
  src.total_tiles = total_tiles;
  const int64_t cap = resident_ctas(fn, smem);
  const int64_t grid = total_tiles < cap ? total_tiles : cap;
  if (grid <= 0) return cudaSuccess;
  ProfToken tok = prof_begin(stream);
  fn<<<(unsigned)grid, kThreads, smem, stream>>>(src);
  cudaError_t e = cudaGetLastError();
  prof_end(tok, kind, l, inv, 16.0 * points, stream);
  return e;
}

}  // namespace sgh
