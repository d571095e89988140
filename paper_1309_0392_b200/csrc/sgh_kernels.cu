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
//   REG<L>                    one thread per column holding the whole pole (n <= 15) in registers.
// All kernels are persistent: a CTA walks tiles q = blockIdx.x, +gridDim.x, ...
// over a task table (batched) or a single task (one grid).
//
// Memory-level parallelism: a tile is staged with cp.async (LDGSTS) -- every
// thread issues all of its copies back to back, so the whole tile (up to 33 KB
// per CTA, ~200 KB per SM) is in flight at once -- 16-byte copies on the
// aligned body of contiguous ranges, 8-byte copies otherwise (rows of odd
// length are only 8-byte aligned: SURVEY H1).
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>

#include "sgh_common.cuh"
#include "sgh_plan.hpp"

namespace sgh {

struct Src {
  const Task *tasks;      // device task table, or nullptr -> use `single`
  const int64_t *prefix;  // device exclusive prefix of task tiles, ntasks+1 entries
  int32_t ntasks;
  int32_t stage_doubles;  // FUSED: SMEM doubles per pipeline stage (2 stages)
  int64_t total_tiles;
  Task single;
};

// ------------------------------------------------------------- async copies
__device__ __forceinline__ void cp_async8(double *sdst, const double *gsrc) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(sdst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void cp_async16(double *sdst, const double *gsrc) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(sdst);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;\n" ::: "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory"); }

// 8-byte phase of a global address (0: 16-byte aligned, 1: 8 mod 16)
__device__ __forceinline__ int phase8(const double *p) { return (int)((reinterpret_cast<uintptr_t>(p) >> 3) & 1); }

// Copy len doubles gsrc[0..len) -> sdst[0..len) where sdst and gsrc have the
// same 16-byte phase: 8-byte head/tail, 16-byte body.  Issue only.
__device__ __forceinline__ void copy_range_async(double *sdst, const double *gsrc, int len) {
  if (len <= 0) return;
  const int head = phase8(gsrc) ? 1 : 0;
  const int pairs = (len - head) >> 1;
  const int tail = len - head - 2 * pairs;
  if (head && threadIdx.x == 0) cp_async8(sdst, gsrc);
  if (tail && threadIdx.x == kThreads - 1) cp_async8(sdst + len - 1, gsrc + len - 1);
  const double *g = gsrc + head;
  double *s = sdst + head;
#pragma unroll 4
  for (int p = threadIdx.x; p < pairs; p += kThreads) cp_async16(s + 2 * p, g + 2 * p);
}

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
  // The current task descriptor lives in SMEM: tile setup then reads its
  // fields with LDS instead of dependent global loads (measured: ~12 % of the
  // stall samples of STRIDED in the C5 step).  Reloaded only when the CTA
  // crosses into the next task (tiles of a CTA only increase).
  __shared__ Task s_task;
  __shared__ int64_t s_first;
  int idx = -1, cur = -1;
  for (int64_t q = blockIdx.x; q < src.total_tiles; q += gridDim.x) {
    idx = (idx < 0) ? first_task(src, q) : advance_task(src, idx, q);
    if (idx != cur) {
      __syncthreads();                           // everyone is done with the previous descriptor
      const uint64_t *a = reinterpret_cast<const uint64_t *>(&src.tasks[idx]);
      uint64_t *b = reinterpret_cast<uint64_t *>(&s_task);
      for (int i = threadIdx.x; i < (int)(sizeof(Task) / 8); i += kThreads) b[i] = a[i];
      if (threadIdx.x == 0) s_first = src.prefix[idx];
      __syncthreads();
      cur = idx;
    }
    body(s_task, q - s_first);
  }
}

// ----------------------------------------------------------------- FLAT_SLABS
// Tile = R consecutive slabs (o0 .. o0+R-1), each n*S contiguous doubles.
template <bool INV>
__global__ void __launch_bounds__(kThreads) k_flat_slabs(const __grid_constant__ Src src) {
  extern __shared__ __align__(16) double smem[];  // 1 + R*n*S doubles (<= kFlatT + 1)
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
    double *sm = smem + phase8(g);                      // same 16-byte phase as g
    copy_range_async(sm, g, len);
    cp_async_wait_all();
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
  extern __shared__ __align__(16) double smem[];  // 1 + (2^t + 1) * S doubles
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
    // global element of local e = rb*S + r is  gr[e]
    double *__restrict__ gr = T.grid + T.base + o * T.OS + (int64_t)(i0 - 1) * S;
    double *sm = smem + phase8(gr);
    copy_range_async(sm + rb_lo * S, gr + rb_lo * S, (rb_hi - rb_lo + 1) * S);
    cp_async_wait_all();
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
        gr[e] = x;
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
      for (int e = S + threadIdx.x; e < e1; e += kThreads) gr[e] = sm[e];
    }
    __syncthreads();
  });
}

// ------------------------------------------------------------------- STRIDED
// Tile = (o, block b, column group cb): rows rb = 0..2^t (pole index b 2^t + rb),
// W adjacent columns c0 .. c0+W-1 (W = 32/64/128, T.W).  t == l: whole pole.
// SMEM rows have stride W + 2 doubles (16-byte aligned) and element c of row
// rb sits at rb*(W+2) + c + par(rb), par = the 8-byte phase of the row's global
// start, so global 16-byte pairs land on 16-byte aligned SMEM and are copied
// with 16-byte cp.async.cg (no L1 allocation); the odd head / tail element of a
// row uses an 8-byte copy.
template <int W>
__device__ __forceinline__ void strided_load_rows(double *sm, const double *rowbase, int64_t PS, int par0,
                                                  int i0, int rb_lo, int rb_hi, int wc) {
  constexpr int RS = W + 2;
  constexpr int P = W / 2;          // 16-byte slots per row
  constexpr int LOGP = (P == 4) ? 2 : (P == 8) ? 3 : (P == 16) ? 4 : (P == 32) ? 5 : (P == 64) ? 6 : 7;
  const int psodd = (int)(PS & 1);
  const int nslots = (rb_hi - rb_lo + 1) * P;
#pragma unroll 4
  for (int p = threadIdx.x; p < nslots; p += kThreads) {
    const int rb = rb_lo + (p >> LOGP);
    const int k = p & (P - 1);
    const int i = i0 + rb;
    const int par = (par0 + (i - 1) * psodd) & 1;
    const double *gr = rowbase + (int64_t)(i - 1) * PS;
    double *sr = sm + rb * RS + par;
    const int npairs = (wc - par) >> 1;
    const int c = par + 2 * k;
    if (k < npairs) cp_async16(sr + c, gr + c);
    if (k == P - 1 && par) cp_async8(sr, gr);                       // head element 0
    const int last = par + 2 * npairs;                              // first element not covered
    if (k == P - 2 && last < wc) cp_async8(sr + last, gr + last);   // tail element
  }
}

template <bool INV, int W>
__global__ void __launch_bounds__(kThreads) k_strided(const __grid_constant__ Src src) {
  extern __shared__ __align__(16) double sm[];  // (2^t + 1) rows of W + 2 doubles
  constexpr int RS = W + 2;
  constexpr int CPL = W / 32;                    // columns per lane
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
    const int64_t c0 = cb * W;
    const int wc = (int)min((int64_t)W, T.S - c0);
    const int n = (1 << T.l) - 1;
    const int i0 = b * B;
    const int rb_lo = (i0 == 0) ? 1 : 0;
    const int rb_hi = min(B, n - i0);
    const int64_t PS = T.PS;
    const int psodd = (int)(PS & 1);
    double *__restrict__ rowbase = T.grid + T.base + o * T.OS + c0;  // element (o, i, c0+c) = rowbase[(i-1)PS + c]
    const int par0 = phase8(rowbase);
    strided_load_rows<W>(sm, rowbase, PS, par0, i0, rb_lo, rb_hi, wc);
    cp_async_wait_all();
    __syncthreads();
    auto row = [&](int rb) -> double * { return sm + rb * RS + ((par0 + (i0 + rb - 1) * psodd) & 1); };
    const int rhi = (t == T.l) ? n : B - 1;
    if (!INV) {
      for (int rb = 1 + warp; rb <= rhi; rb += kWarps) {
        const int i = i0 + rb;
        const int s = rb & -rb;
        const double *xm = row(rb), *xl = row(rb - s), *xr = row(rb + s);
        double *gout = rowbase + (int64_t)(i - 1) * PS;
#pragma unroll
        for (int u = 0; u < CPL; ++u) {
          const int c = lane + 32 * u;
          if (c < wc) {
            double x = xm[c];
            if (i - s >= 1) x = x - 0.5 * xl[c];
            if (i + s <= n) x = x - 0.5 * xr[c];
            gout[c] = x;
          }
        }
      }
    } else {
      const int s_top = (t == T.l) ? (B >> 2) : (B >> 1);
      for (int s = s_top; s >= 1; s >>= 1) {
        const int cnt = B / (2 * s);
        for (int j = warp; j < cnt; j += kWarps) {
          const int rb = s * (2 * j + 1);
          const int i = i0 + rb;
          double *xm = row(rb);
          const double *xl = row(rb - s), *xr = row(rb + s);
#pragma unroll
          for (int u = 0; u < CPL; ++u) {
            const int c = lane + 32 * u;
            double x = xm[c];
            if (i - s >= 1) x = x + 0.5 * xl[c];
            if (i + s <= n) x = x + 0.5 * xr[c];
            xm[c] = x;
          }
        }
        __syncthreads();
      }
      for (int rb = 1 + warp; rb <= rhi; rb += kWarps) {
        const double *xm = row(rb);
        double *gout = rowbase + (int64_t)(i0 + rb - 1) * PS;
#pragma unroll
        for (int u = 0; u < CPL; ++u) {
          const int c = lane + 32 * u;
          if (c < wc) gout[c] = xm[c];
        }
      }
    }
    __syncthreads();
  });
}

// ---------------------------------------------------------------------- FUSED
// Several consecutive axes a..a+m-1 in ONE round trip: the
// tile holds whole poles of every axis of the group, so Alg. 1
// runs axis by axis, level by level, in place in SMEM -- exactly the oracle's
// per-point operation order (axes ascending, levels finest first, left then
// right), hence bitwise parity.  Dehierarchization: axes ascending, levels
// coarse to fine (reading R9).
//   W == 1: the group starts at a unit-stride axis; the tile is R units of P
//           contiguous doubles (one contiguous global range).
//   W  > 1: the tile is P rows of W adjacent columns (row stride S, always odd:
//           a product of odd n_k).  SMEM rows have the ODD stride W+1 and start
//           at the global 8-byte phase, so every row's 16-byte global pairs land
//           16-byte aligned and element (row, c) sits at sm[row*(W+1) + c]: a
//           pole has one uniform SMEM stride.
// Per axis, when the tile holds enough poles, each thread owns whole poles and
// runs the levels serially in SMEM (no division per point, no barrier inside
// the axis); otherwise all threads sweep one level at a time (barrier per level).
__device__ __forceinline__ FDiv device_fdiv(uint32_t d) {
  FDiv f;
  f.d = d;
  uint32_t s = 0;
  while (s < 32 && (1ull << s) < d) ++s;
  f.s = s;
  f.m = (uint32_t)((((1ull << 32) * ((1ull << s) - d)) / d) + 1);
  return f;
}

// rows 0..P-1 of W columns (wc valid), global row r at g + r*S (S odd), SMEM row r at sb + r*(W+1).
// Lane = (sub-row, 16-byte slot): one warp instruction covers 32/(W/2) rows.
template <int W>
__device__ __forceinline__ void fused_load_rows_wide(double *sb, const double *g, int64_t S, int par0, int P, int wc) {
  constexpr int RS = W + 1;
  constexpr int NP = W / 2;                       // 16-byte slots per row (32 or 64)
  constexpr int LOGP = (NP == 32) ? 5 : 6;
  const int nslots = P * NP;
#pragma unroll 4
  for (int p = threadIdx.x; p < nslots; p += kThreads) {
    const int r = p >> LOGP;
    const int k = p & (NP - 1);
    const int par = (par0 + r) & 1;
    const double *gr = g + (int64_t)r * S;
    double *sr = sb + r * RS;
    const int npairs = (wc - par) >> 1;
    const int c = par + 2 * k;
    if (k < npairs) cp_async16(sr + c, gr + c);
    if (k == NP - 1 && par) cp_async8(sr, gr);
    const int last = par + 2 * npairs;
    if (k == NP - 2 && last < wc) cp_async8(sr + last, gr + last);
  }
}

template <int W>
__device__ __forceinline__ void fused_load_rows(double *sb, const double *g, int64_t S, int par0, int P, int wc) {
  constexpr int RS = W + 1;
  constexpr int NP = W / 2;                       // 16-byte slots per row
  constexpr int RPI = 32 / NP;                    // rows per warp instruction
  constexpr int STEP = RPI * (kThreads / 32);     // rows per CTA iteration
  const int lane = threadIdx.x & 31;
  const int k = lane % NP;
  int r = (threadIdx.x >> 5) * RPI + lane / NP;
  const double *gr = g + (int64_t)r * S;
  double *sr = sb + r * RS;
  const int64_t gstep = (int64_t)STEP * S;
#pragma unroll 4
  for (; r < P; r += STEP, gr += gstep, sr += STEP * RS) {
    const int par = (par0 + r) & 1;
    const int npairs = (wc - par) >> 1;
    const int c = par + 2 * k;
    if (k < npairs) cp_async16(sr + c, gr + c);
    if (k == NP - 1 && par) cp_async8(sr, gr);
    const int last = par + 2 * npairs;
    if (k == NP - 2 && last < wc) cp_async8(sr + last, gr + last);
  }
}

// Alg. 1 on one pole held in registers (l <= 5): load n points from SMEM,
// transform with the level structure resolved at compile time, store back.
// Hierarchization reads the values entering the axis (one-pass stencil,
// bitwise equal to the in-place level order).
template <int L, bool INV>
__device__ __forceinline__ void pole_regs(double *p, int STR) {
  constexpr int n = (1 << L) - 1;
  double v[n];
#pragma unroll
  for (int i = 0; i < n; ++i) v[i] = p[i * STR];
  if (!INV) {
#pragma unroll
    for (int i = 1; i <= n; ++i) {
      const int s = i & -i;
      double x = v[i - 1];
      if (i - s >= 1) x = x - 0.5 * v[i - s - 1];
      if (i + s <= n) x = x - 0.5 * v[i + s - 1];
      p[(i - 1) * STR] = x;
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
    for (int i = 0; i < n; ++i) p[i * STR] = v[i];
  }
}

// Alg. 1 on one longer pole (5 <= L <= 7) in registers, by the block + coarse
// lattice decomposition of SURVEY 8(a) a3.iii applied inside one thread:
// points with tz(i) < 3 have both predecessors in their aligned 8-point block
// [8b, 8b+8], so each block is transformed from 9 registers; the coarse points
// {8j} form a level-(L-3) pole (stride 8) done by pole_regs.  Hierarchization:
// blocks first (they read the unmodified coarse ends), then the lattice;
// dehierarchization: lattice first, then the blocks coarse -> fine.  Same
// per-point operations as Alg. 1, so bitwise identical.
template <int L, bool INV>
__device__ __forceinline__ void pole_blocked(double *p, int STR) {
  constexpr int T = 3;
  constexpr int B = 1 << T;
  constexpr int n = (1 << L) - 1;
  constexpr int nb = 1 << (L - T);
  if (INV) pole_regs<L - T, true>(p + (B - 1) * STR, B * STR);
#pragma unroll
  for (int b = 0; b < nb; ++b) {
    double v[B + 1];
#pragma unroll
    for (int r = 0; r <= B; ++r) {
      const int i = b * B + r;
      v[r] = (i >= 1 && i <= n) ? p[(i - 1) * STR] : 0.0;   // i = 0 / 2^L: boundary, never used
    }
    if (!INV) {
#pragma unroll
      for (int r = 1; r < B; ++r) {
        const int i = b * B + r;
        const int s = r & -r;
        double x = v[r];
        if (i - s >= 1) x = x - 0.5 * v[r - s];
        if (i + s <= n) x = x - 0.5 * v[r + s];
        p[(i - 1) * STR] = x;
      }
    } else {
#pragma unroll
      for (int s = B / 2; s >= 1; s >>= 1) {
#pragma unroll
        for (int r = s; r < B; r += 2 * s) {
          const int i = b * B + r;
          double x = v[r];
          if (i - s >= 1) x = x + 0.5 * v[r - s];
          if (i + s <= n) x = x + 0.5 * v[r + s];
          v[r] = x;
        }
      }
#pragma unroll
      for (int r = 1; r < B; ++r) p[(b * B + r - 1) * STR] = v[r];
    }
  }
  if (!INV) pole_regs<L - T, false>(p + (B - 1) * STR, B * STR);
}

// One aligned 8-point block of a (lattice) pole held in 9 registers.  p0 is the
// address of the virtual point j = 0 of the lattice (never dereferenced), point
// j at p0[j*STR]; the lattice has nblk blocks, i.e. n = 8*nblk - 1 points.
// Writes only the block's fine points j = 8b+1 .. 8b+7 (a3.iii).
template <bool INV>
__device__ __forceinline__ void block8(double *p0, int STR, int b, int nblk) {
  double v[9];
  const int n = 8 * nblk - 1;
#pragma unroll
  for (int r = 0; r <= 8; ++r) {
    const int j = 8 * b + r;
    v[r] = (j >= 1 && j <= n) ? p0[j * STR] : 0.0;
  }
  if (!INV) {
#pragma unroll
    for (int r = 1; r < 8; ++r) {
      const int s = r & -r;
      const int j = 8 * b + r;
      double x = v[r];
      if (j - s >= 1) x = x - 0.5 * v[r - s];    // left predecessor
      if (j + s <= n) x = x - 0.5 * v[r + s];    // right predecessor
      p0[j * STR] = x;
    }
  } else {
#pragma unroll
    for (int s = 4; s >= 1; s >>= 1) {
#pragma unroll
      for (int r = s; r < 8; r += 2 * s) {
        const int j = 8 * b + r;
        double x = v[r];
        if (j - s >= 1) x = x + 0.5 * v[r - s];
        if (j + s <= n) x = x + 0.5 * v[r + s];
        v[r] = x;
      }
    }
#pragma unroll
    for (int r = 1; r < 8; ++r) p0[(8 * b + r) * STR] = v[r];
  }
}

template <bool INV>
__device__ __forceinline__ void pole_regs_rt(double *p, int L, int STR) {
  switch (L) {
    case 2: pole_regs<2, INV>(p, STR); break;
    case 3: pole_regs<3, INV>(p, STR); break;
    case 4: pole_regs<4, INV>(p, STR); break;
    default: break;                              // L = 1: a single point, no update
  }
}

// One axis of a staged tile, all npoles poles of level l (pole p = (oo, rk, c)
// at sm + (oo*n*R + rk)*RS + c, point stride R*RS), in parallel work items:
// l <= 4: one register pole per thread; l >= 5: (pole, 8-block) items on the
// level-l pole, then on its coarse lattice (stride x8, level l-3), ... until
// the lattice has l' <= 4, done as register poles.  A barrier between lattice
// levels; hierarchization runs fine -> coarse, dehierarchization the reverse.
template <bool INV, int W>
__device__ __forceinline__ void fused_axis(double *sm, int RS, int l, int R, const FDiv &fR, int Ok) {
  constexpr int LOGW = (W == 1) ? 0 : (W == 8) ? 3 : (W == 16) ? 4 : (W == 32) ? 5 : (W == 64) ? 6 : 7;
  const int n = (1 << l) - 1;
  const int npoles = Ok * R * W;
  const int STR = R * RS;
  auto pole_base = [&](int p) -> double * {
    const int c = p & (W - 1);
    const int rest = p >> LOGW;
    const int oo = (int)fdiv((uint32_t)rest, fR);
    const int rk = rest - oo * R;
    return sm + (oo * n * R + rk) * RS + c;
  };
  if (l <= 4) {
    for (int p = threadIdx.x; p < npoles; p += kThreads) pole_regs_rt<INV>(pole_base(p), l, STR);
    __syncthreads();
    return;
  }
  // lattice levels visited: l, l-3, l-6, ... (> 4), then the register lattice
  int levels[8], nlev = 0, lf = l;
  while (lf > 4) {
    levels[nlev++] = lf;
    lf -= 3;
  }
  const FDiv fP = device_fdiv((uint32_t)npoles);
  auto block_phase = [&](int k) {                // k-th lattice level: stride 8^k
    const int m = 1 << (3 * k);
    const int nblk = 1 << (levels[k] - 3);
    const int items = npoles * nblk;
    for (int it = threadIdx.x; it < items; it += kThreads) {
      const int b = (int)fdiv((uint32_t)it, fP);
      const int p = it - b * npoles;             // lanes run over poles: conflict-free SMEM
      block8<INV>(pole_base(p) - STR, m * STR, b, nblk);
    }
    __syncthreads();
  };
  auto lattice_phase = [&]() {
    const int m = 1 << (3 * nlev);
    for (int p = threadIdx.x; p < npoles; p += kThreads) {
      double *p0 = pole_base(p) - STR;           // virtual point 0
      pole_regs_rt<INV>(p0 + m * STR, lf, m * STR);
    }
    __syncthreads();
  };
  if (!INV) {
    for (int k = 0; k < nlev; ++k) block_phase(k);
    lattice_phase();
  } else {
    lattice_phase();
    for (int k = nlev - 1; k >= 0; --k) block_phase(k);
  }
}

// Alg. 1 on one pole of n = 2^l - 1 points at p[0], p[STR], ... (serial)
template <bool INV>
__device__ __forceinline__ void pole_serial(double *p, int l, int STR) {
  const int n = (1 << l) - 1;
  if (!INV) {
    for (int s = 1; s < (1 << (l - 1)); s <<= 1) {        // levels l .. 2, finest first
#pragma unroll 2
      for (int i = s; i <= n; i += 2 * s) {
        double x = p[(i - 1) * STR];
        if (i - s >= 1) x = x - 0.5 * p[(i - s - 1) * STR];
        if (i + s <= n) x = x - 0.5 * p[(i + s - 1) * STR];
        p[(i - 1) * STR] = x;
      }
    }
  } else {
    for (int s = 1 << (l - 2); s >= 1; s >>= 1) {           // levels 2 .. l (reading R9)
#pragma unroll 2
      for (int i = s; i <= n; i += 2 * s) {
        double x = p[(i - 1) * STR];
        if (i - s >= 1) x = x + 0.5 * p[(i - s - 1) * STR];
        if (i + s <= n) x = x + 0.5 * p[(i + s - 1) * STR];
        p[(i - 1) * STR] = x;
      }
    }
  }
}

// geometry of one FUSED tile
struct FusedTile {
  double *g;   // global base: W == 1 start of the range; W > 1 row 0 at column c0
  int units;   // W == 1: units in this tile
  int wc;      // W > 1: valid columns
  int par;     // 8-byte phase of g (SMEM data starts at stage + par)
};

template <int W>
__device__ __forceinline__ FusedTile fused_tile(const Task &T, int64_t q) {
  FusedTile f;
  if (W == 1) {
    const int64_t u0 = q * T.R;
    f.units = (int)min((int64_t)T.R, T.O - u0);
    f.g = T.grid + T.base + u0 * T.P;
    f.wc = 1;
  } else {
    const int64_t cb = q % T.ncb;
    const int64_t o = q / T.ncb;
    const int64_t c0 = cb * W;
    f.units = 1;
    f.wc = (int)min((int64_t)W, T.S - c0);
    f.g = T.grid + T.base + o * T.OS + c0;        // (row r, col c) at g[r*S + c]
  }
  f.par = phase8(f.g);
  return f;
}

template <int W>
__device__ __forceinline__ void fused_issue(const Task &T, const FusedTile &f, double *stage) {
  if (W == 1) copy_range_async(stage + f.par, f.g, f.units * T.P);
  else if (W >= 64) fused_load_rows_wide<(W >= 64 ? W : 64)>(stage + f.par, f.g, T.S, f.par, T.P, f.wc);
  else fused_load_rows<(W == 1 || W >= 64 ? 8 : W)>(stage + f.par, f.g, T.S, f.par, T.P, f.wc);
}

// all axes of the group on a staged tile, then the store
template <bool INV, int W>
__device__ __forceinline__ void fused_compute_store(const Task &T, const FusedTile &f, double *sm) {
  constexpr int RS = (W == 1) ? 1 : W + 1;
  constexpr int LOGW = (W == 1) ? 0 : (W == 8) ? 3 : (W == 16) ? 4 : (W == 32) ? 5 : (W == 64) ? 6 : 7;
  const int P = T.P;
  const int units = f.units, wc = f.wc;
  const int64_t S = T.S;
  double *gbase = f.g;
    const int rows_total = units * P;
    for (int j = 0; j < T.m; ++j) {                   // axes ascending
      const int l = T.gl[j];
      if (l <= 1) continue;
      const int n = (1 << l) - 1;
      const int R = T.gR[j];
      const FDiv fR = T.fR[j];
      const int Ok = rows_total / (n * R);
      fused_axis<INV, W>(sm, RS, l, R, fR, Ok);
    }
    if (W == 1) {
      for (int e = threadIdx.x; e < rows_total; e += kThreads) __stcg(gbase + e, sm[e]);
    } else {
      constexpr int RPI = (W >= 32) ? 1 : 32 / W;   // rows per warp instruction
      constexpr int CPL = (W >= 32) ? W / 32 : 1;   // columns per lane
      constexpr int STEP = RPI * (kThreads / 32);
      const int lane = threadIdx.x & 31;
      const int c0 = (W >= 32) ? lane : lane % W;
      int row = (threadIdx.x >> 5) * RPI + ((W >= 32) ? 0 : lane / W);
      double *gr = gbase + (int64_t)row * S;
      const double *sr = sm + row * RS;
      const int64_t gstep = (int64_t)STEP * S;
#pragma unroll 2
      for (; row < P; row += STEP, gr += gstep, sr += STEP * RS) {
#pragma unroll
        for (int u = 0; u < CPL; ++u) {
          const int c = c0 + 32 * u;
          if (c < wc) __stcg(gr + c, sr[c]);
        }
      }
    }
}

// Persistent, double-buffered: while a CTA transforms tile k in one SMEM stage,
// the cp.async copies of tile k+1 fill the other, so HBM reads overlap the
// SMEM work instead of alternating with it.
#ifndef FUSED_MINB
#define FUSED_MINB 3   // resident CTAs per SM the FUSED register budget is sized for
#endif
template <bool INV, int W, int STAGES>
__global__ void __launch_bounds__(kThreads, (STAGES == 1 ? FUSED_MINB : 2)) k_fused(const __grid_constant__ Src src) {
  extern __shared__ __align__(16) double smem[];
  __shared__ Task s_task[2];                      // descriptors of the two in-flight tiles
  int64_t q = blockIdx.x;
  if (q >= src.total_tiles) return;
  int idx = -1;
  auto stage_task = [&](Task *dst, const Task *from) {
    const uint64_t *a = reinterpret_cast<const uint64_t *>(from);
    uint64_t *b = reinterpret_cast<uint64_t *>(dst);
    for (int i = threadIdx.x; i < (int)(sizeof(Task) / 8); i += kThreads) b[i] = a[i];
  };
  auto ref = [&](int64_t qq, int64_t &ql) -> const Task * {
    if (!src.tasks) {
      ql = qq;
      return &src.single;
    }
    idx = (idx < 0) ? first_task(src, qq) : advance_task(src, idx, qq);
    ql = qq - __ldg(&src.prefix[idx]);
    return &src.tasks[idx];
  };
  int64_t ql;
  const Task *Tc = ref(q, ql);
  FusedTile fc = fused_tile<W>(*Tc, ql);
  fused_issue<W>(*Tc, fc, smem);
  cp_async_commit();
  stage_task(&s_task[0], Tc);
  for (int k = 0;; ++k) {
    double *cur = smem + (STAGES == 2 ? (k & 1) * src.stage_doubles : 0);
    const int64_t qn = q + gridDim.x;
    const bool more = qn < src.total_tiles;
    const Task *Tn = Tc;
    FusedTile fn = fc;
    if (STAGES == 2 && more) {
      int64_t qln;
      Tn = ref(qn, qln);
      fn = fused_tile<W>(*Tn, qln);
      fused_issue<W>(*Tn, fn, smem + ((k + 1) & 1) * src.stage_doubles);
      cp_async_commit();
      stage_task(&s_task[(k + 1) & 1], Tn);
      cp_async_wait<1>();                         // tile k has landed (tile k+1 may be in flight)
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();
    fused_compute_store<INV, W>(s_task[STAGES == 2 ? (k & 1) : 0], fc, cur + fc.par);
    __syncthreads();                              // the stage is free for the next load
    if (!more) break;
    q = qn;
    if (STAGES == 1) {                            // single stage: load the next tile now
      int64_t qln;
      Tn = ref(qn, qln);
      fn = fused_tile<W>(*Tn, qln);
      fused_issue<W>(*Tn, fn, smem);
      cp_async_commit();
      stage_task(&s_task[0], Tn);
    }
    Tc = Tn;
    fc = fn;
  }
}

// ----------------------------------------------------------------------- REG
// One thread per column (o, r); the whole pole of n = 2^L - 1 points lives in
// registers; the level structure is resolved at compile time.  Each thread
// handles CPT columns (c, c + 256, ...) so that ~16 independent loads are in
// flight per thread.  A tile = kThreads * CPT columns.
template <int L>
struct RegCfg {
  static constexpr int n = (1 << L) - 1;
  static constexpr int CPT = (16 / n) > 0 ? (16 / n) : 1;
};

template <int L, bool INV>
__global__ void __launch_bounds__(kThreads) k_reg(const __grid_constant__ Src src) {
  constexpr int n = RegCfg<L>::n;
  constexpr int CPT = RegCfg<L>::CPT;
  for_each_tile(src, [&](const Task &T, int64_t q) {
    const int64_t ncol = T.O * T.S;
    const int64_t PS = T.PS;
    double *p[CPT];
    double v[CPT][n];
#pragma unroll
    for (int c = 0; c < CPT; ++c) {
      const int64_t gcol = (q * CPT + c) * kThreads + threadIdx.x;
      p[c] = nullptr;
      if (gcol < ncol) {
        const int64_t o = gcol / T.S;
        const int64_t r = gcol - o * T.S;
        p[c] = T.grid + T.base + o * T.OS + r;
#pragma unroll
        for (int i = 0; i < n; ++i) v[c][i] = p[c][i * PS];
      }
    }
#pragma unroll
    for (int c = 0; c < CPT; ++c) {
      if (!p[c]) continue;
      if (!INV) {
        // v keeps the values entering the sweep; results go straight to memory
#pragma unroll
        for (int i = 1; i <= n; ++i) {
          const int s = i & -i;
          double x = v[c][i - 1];
          if (i - s >= 1) x = x - 0.5 * v[c][i - s - 1];
          if (i + s <= n) x = x - 0.5 * v[c][i + s - 1];
          p[c][(i - 1) * PS] = x;
        }
      } else {
#pragma unroll
        for (int lam = 2; lam <= L; ++lam) {
          const int s = 1 << (L - lam);
#pragma unroll
          for (int i = s; i <= n; i += 2 * s) {
            double x = v[c][i - 1];
            if (i - s >= 1) x = x + 0.5 * v[c][i - s - 1];
            if (i + s <= n) x = x + 0.5 * v[c][i + s - 1];
            v[c][i - 1] = x;
          }
        }
#pragma unroll
        for (int i = 0; i < n; ++i) p[c][i * PS] = v[c][i];
      }
    }
  });
}

// ------------------------------------------------------------ host launchers
using KernelFn = void (*)(Src);

// FUSED pipeline depth: 1 (default) or 2 stages (tuning override SGH_FUSED_STAGES)
int fused_stages() {
  static int st = -1;
  if (st < 0) {
    const char *e = getenv("SGH_FUSED_STAGES");
    st = (e && atoi(e) == 2) ? 2 : 1;
  }
  return st;
}

static KernelFn kernel_for(int kind, int l, int w, bool inv) {
  switch (kind) {
    case KIND_FLAT_SLABS: return inv ? k_flat_slabs<true> : k_flat_slabs<false>;
    case KIND_FLAT_BLOCKS: return inv ? k_flat_blocks<true> : k_flat_blocks<false>;
    case KIND_STRIDED:
      switch (w) {
        case 32: return inv ? k_strided<true, 32> : k_strided<false, 32>;
        case 64: return inv ? k_strided<true, 64> : k_strided<false, 64>;
        case 128: return inv ? k_strided<true, 128> : k_strided<false, 128>;
        case 256: return inv ? k_strided<true, 256> : k_strided<false, 256>;
        default: return nullptr;
      }
    case KIND_FUSED:
      if (fused_stages() == 2) {
        switch (w) {
          case 1: return inv ? k_fused<true, 1, 2> : k_fused<false, 1, 2>;
          case 8: return inv ? k_fused<true, 8, 2> : k_fused<false, 8, 2>;
          case 16: return inv ? k_fused<true, 16, 2> : k_fused<false, 16, 2>;
          case 32: return inv ? k_fused<true, 32, 2> : k_fused<false, 32, 2>;
          case 64: return inv ? k_fused<true, 64, 2> : k_fused<false, 64, 2>;
          case 128: return inv ? k_fused<true, 128, 2> : k_fused<false, 128, 2>;
          default: return nullptr;
        }
      }
      switch (w) {
        case 1: return inv ? k_fused<true, 1, 1> : k_fused<false, 1, 1>;
        case 8: return inv ? k_fused<true, 8, 1> : k_fused<false, 8, 1>;
        case 16: return inv ? k_fused<true, 16, 1> : k_fused<false, 16, 1>;
        case 32: return inv ? k_fused<true, 32, 1> : k_fused<false, 32, 1>;
        case 64: return inv ? k_fused<true, 64, 1> : k_fused<false, 64, 1>;
        case 128: return inv ? k_fused<true, 128, 1> : k_fused<false, 128, 1>;
        default: return nullptr;
      }
    case KIND_REG:
      switch (l) {
        case 2: return inv ? k_reg<2, true> : k_reg<2, false>;
        case 3: return inv ? k_reg<3, true> : k_reg<3, false>;
        case 4: return inv ? k_reg<4, true> : k_reg<4, false>;
        default: return nullptr;
      }
    default: return nullptr;
  }
}

// dynamic shared memory a task needs
size_t task_smem(const Task &t) {
  const int64_t n = (int64_t(1) << t.l) - 1;
  switch (t.kind) {
    case KIND_FLAT_SLABS: return (size_t(t.R) * size_t(n * t.S) + 2) * 8;            // +1 phase shift
    case KIND_FLAT_BLOCKS: return (size_t((int64_t(1) << t.t) + 1) * size_t(t.S) + 2) * 8;
    case KIND_STRIDED: return size_t((int64_t(1) << t.t) + 1) * size_t(t.W + 2) * 8;
    case KIND_FUSED:
      return t.W == 1 ? (size_t(t.R) * size_t(t.P) + 2) * 8 : (size_t(t.P) * size_t(t.W + 1) + 2) * 8;
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
  if (smem > 48 * 1024) {
    // opt in to large dynamic shared memory (FUSED tiles up to ~70 KB)
    cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  }
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
  KernelFn fn = kernel_for(task.kind, task.l, task.W, inv);
  if (!fn) return cudaErrorInvalidValue;
  Src src{};
  src.tasks = nullptr;
  src.prefix = nullptr;
  src.ntasks = 1;
  src.total_tiles = task.tiles;
  src.single = task;
  size_t smem = task_smem(task);
  if (task.kind == KIND_FUSED) {                 // pipeline stages, 16-byte aligned
    src.stage_doubles = (int32_t)((smem + 15) / 16 * 2);
    smem = size_t(fused_stages()) * src.stage_doubles * 8;
  }
  const int64_t cap = resident_ctas(fn, smem);
  const int64_t grid = task.tiles < cap ? task.tiles : cap;
  if (grid <= 0) return cudaSuccess;
  ProfToken tok = prof_begin(stream);
  fn<<<(unsigned)grid, kThreads, smem, stream>>>(src);
  cudaError_t e = cudaGetLastError();
  prof_end(tok, task.kind, task.kind == KIND_FUSED || task.kind == KIND_STRIDED ? task.W : task.l, inv,
           16.0 * task_points(task), stream);
  return e;
}

// Launch a group of tasks of one kernel instance from a device task table;
// smem = max task_smem over the group.
cudaError_t launch_table(int kind, int l, int w, bool inv, const Task *d_tasks, const int64_t *d_prefix,
                         int32_t ntasks, int64_t total_tiles, size_t smem, double points, cudaStream_t stream) {
  KernelFn fn = kernel_for(kind, l, w, inv);
  if (!fn) return cudaErrorInvalidValue;
  Src src{};
  src.tasks = d_tasks;
  src.prefix = d_prefix;
  src.ntasks = ntasks;
  src.total_tiles = total_tiles;
  if (kind == KIND_FUSED) {
    src.stage_doubles = (int32_t)((smem + 15) / 16 * 2);
    smem = size_t(fused_stages()) * src.stage_doubles * 8;
  }
  const int64_t cap = resident_ctas(fn, smem);
  const int64_t grid = total_tiles < cap ? total_tiles : cap;
  if (grid <= 0) return cudaSuccess;
  ProfToken tok = prof_begin(stream);
  fn<<<(unsigned)grid, kThreads, smem, stream>>>(src);
  cudaError_t e = cudaGetLastError();
  prof_end(tok, kind, kind == KIND_FUSED || kind == KIND_STRIDED ? w : l, inv, 16.0 * points, stream);
  return e;
}

}  // namespace sgh
