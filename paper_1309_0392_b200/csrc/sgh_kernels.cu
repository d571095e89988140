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
#include <type_traits>
#include <algorithm>
#include <cstdlib>
#include <mutex>

#include "sgh_common.cuh"
#include "sgh_plan.hpp"

namespace sgh {

// One term of an update with the oracle's rounding (oracle.c is built with
// -ffp-contract=off): the product 0.5 e is rounded on its own, then the sum.
// Written with explicit _rn intrinsics so nvcc cannot contract them into a
// DFMA -- 0.5 e is exact for normal e, but not for subnormal e with an odd
// last bit, where a fused multiply-add would round once instead of twice.
__device__ __forceinline__ double hsub(double x, double e) { return __dsub_rn(x, __dmul_rn(0.5, e)); }
__device__ __forceinline__ double hadd(double x, double e) { return __dadd_rn(x, __dmul_rn(0.5, e)); }

// The hierarchization update of one point from its two predecessors, each
// skipped if it lies on the boundary: x - 0.5 L, then
// - 0.5 R (reading R5).  -DSGH_REDUCED_OP builds the paper's reduced-op
// variant x - 0.5 (L + R) as an ablation: one multiply less, different
// rounding (the paper saw no runtime gain; DESIGN.md reports B200).
#ifdef SGH_REDUCED_OP
#define HIER_UPDATE(x, cl, el, cr, er)           \
  do {                                           \
    const bool hl_ = (cl), hr_ = (cr);           \
    if (hl_ && hr_) x = hsub(x, __dadd_rn((el), (er))); \
    else if (hl_) x = hsub(x, (el));             \
    else if (hr_) x = hsub(x, (er));             \
  } while (0)
#else
#define HIER_UPDATE(x, cl, el, cr, er) \
  do {                                 \
    if (cl) x = hsub(x, (el));         \
    if (cr) x = hsub(x, (er));         \
  } while (0)
#endif

// threads of a FUSED CTA, per tile kind (W == 1 contiguous / W > 1 column
// tiles): 128 threads, 3 CTAs per SM, 70 KB tiles.  Measured on C5 (with the
// host planning cached, so the step is GPU-bound): 128 threads 150.9, 192
// 146.7, 256 143.0, 96 146.5 Gpoints/s -- a tile's in-SMEM transform is a
// sequence of barrier-separated phases, and fewer warps per barrier wait less.
// Tuning: SGH_FUSED_THREADS(_W1), FUSED_MINB(_W1), planner SGH_FUSED_T(1).
#ifndef SGH_FUSED_THREADS
#define SGH_FUSED_THREADS 128
#endif
#ifndef SGH_FUSED_THREADS_W1
#define SGH_FUSED_THREADS_W1 128
#endif
template <int W>
struct FT {
  static constexpr int v = (W == 1) ? SGH_FUSED_THREADS_W1 : SGH_FUSED_THREADS;
};

struct Src {
  const Task *tasks;      // device task table, or nullptr -> use `single`
  const int64_t *prefix;  // device exclusive prefix of task tiles, ntasks+1 entries
  int32_t ntasks;
  int32_t stage_doubles;  // FUSED: SMEM doubles per pipeline stage (2 stages)
  int64_t total_tiles;
  int32_t nstages;        // k_fpipe: stages of the SMEM ring
  int32_t pad_;
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

// TMA bulk store (cp.async.bulk shared -> global, SASS UBLKCP): the FUSED W == 1
// tiles write their contiguous ranges back through the async copy engine
// instead of an LDS + STG per element.  SMEM element e sits at the same 16-byte
// phase as its global address (the stage is offset by the tile's phase), so the
// 16-byte aligned interior of a range is one bulk copy; its 8-byte ends are
// stored by the issuing thread.  Issued by ONE thread, after
// fence.proxy.async + a barrier (the tile's SMEM writes come from the generic
// proxy); the stage is reused only after cp.async.bulk.wait_group.read.
#ifndef SGH_BULK_STORE
#define SGH_BULK_STORE 1
#endif
__device__ __forceinline__ void bulk_store_range(double *g, const double *s, int len) {
  if (len <= 0) return;
  const int head = phase8(g);
  const int pairs = (len - head) >> 1;
  const int last = head + 2 * pairs;
  if (head) __stcg(g, s[0]);
  if (last < len) __stcg(g + last, s[last]);
  if (pairs > 0) {
    const unsigned sa = (unsigned)__cvta_generic_to_shared(s + head);
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;\n" ::"l"(g + head), "r"(sa),
                 "r"(pairs * 16)
                 : "memory");
  }
}
__device__ __forceinline__ void bulk_fence_barrier() {
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  __syncthreads();
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;\n" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read() { asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory"); }

// Copy len doubles gsrc[0..len) -> sdst[0..len) where sdst and gsrc have the
// same 16-byte phase: 8-byte head/tail, 16-byte body.  Issue only.
template <int NT = kThreads>
__device__ __forceinline__ void copy_range_async(double *sdst, const double *gsrc, int len) {
  if (len <= 0) return;
  const int head = phase8(gsrc) ? 1 : 0;
  const int pairs = (len - head) >> 1;
  const int tail = len - head - 2 * pairs;
  if (head && threadIdx.x == 0) cp_async8(sdst, gsrc);
  if (tail && threadIdx.x == NT - 1) cp_async8(sdst + len - 1, gsrc + len - 1);
  const double *g = gsrc + head;
  double *s = sdst + head;
#pragma unroll 4
  for (int p = threadIdx.x; p < pairs; p += NT) cp_async16(s + 2 * p, g + 2 * p);
}

// Task index owning tile q.  `idx` is the cursor from the previous tile of this
// CTA (tiles only increase).  A CTA's tiles are gridDim.x apart, which can skip
// hundreds of small tasks (the C5 set: thousands of grids with a few tiles
// each), so the search gallops from the cursor (1, 2, 4, .. tasks ahead) and
// then bisects: O(log gap) dependent loads instead of O(gap).
__device__ __forceinline__ int advance_task(const Src &src, int idx, int64_t q) {
  if (idx + 1 >= src.ntasks || __ldg(&src.prefix[idx + 1]) > q) return idx;
  int lo = idx + 1, step = 1;                      // prefix[lo] <= q
  int hi = lo + 1;
  while (hi < src.ntasks && __ldg(&src.prefix[hi]) <= q) {
    lo = hi;
    step <<= 1;
    hi = lo + step;
  }
  if (hi > src.ntasks) hi = src.ntasks;            // answer in [lo, hi): prefix[hi] > q or hi == ntasks
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if (__ldg(&src.prefix[mid]) <= q) lo = mid; else hi = mid;
  }
  return lo;
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
    const int64_t cb = q % T.ncb;
    const int64_t rest = q / T.ncb;
    const int b = (int)(T.blk0 + (rest & ((int64_t(1) << T.rlog) - 1)));
    const int64_t o = rest >> T.rlog;
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
            HIER_UPDATE(x, i - s >= 1, xl[c], i + s <= n, xr[c]);
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
            if (i - s >= 1) x = hadd(x, xl[c]);
            if (i + s <= n) x = hadd(x, xr[c]);
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

// rows 0..P-1 of W columns (wc valid), global row r at g + r*S (S odd), SMEM row r at sb + r*(W+1).
// Lane = (sub-row, 16-byte slot): one warp instruction covers 32/(W/2) rows.
template <int W>
__device__ __forceinline__ void fused_load_rows_wide(double *sb, const double *g, int64_t S, int par0, int P, int wc) {
  constexpr int RS = W + 1;
  constexpr int NP = W / 2;                       // 16-byte slots per row (32 or 64)
  constexpr int LOGP = (NP == 32) ? 5 : 6;
  const int nslots = P * NP;
#pragma unroll 4
  for (int p = threadIdx.x; p < nslots; p += FT<W>::v) {
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
  constexpr int STEP = RPI * (FT<W>::v / 32);     // rows per CTA iteration
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
      HIER_UPDATE(x, i - s >= 1, v[i - s - 1], i + s <= n, v[i + s - 1]);
      p[(i - 1) * STR] = x;
    }
  } else {
#pragma unroll
    for (int lam = 2; lam <= L; ++lam) {
      const int s = 1 << (L - lam);
#pragma unroll
      for (int i = s; i <= n; i += 2 * s) {
        double x = v[i - 1];
        if (i - s >= 1) x = hadd(x, v[i - s - 1]);
        if (i + s <= n) x = hadd(x, v[i + s - 1]);
        v[i - 1] = x;
      }
    }
#pragma unroll
    for (int i = 0; i < n; ++i) p[i * STR] = v[i];
  }
}

// Fine part of one aligned block of 2^T points of a pole together with its two
// end points: local point r = 0..2^T at p0[r*STR].  Every
// r = 1..2^T-1 has both predecessors r -+ 2^{tz(r)} inside [0, 2^T], so the
// block is transformed from 2^T + 1 registers: hierarchization from the values
// entering the pass (one-pass stencil), dehierarchization coarse -> fine with
// nodal ends.  An end with !lo_ok / !hi_ok is the zero boundary: it is
// never read and the update that would use it is skipped -- the same
// operations as Alg. 1 on the whole pole, hence bitwise identical.
// ENDS: both ends are known to be grid points (an interior block): the
// boundary predicates fold away at compile time.
template <int T, bool INV, bool ENDS = false>
__device__ __forceinline__ void block_fine(double *p0, int STR, bool lo_ok, bool hi_ok) {
  constexpr int B = 1 << T;
  if (ENDS) lo_ok = hi_ok = true;
  double v[B + 1];
  v[0] = lo_ok ? p0[0] : 0.0;
#pragma unroll
  for (int r = 1; r < B; ++r) v[r] = p0[r * STR];
  v[B] = hi_ok ? p0[B * STR] : 0.0;
  if (!INV) {
#pragma unroll
    for (int r = 1; r < B; ++r) {
      const int s = r & -r;
      double x = v[r];
      HIER_UPDATE(x, r - s > 0 || lo_ok, v[r - s], r + s < B || hi_ok, v[r + s]);   // left, right
      p0[r * STR] = x;
    }
  } else {
#pragma unroll
    for (int s = B / 2; s >= 1; s >>= 1) {               // coarse -> fine (reading R9)
#pragma unroll
      for (int r = s; r < B; r += 2 * s) {
        double x = v[r];
        if (r - s > 0 || lo_ok) x = hadd(x, v[r - s]);
        if (r + s < B || hi_ok) x = hadd(x, v[r + s]);
        v[r] = x;
      }
    }
#pragma unroll
    for (int r = 1; r < B; ++r) p0[r * STR] = v[r];
  }
}

// Work items of the in-SMEM pole transforms are aligned blocks of 2^kTB points
// (kTB fine levels in 2^kTB + 1 registers per item; kTB = 4 with 128-thread CTAs: C2 +1.5 %,
// C3 +3 %, C5 +0.5 % over kTB = 3); a pole of level l
// is done as blocks at stride 1, then its coarse lattice (stride 2^kTB, level
// l - kTB) the same way, until the lattice fits one register pole.
#ifndef SGH_TB
#define SGH_TB 4
#endif
constexpr int kTB = SGH_TB;


// One aligned block b of 2^kTB points of a (lattice) pole of nblk blocks: p0 is
// the address of the virtual point j = 0 of the lattice (never dereferenced),
// point j at p0[j*STR], n = 2^kTB nblk - 1 points; its ends are the boundary
// only for the first / last block.  Writes only the block's fine points.
template <bool INV>
__device__ __forceinline__ void block_item(double *p0, int STR, int b, int nblk) {
  if (b > 0 && b < nblk - 1) block_fine<kTB, INV, true>(p0 + (b << kTB) * STR, STR, true, true);
  else block_fine<kTB, INV>(p0 + (b << kTB) * STR, STR, b > 0, b < nblk - 1);
}

// block b of a BLOCKED axis' sub-lattice: its ends are grid points unless it is
// the first / last sub-block of a tile block that touches the boundary
template <bool INV>
__device__ __forceinline__ void block_item_ends(double *p0, int STR, bool lo, bool hi) {
  if (lo && hi) block_fine<kTB, INV, true>(p0, STR, true, true);
  else block_fine<kTB, INV>(p0, STR, lo, hi);
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

// Thread-strided walk over work items it = b * npoles + p (p fastest) without a
// division per item: (b, p) advance by (step / npoles, step % npoles).
struct ItemWalk {
  int np, db, dp, b0, p0;
  __device__ __forceinline__ ItemWalk(int npoles, int start, int step, const FDiv *f = nullptr)
      : np(npoles) {
    if (f) {                                      // host-precomputed division by npoles
      db = (int)fdiv((uint32_t)step, *f);
      b0 = (int)fdiv((uint32_t)start, *f);
    } else {
      db = step / npoles;
      b0 = start / npoles;
    }
    dp = step - db * npoles;
    p0 = start - b0 * npoles;
  }
  __device__ __forceinline__ void next(int &b, int &p) const {
    b += db;
    p += dp;
    if (p >= np) {
      p -= np;
      ++b;
    }
  }
};

// Dehierarchization of a tile with a BLOCKED axis: a pole of an axis before the
// blocked one lies in one local row y of the blocked axis.  The end rows
// y = 0 and y = 2^bt hold values that are already final (their coarse lattice
// ran first) and must not be transformed again.
struct HaloSkip {
  bool on;
  bool zs;      // also the second blocked axis' end rows (z = 0, ez2 - 1): the
                // inverse prefix two-blocked tile, whose b-end rows are final
  FDiv fA, fE;  // division by A (tile rows before the blocked axis), by ej
  int ej, ez2;
  __device__ __forceinline__ bool skip(int row) const {  // row: the pole's first local row
    if (!on) return false;
    const uint32_t q = fdiv((uint32_t)row, fA);
    const uint32_t z = fdiv(q, fE);
    const int y = (int)(q - z * (uint32_t)ej);
    return y == 0 || y == ej - 1 || (zs && (z == 0 || (int)z == ez2 - 1));
  }
};

// The threads that transform a tile together, with their barrier: the whole
// CTA (CtaSync, k_fused) or one consumer warp group of the warp-specialised
// pipelined kernel (GroupSync: named barrier `id` over NT threads, k_fpipe).
struct CtaSync {
  __device__ __forceinline__ int tid() const { return (int)threadIdx.x; }
  __device__ __forceinline__ void bar() const { __syncthreads(); }
};
template <int NT>
struct GroupSync {
  int t, id;
  __device__ __forceinline__ int tid() const { return t; }
  __device__ __forceinline__ void bar() const { asm volatile("bar.sync %0, %1;\n" ::"r"(id), "n"(NT) : "memory"); }
};

// One axis of a staged tile, all npoles poles of level l (pole p = (oo, rk, c)
// at sm + (oo*n*R + rk)*RS + c, point stride R*RS), in parallel work items:
// l <= 4: one register pole per thread; l >= 5: (pole, 2^kTB-block) items on
// the level-l pole, then on its coarse lattice (stride x2^kTB, level l-kTB),
// ... until the lattice has l' <= 4, done as register poles.  A barrier between lattice
// levels; hierarchization runs fine -> coarse, dehierarchization the reverse.
// UNIT: the axis is the tile's first (R == 1): the point stride RS is a
// compile-time constant (immediate SMEM offsets) and a pole index needs no division.
// Dense tile row -> SMEM offset: the identity (dense tiles), or the PADDED
// layout of a W == 1 tile (Task::sy > 0): row r = x + A (y + ej z) at
// x + y sy + z sz.  Poles keep their dense row enumeration; only addresses
// are remapped, and the point stride along the axis (STR) is the padded one.
struct NoRemap {
  __device__ __forceinline__ int operator()(int r) const { return r; }
};
struct PadRemap {
  FDiv fA, fE;
  int A, ej, sy, sz;
  __device__ __forceinline__ int operator()(int r) const {
    const int w = (int)fdiv((uint32_t)r, fA);
    const int z = (int)fdiv((uint32_t)w, fE);
    return r - w * A + (w - z * ej) * sy + z * sz;
  }
};

template <bool INV, int W, bool UNIT = false, int NT = FT<W>::v, class SY = CtaSync, class RM = NoRemap>
__device__ __forceinline__ void fused_axis(double *sm, int RS, int l, int R, const FDiv fR, int Ok,
                                           const HaloSkip hs, const FDiv *fnp = nullptr, const SY sy = SY(),
                                           const RM rm = RM(), int str = 0) {
  constexpr int LOGW = (W == 1) ? 0 : (W == 8) ? 3 : (W == 16) ? 4 : (W == 32) ? 5 : (W == 64) ? 6 : 7;
  if (UNIT) {
    RS = (W == 1) ? 1 : W + 1;
    R = 1;
  }
  const int n = (1 << l) - 1;
  const int npoles = Ok * R * W;
  const int STR = str > 0 ? str : R * RS;
  auto pole_row = [&](int p) -> int {
    const int rest = p >> LOGW;
    if (UNIT) return rest * n;
    const int oo = (int)fdiv((uint32_t)rest, fR);
    const int rk = rest - oo * R;
    return oo * n * R + rk;
  };
  auto pole_base = [&](int p) -> double * { return sm + rm(pole_row(p)) * RS + (p & (W - 1)); };
  // register poles of level L over all poles: the level dispatch is hoisted
  // out of the pole loop
  auto reg_poles = [&](auto LC, int off, int str) {
    constexpr int L = decltype(LC)::value;
    for (int p = sy.tid(); p < npoles; p += NT) {
      if (hs.on && hs.skip(pole_row(p))) continue;
      pole_regs<L, INV>(pole_base(p) + off, str);
    }
  };
  auto reg_poles_rt = [&](int L, int off, int str) {
    switch (L) {
      case 2: reg_poles(std::integral_constant<int, 2>(), off, str); break;
      case 3: reg_poles(std::integral_constant<int, 3>(), off, str); break;
      case 4: reg_poles(std::integral_constant<int, 4>(), off, str); break;
      default: break;                            // L = 1: a single point, no update
    }
  };
  if (l <= 4) {
    reg_poles_rt(l, 0, STR);
    sy.bar();
    return;
  }
  // lattice levels visited: l, l-kTB, l-2kTB, ... (> 4), then the register
  // lattice of level lf <= 4 (level k is l - kTB k: no array, which would
  // live in local memory)
  int nlev = 0, lf = l;
  while (lf > 4) {
    ++nlev;
    lf -= kTB;
  }
  const ItemWalk walk(npoles, (int)sy.tid(), NT, fnp);
  auto block_phase = [&](int k) {                // k-th lattice level: stride 2^{kTB k}
    const int m = 1 << (kTB * k);
    const int nblk = 1 << (l - kTB * k - kTB);
    // items (b, p), p fastest: lanes run over poles (conflict-free SMEM)
    for (int b = walk.b0, p = walk.p0; b < nblk; walk.next(b, p)) {
      if (hs.on && hs.skip(pole_row(p))) continue;
      block_item<INV>(pole_base(p) - STR, m * STR, b, nblk);
    }
    sy.bar();
  };
  auto lattice_phase = [&]() {
    if (lf <= 1) return;                         // a single point: no update
    const int m = 1 << (kTB * nlev);
    reg_poles_rt(lf, (m - 1) * STR, m * STR);    // point j of the lattice at (j m - 1) STR
    sy.bar();
  };
  if (!INV) {
    for (int k = 0; k < nlev; ++k) block_phase(k);
    lattice_phase();
  } else {
    lattice_phase();
    for (int k = nlev - 1; k >= 0; --k) block_phase(k);
  }
}

// Hierarchization of a W == 1 tile's FIRST axis (rows contiguous in SMEM,
// levels 5..9) without CTA barriers: one warp per row, the one-pass stencil
// (SURVEY 8(a)): every lane reads its points i = lane + 1 + 32 m and their two
// predecessors i -+ 2^{tz(i)} -- all values entering the pass -- then, after a
// __syncwarp, writes them.  The warp owns its row, so no other warp races it;
// the same operations as Alg. 1 per point (bitwise).
template <int C>
__device__ __forceinline__ void warp_rows_hier(double *sm, int nrows, int l) {
  const int lane = threadIdx.x & 31;
  const int n = (1 << l) - 1;
  for (int r = threadIdx.x >> 5; r < nrows; r += FT<1>::v / 32) {
    double *row = sm + r * n;                      // point i (1-based) at row[i - 1]
    double out[C];
#pragma unroll
    for (int m = 0; m < C; ++m) {
      const int i = lane + 1 + 32 * m;
      const int s = i & -i;
      if (i <= n) {
        double x = row[i - 1];
        HIER_UPDATE(x, i - s >= 1, row[i - s - 1], i + s <= n, row[i + s - 1]);
        out[m] = x;
      }
    }
    __syncwarp();
#pragma unroll
    for (int m = 0; m < C; ++m) {
      const int i = lane + 1 + 32 * m;
      if (i <= n) row[i - 1] = out[m];
    }
    __syncwarp();
  }
}

#ifndef SGH_WARP_ROWS_MAXL
#define SGH_WARP_ROWS_MAXL 7
#endif
__device__ __forceinline__ bool warp_rows_dispatch(double *sm, int nrows, int l) {
  switch (l) {
    case 5: warp_rows_hier<1>(sm, nrows, l); return true;
    case 6: warp_rows_hier<2>(sm, nrows, l); return true;
    case 7: warp_rows_hier<4>(sm, nrows, l); return true;
#if SGH_WARP_ROWS_MAXL >= 8
    case 8: warp_rows_hier<8>(sm, nrows, l); return true;
#endif
#if SGH_WARP_ROWS_MAXL >= 9
    case 9: warp_rows_hier<16>(sm, nrows, l); return true;
#endif
    default: return false;
  }
}

// The BLOCKED axis of a tile: every pole holds one aligned block of 2^t points
// plus its two ends (local y = 0..2^t, point stride R*RS); only the fine points
// y = 1..2^t-1 are transformed.  Inside the block the same
// lattice recursion as fused_axis: 2^kTB-point sub-blocks at strides 1, 2^kTB,
// .. (K = t / kTB levels), then the top lattice of 2^{t - kTB K} + 1 points.
// lo_ok / hi_ok: the block's ends are grid points (false: the zero boundary).
// skip_oe (dehierarchization of a two-blocked tile, axis a): poles in the
// first / last outer row (oo = 0, Ok - 1: the second blocked axis' end rows,
// final values) are left untouched.
template <bool INV, int W, int NT = FT<W>::v, class SY = CtaSync, class RM = NoRemap>
__device__ __forceinline__ void fused_axis_block(double *sm, int RS, int t, int R, const FDiv fR, int Ok,
                                                 bool lo_ok, bool hi_ok, const FDiv *fnp = nullptr,
                                                 bool skip_oe = false, const SY sy = SY(), const RM rm = RM(),
                                                 int str = 0) {
  constexpr int LOGW = (W == 1) ? 0 : (W == 8) ? 3 : (W == 16) ? 4 : (W == 32) ? 5 : (W == 64) ? 6 : 7;
  const int ej = (1 << t) + 1;
  const int npoles = Ok * R * W;
  const int STR = str > 0 ? str : R * RS;
  auto pole_base = [&](int p) -> double * {
    const int c = p & (W - 1);
    const int rest = p >> LOGW;
    const int oo = (int)fdiv((uint32_t)rest, fR);
    const int rk = rest - oo * R;
    return sm + rm(oo * ej * R + rk) * RS + c;   // local point y = 0
  };
  const int K = t / kTB;
  const int tr = t - kTB * K;
  const ItemWalk walk(npoles, (int)sy.tid(), NT, fnp);
  auto skip = [&](int p) -> bool {
    if (!skip_oe) return false;
    const int oo = (int)fdiv((uint32_t)(p >> LOGW), fR);
    return oo == 0 || oo == Ok - 1;
  };
  auto sub_phase = [&](int k) {
    const int m = 1 << (kTB * k);
    const int nblk = 1 << (t - kTB * k - kTB);
    for (int b = walk.b0, p = walk.p0; b < nblk; walk.next(b, p)) {
      if (skip(p)) continue;
      block_item_ends<INV>(pole_base(p) + (b << kTB) * m * STR, m * STR, lo_ok || b > 0, hi_ok || b < nblk - 1);
    }
    sy.bar();
  };
  auto top_phase = [&]() {
    if (tr == 0) return;                         // the top lattice is just the two ends
    const int m = 1 << (kTB * K);
    for (int p = sy.tid(); p < npoles; p += NT) {
      if (skip(p)) continue;
      if (tr == 1) block_fine<1, INV>(pole_base(p), m * STR, lo_ok, hi_ok);
      else if (tr == 2 || kTB <= 3) block_fine<2, INV>(pole_base(p), m * STR, lo_ok, hi_ok);
      else block_fine<(kTB > 3 ? 3 : 2), INV>(pole_base(p), m * STR, lo_ok, hi_ok);
    }
    sy.bar();
  };
  if (!INV) {
    for (int k = 0; k < K; ++k) sub_phase(k);
    top_phase();
  } else {
    top_phase();
    for (int k = K - 1; k >= 0; --k) sub_phase(k);
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
    // dehierarchization with few columns (S < 32): the lanes of a level are
    // 2s S doubles apart, so the SMEM tile is padded by one double per 32
    // (element e at e + e/32) to spread them over the banks
    const bool padded = INV && S < 32;
    if (padded) {
      for (int e = threadIdx.x; e < len; e += kThreads) cp_async8(smem + e + (e >> 5), g + e);
    } else {
      copy_range_async(sm, g, len);
    }
    cp_async_wait_all();
    __syncthreads();
    if (padded) {
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
          double x = smem[e + (e >> 5)];
          if (i - s >= 1) x = hadd(x, smem[(e - sS) + ((e - sS) >> 5)]);
          if (i + s <= n) x = hadd(x, smem[(e + sS) + ((e + sS) >> 5)]);
          smem[e + (e >> 5)] = x;
        }
        __syncthreads();
      }
      for (int e = threadIdx.x; e < len; e += kThreads) g[e] = smem[e + (e >> 5)];
    } else if (!INV) {
      for (int e = threadIdx.x; e < len; e += kThreads) {
        const uint32_t slab = fdiv((uint32_t)e, fNS);
        const uint32_t p = (uint32_t)e - slab * (uint32_t)nS;
        const int i = (int)fdiv(p, fS) + 1;           // 1-based pole index
        const int s = i & -i;                          // 2^{tz(i)}
        const int sS = s * S;
        double x = sm[e];
        HIER_UPDATE(x, i - s >= 1, sm[e - sS], i + s <= n, sm[e + sS]);   // left, right
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
          if (i - s >= 1) x = hadd(x, sm[e - sS]);
          if (i + s <= n) x = hadd(x, sm[e + sS]);
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
    const int nb_log = T.l - t;                            // global blocks per pole
    // a tile holds NB = T.R consecutive blocks (power of two; 0 / 1: one) of one
    // pole: rows 0 .. NB 2^t, block boundaries (rb % 2^t == 0) read-only
    const int nbl = (T.R > 1) ? __ffs(T.R) - 1 : 0;
    const int NB = 1 << nbl;
    const int64_t o = q >> (T.rlog - nbl);
    const int b = (int)(T.blk0 + ((q & ((int64_t(1) << (T.rlog - nbl)) - 1)) << nbl));   // first block
    const int S = (int)T.S;
    const int n = (1 << T.l) - 1;
    const int i0 = b * B;                                  // pole index of local row 0
    const int rb_lo = (b == 0) ? 1 : 0;                    // row 0 of block 0 is the boundary
    const int rb_hi = (b + NB == (1 << nb_log)) ? NB * B - 1 : NB * B;  // row 2^l is the boundary
    const FDiv fS = T.fS;
    // global element of local e = rb*S + r is  gr[e]
    double *__restrict__ gr = T.grid + T.base + o * T.OS + (int64_t)(i0 - 1) * S;
    double *sm = smem + phase8(gr);
    const bool padded = INV && S < 32;                 // see k_flat_slabs: one pad double per 32
    if (padded) {
      const int e0 = rb_lo * S, e1 = (rb_hi + 1) * S;
      for (int e = e0 + threadIdx.x; e < e1; e += kThreads) cp_async8(smem + e + (e >> 5), gr + e);
    } else {
      copy_range_async(sm + rb_lo * S, gr + rb_lo * S, (rb_hi - rb_lo + 1) * S);
    }
    cp_async_wait_all();
    __syncthreads();
    // level s of every block of the tile: the rows s (2 jj + 1), jj < NB 2^t / (2 s)
    // (odd multiples of s < 2^t are never block boundaries)
    if (padded) {
      for (int s = B >> 1; s >= 1; s >>= 1) {              // block-local levels, coarse -> fine
        const int cnt = (NB * B / (2 * s)) * S;
        const int sS = s * S;
        for (int k = threadIdx.x; k < cnt; k += kThreads) {
          const int jj = (int)fdiv((uint32_t)k, fS);
          const int r = k - jj * S;
          const int rb = s * (2 * jj + 1);
          const int e = rb * S + r;
          const int i = i0 + rb;
          double x = smem[e + (e >> 5)];
          if (i - s >= 1) x = hadd(x, smem[(e - sS) + ((e - sS) >> 5)]);
          if (i + s <= n) x = hadd(x, smem[(e + sS) + ((e + sS) >> 5)]);
          smem[e + (e >> 5)] = x;
        }
        __syncthreads();
      }
      const int e1 = NB * B * S;
      for (int e = S + threadIdx.x; e < e1; e += kThreads)
        if (NB == 1 || (fdiv((uint32_t)e, fS) & (B - 1))) gr[e] = smem[e + (e >> 5)];
    } else if (!INV) {
      const int e1 = NB * B * S;
      for (int e = S + threadIdx.x; e < e1; e += kThreads) {
        const int rb = (int)fdiv((uint32_t)e, fS);
        if ((rb & (B - 1)) == 0) continue;                 // a block boundary (NB > 1)
        const int i = i0 + rb;
        const int s = rb & -rb;                            // tz(i) = tz(rb) < t
        const int sS = s * S;
        double x = sm[e];
        HIER_UPDATE(x, i - s >= 1, sm[e - sS], i + s <= n, sm[e + sS]);
        gr[e] = x;
      }
    } else {
      for (int s = B >> 1; s >= 1; s >>= 1) {              // block-local levels, coarse -> fine
        const int cnt = (NB * B / (2 * s)) * S;
        const int sS = s * S;
        for (int k = threadIdx.x; k < cnt; k += kThreads) {
          const int jj = (int)fdiv((uint32_t)k, fS);
          const int r = k - jj * S;
          const int rb = s * (2 * jj + 1);
          const int e = rb * S + r;
          const int i = i0 + rb;
          double x = sm[e];
          if (i - s >= 1) x = hadd(x, sm[e - sS]);
          if (i + s <= n) x = hadd(x, sm[e + sS]);
          sm[e] = x;
        }
        __syncthreads();
      }
      const int e1 = NB * B * S;
      for (int e = S + threadIdx.x; e < e1; e += kThreads)
        if (NB == 1 || (fdiv((uint32_t)e, fS) & (B - 1))) gr[e] = sm[e];
    }
    __syncthreads();
  });
}

// geometry of one FUSED tile
struct FusedTile {
  double *g;      // global address of local row 0 (W > 1: at column c0); with a
                  // blocked axis, local y = 0 of block 0 is virtual (never accessed)
  int units;      // W == 1 dense: units in this tile
  int wc;         // W > 1: valid columns
  int par;        // 8-byte phase of the SMEM data start
  int ylo, yhi;   // special axis: local rows that exist in the grid
  int zlo, zhi;   // second blocked axis: local rows that exist in the grid
  bool lo_ok, hi_ok;    // blocked axis: the block's end points are grid points
  bool lo2_ok, hi2_ok;  // second blocked axis: the same
};

template <int W>
__device__ __forceinline__ FusedTile fused_tile(const Task &T, int64_t q) {
  FusedTile f;
  f.ylo = 0;
  f.yhi = 0;
  f.lo_ok = f.hi_ok = true;
  if (T.bj < 0) {
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
  const bool blocked = T.bt < T.gl[T.bj];
  int64_t rest = q, c0 = 0;
  if (W > 1) {
    c0 = (q % T.ncb) * W;
    rest = q / T.ncb;
  }
  const int b = (int)(rest & ((int64_t(1) << T.nb_log) - 1));
  rest >>= T.nb_log;
  f.zlo = 0;
  f.zhi = 0;
  f.lo2_ok = f.hi2_ok = true;
  int64_t z0 = 0;
  if (T.bt2 >= 0) {                                // second blocked axis (bj + 1)
    const int64_t b2 = (rest & ((int64_t(1) << T.nb2_log) - 1)) + T.blk2_0;   // block range (sharded)
    rest >>= T.nb2_log;
    z0 = (b2 << T.bt2) - 1;
    f.lo2_ok = b2 > 0;
    f.hi2_ok = b2 < (int64_t(1) << (T.nb2_tot > 0 ? T.nb2_tot : T.nb2_log)) - 1;
    f.zlo = f.lo2_ok ? 0 : 1;
    f.zhi = f.hi2_ok ? (1 << T.bt2) : (1 << T.bt2) - 1;
  }
  int units = 1;
  if (W == 1 && T.R > 1) {                         // a coarse-lattice view: R consecutive outer units per tile
    const int64_t o0 = rest * T.R;
    units = (int)min((int64_t)T.R, T.O - o0);
    rest = o0;
  }
  int64_t ooff = rest * T.OS;
  if (T.O1 > 0) {                                  // two-level outer index
    const int64_t o2 = rest / T.O1;
    ooff = (rest - o2 * T.O1) * T.OS + o2 * T.OS2;
  }
  const int64_t y0 = blocked ? (int64_t(b) << T.bt) - 1 : 0;   // 0-based pole index of local y = 0
  f.g = T.grid + T.base + ooff + c0 + y0 * T.Gj + z0 * T.Gnext;
  f.units = units;
  f.wc = (W > 1) ? (int)min((int64_t)W, T.S - c0) : 1;
  f.lo_ok = !blocked || b > 0;
  f.hi_ok = !blocked || b < (1 << T.nb_log) - 1;
  f.ylo = f.lo_ok ? 0 : 1;
  f.yhi = f.hi_ok ? T.ej - 1 : T.ej - 2;
  f.par = T.aligned ? phase8(f.g) : 0;
  return f;
}

// W == 1 tile with a special axis: contiguous global runs (segments).  With a
// dense special axis (Gj == A) a segment is rows y0..y1 of one z; otherwise one
// row y of A elements.  Loads issue cp.async (16-byte pairs when the task's
// phases agree), stores write the fine rows only.
template <bool STORE>
__device__ __forceinline__ void fused_segments(const Task &T, const FusedTile &f, double *sm) {
  const int A = T.A, ej = T.ej;
  const bool blocked = T.bt < T.gl[T.bj];
  const int y0 = (STORE && blocked) ? 1 : f.ylo;
  const int y1 = (STORE && blocked) ? ej - 2 : f.yhi;
  const int ny = y1 - y0 + 1;
  // rows z of the axes after the special one: all of them, or the existing /
  // fine rows of a second blocked axis
  const int ez = T.P / (A * ej);                   // rows after the special axis per unit
  int z0 = 0, nz = ez * f.units;                    // units (lattice views, R > 1) stack along z
  if (T.bt2 >= 0) {
    z0 = STORE ? 1 : f.zlo;
    nz = (STORE ? nz - 2 : f.zhi) - z0 + 1;
  }
  const int64_t Gj = T.Gj, Gn = T.Gnext;         // registers: the cp.async "memory" clobbers
  const int64_t OSu = T.OS;
  const bool multi = f.units > 1;
  const bool aligned = T.aligned != 0;              // would otherwise reload Task fields per run
  double *const g0 = f.g;
  const int psy = T.sy, psz = T.sz;                 // padded layout (sy > 0)
  const bool dense_y = (Gj == (int64_t)A) && psy == 0;
  const int len = dense_y ? ny * A : A;
  const int nseg = dense_y ? nz : nz * ny;
  const int nyw = dense_y ? 1 : ny;                // segment s = z * nyw + (y - y0)
  auto seg_lo = [=](int z, int yy) {
    return psy > 0 ? (z0 + z) * psz + (y0 + yy) * psy : ((z0 + z) * ej + y0 + yy) * A;
  };
  auto seg_g = [=](int z, int yy) {
    const int zz = z0 + z;
    if (!multi) return g0 + (int64_t)(y0 + yy) * Gj + (int64_t)zz * Gn;
    const int u = zz / ez;                          // unit u of the tile at u OS
    return g0 + (int64_t)u * OSu + (int64_t)(y0 + yy) * Gj + (int64_t)(zz - u * ez) * Gn;
  };
  if (STORE && SGH_BULK_STORE && aligned && nseg <= 64 && len >= 64) {   // bulk stores by one thread
    bulk_fence_barrier();
    if (threadIdx.x == 0) {
      for (int z = 0; z < nseg / nyw; ++z)
        for (int yy = 0; yy < nyw; ++yy) bulk_store_range(seg_g(z, yy), sm + seg_lo(z, yy), len);
      bulk_commit();
    }
    return;
  }
  if (nseg < 16 && len >= 128) {                  // few long runs: the whole CTA on each
    for (int z = 0; z < nseg / nyw; ++z)
      for (int yy = 0; yy < nyw; ++yy) {
        const int lo = seg_lo(z, yy);
        double *gp = seg_g(z, yy);
        if (STORE) {
          for (int e = threadIdx.x; e < len; e += FT<1>::v) __stcg(gp + e, sm[lo + e]);
        } else if (aligned) {
          copy_range_async<FT<1>::v>(sm + lo, gp, len);
        } else {
          for (int e = threadIdx.x; e < len; e += FT<1>::v) cp_async8(sm + lo + e, gp + e);
        }
      }
    return;
  }
  // many runs: a group of L lanes per run (16-byte pairs + 8-byte head / tail),
  // runs walked as (z, yy) without divisions
  // L = lanes per run: enough for one 16-byte pair each (len/2 pairs at most);
  // stores and 8-byte copies then take 2 elements per lane
  const int half = len >> 1;
  const int logL = half > 16 ? 5 : half > 8 ? 4 : half > 4 ? 3 : half > 2 ? 2 : len > 1 ? 1 : 0;
  const int L = 1 << logL;
  const int lane = threadIdx.x & (L - 1);
  const ItemWalk walk(nyw, (int)threadIdx.x >> logL, FT<1>::v >> logL);
  if (!STORE && aligned && len > 1 && len <= 2 * L + 1) {   // straight-line: one 16-byte pair per lane
    const int c0 = 2 * lane;
    for (int z = walk.b0, yy = walk.p0; z < nz; walk.next(z, yy)) {
      double *sp = sm + seg_lo(z, yy);
      double *gp = seg_g(z, yy);
      const int par = phase8(gp);
      const int npairs = (len - par) >> 1;
      const int last = par + 2 * npairs;
      if (lane < npairs) cp_async16(sp + par + c0, gp + par + c0);
      if (lane == L - 1 && par) cp_async8(sp, gp);
      if (lane == L - 2 && last < len) cp_async8(sp + last, gp + last);
    }
    return;
  }
  for (int z = walk.b0, yy = walk.p0; z < nz; walk.next(z, yy)) {
    double *sp = sm + seg_lo(z, yy);
    double *gp = seg_g(z, yy);
    if (STORE) {
      for (int c = lane; c < len; c += L) __stcg(gp + c, sp[c]);
    } else if (aligned) {
      const int par = phase8(gp);
      const int npairs = (len - par) >> 1;
      const int last = par + 2 * npairs;
      for (int k = lane; k < npairs; k += L) cp_async16(sp + par + 2 * k, gp + par + 2 * k);
      if (lane == L - 1 && par) cp_async8(sp, gp);
      if (lane == L - 2 && last < len) cp_async8(sp + last, gp + last);
    } else {
      for (int c = lane; c < len; c += L) cp_async8(sp + c, gp + c);
    }
  }
}

// W > 1 tile with a special axis: row r_local = x + A (y + ej z) of W columns at
// global g + x S + y Gj + z Gnext; rows whose y lies outside the grid (load) or
// on the block ends (store) are skipped.
template <int W, bool STORE>
__device__ __forceinline__ void fused_rows_special(const Task &T, const FusedTile &f, double *sm) {
  constexpr int RS = W + 1;
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const bool blocked = T.bt < T.gl[T.bj];
  const int y0 = (STORE && blocked) ? 1 : f.ylo;
  const int y1 = (STORE && blocked) ? T.ej - 2 : f.yhi;
  const int P = T.P, A = T.A, ej = T.ej, wc = f.wc;
  const int64_t S = T.S, Gj = T.Gj, Gn = T.Gnext;
  const FDiv fA = T.fA, fE = T.fE;
  const bool aligned = T.aligned != 0;
  double *const g0 = f.g;
  auto row_ptr = [=](int r, double *&gr) -> bool {
    const uint32_t q = fdiv((uint32_t)r, fA);
    const int x = r - (int)q * A;
    const uint32_t z = fdiv(q, fE);
    const int y = (int)(q - z * (uint32_t)ej);
    gr = g0 + (int64_t)x * S + (int64_t)y * Gj + (int64_t)z * Gn;
    return y >= y0 && y <= y1;
  };
  if (STORE) {
    constexpr int RPI = (W >= 32) ? 1 : 32 / W;   // rows per warp instruction
    constexpr int CPL = (W >= 32) ? W / 32 : 1;   // columns per lane
    constexpr int STEP = RPI * (FT<W>::v / 32);
    const int c0 = (W >= 32) ? lane : lane % W;
    for (int r = warp * RPI + ((W >= 32) ? 0 : lane / W); r < P; r += STEP) {
      double *gr;
      if (!row_ptr(r, gr)) continue;
      const double *sr = sm + r * RS;
#pragma unroll
      for (int u = 0; u < CPL; ++u) {
        const int c = c0 + 32 * u;
        if (c < wc) __stcg(gr + c, sr[c]);
      }
    }
    return;
  }
  constexpr int NP = W / 2;                        // 16-byte slots per row
  constexpr int RPI = (NP >= 32) ? 1 : 32 / NP;
  constexpr int SPL = (NP >= 32) ? NP / 32 : 1;    // slots per lane
  constexpr int STEP = RPI * (FT<W>::v / 32);
  const int k0 = (NP >= 32) ? lane : lane % NP;
  for (int r = warp * RPI + ((NP >= 32) ? 0 : lane / NP); r < P; r += STEP) {
    double *gr;
    if (!row_ptr(r, gr)) continue;
    double *sr = sm + r * RS;
    if (aligned) {
      const int par = phase8(gr);
      const int npairs = (wc - par) >> 1;
      const int last = par + 2 * npairs;
#pragma unroll
      for (int u = 0; u < SPL; ++u) {
        const int k = k0 + 32 * u;
        const int c = par + 2 * k;
        if (k < npairs) cp_async16(sr + c, gr + c);
        if (k == NP - 1 && par) cp_async8(sr, gr);
        if (k == NP - 2 && last < wc) cp_async8(sr + last, gr + last);
      }
    } else {
#pragma unroll
      for (int u = 0; u < SPL; ++u) {
        const int c = 2 * (k0 + 32 * u);
        if (c < wc) cp_async8(sr + c, gr + c);
        if (c + 1 < wc) cp_async8(sr + c + 1, gr + c + 1);
      }
    }
  }
}

template <int W>
__device__ __forceinline__ void fused_issue(const Task &T, const FusedTile &f, double *stage) {
#ifdef SGH_DEBUG_NOMEMORY
  return;                                         // timing experiment: compute only
#endif
  if (T.bj >= 0) {
    if (W == 1) fused_segments<false>(T, f, stage + f.par);
    else fused_rows_special<(W == 1 ? 8 : W), false>(T, f, stage + f.par);
    return;
  }
  if (W == 1) copy_range_async<FT<1>::v>(stage + f.par, f.g, f.units * T.P);
  else if (W >= 64) fused_load_rows_wide<(W >= 64 ? W : 64)>(stage + f.par, f.g, T.S, f.par, T.P, f.wc);
  else fused_load_rows<(W == 1 || W >= 64 ? 8 : W)>(stage + f.par, f.g, T.S, f.par, T.P, f.wc);
}

// -DSGH_PIPE_TRACE (diagnostic build only): %globaltimer stamps of the first
// kTraceTiles tiles of every CTA of launches with >= g_ptrace_min tiles, read
// back with sgh_debug_pipe_trace().  Events per tile: 0 descriptor published,
// 1 producer starts issuing, 2 loads issued, 3 consumer starts waiting,
// 4 data ready, 5 computed, 6 stores issued, 7 stores have read the stage,
// 8 + j: axis j of the group transformed (j < 8); words 16..23 describe the
// tile (m, levels packed 8 bits each, bj, bt, bt2, P, units, W).
#ifdef SGH_PIPE_TRACE
constexpr int kTraceTiles = 64;
__device__ unsigned long long g_ptrace[160 * kTraceTiles * 24];
__device__ long long g_ptrace_min = 1ll << 62;
__device__ __forceinline__ unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#define PTRACE(k, ev) PTRACE_IF(trace_on, k, ev)
#define PTRACE_IF(on, k, ev)                                                                   \
  do {                                                                                         \
    if ((on) && (k) < kTraceTiles && blockIdx.x < 160)                                         \
      g_ptrace[((size_t)blockIdx.x * kTraceTiles + (k)) * 24 + (ev)] = gtime();                \
  } while (0)
#else
#define PTRACE(k, ev) \
  do {                \
  } while (0)
#define PTRACE_IF(on, k, ev) \
  do {                       \
  } while (0)
#endif

// all axes of the group on a staged tile (Alg. 1's axis loop, in SMEM)
template <bool INV, int W, int NT, class SY, class RM>
__device__ __forceinline__ void fused_compute_rm(const Task &T, const FusedTile &f, double *sm, const SY sy,
                                                 int trace_k, const RM rm);

template <bool INV, int W, int NT = FT<W>::v, class SY = CtaSync>
__device__ __forceinline__ void fused_compute(const Task &T, const FusedTile &f, double *sm, const SY sy = SY(),
                                              int trace_k = -1) {
  if (W == 1 && T.sy > 0) {                         // padded layout (lattice views)
    PadRemap rm;
    rm.fA = T.fA;
    rm.fE = T.fE;
    rm.A = T.A;
    rm.ej = T.ej;
    rm.sy = T.sy;
    rm.sz = T.sz;
    fused_compute_rm<INV, W, NT, SY, PadRemap>(T, f, sm, sy, trace_k, rm);
  } else {
    fused_compute_rm<INV, W, NT, SY, NoRemap>(T, f, sm, sy, trace_k, NoRemap());
  }
}

template <bool INV, int W, int NT, class SY, class RM>
__device__ __forceinline__ void fused_compute_rm(const Task &T, const FusedTile &f, double *sm, const SY sy,
                                                 int trace_k, const RM rm) {
  constexpr bool PAD = !std::is_same<RM, NoRemap>::value;
  constexpr int RS = (W == 1) ? 1 : W + 1;
  const int rows_total = f.units * T.P;
  const bool blocked = T.bj >= 0 && T.bt < T.gl[T.bj];
  HaloSkip hs;
  hs.on = false;
  hs.zs = false;
  if (blocked) {
    hs.fA = T.fA;
    hs.fE = T.fE;
    hs.ej = T.ej;
    hs.zs = INV && T.bt2 >= 0;
    hs.ez2 = (1 << (T.bt2 >= 0 ? T.bt2 : 0)) + 1;
  }
#ifdef SGH_DEBUG_NOCOMPUTE
  for (int j = 0; j < 0; ++j) {                     // timing experiment: load + store only
#else
  for (int j = 0; j < T.m; ++j) {                   // axes ascending
#endif
    const int l = T.gl[j];
    if (l <= 1 || ((T.skipmask >> j) & 1u)) continue;
    const int R = T.gR[j];
    const FDiv fR = T.fR[j];
    const bool full = (f.units == T.R);               // precomputed per-axis constants apply
    const FDiv fnp = T.fNP[j];
    // padded layout: the point stride of axis j (x axes: unchanged; the
    // special axis: sy; the axes after it: their z stride times sz)
    int str = 0;
    if (PAD) str = (j < T.bj) ? R : (j == T.bj) ? T.sy : (R / (T.A * T.ej)) * T.sz;
    if (blocked && j == T.bj) {
      // dehierarchization of a two-blocked tile: the second axis' end rows are final
      fused_axis_block<INV, W, NT, SY, RM>(sm, RS, T.bt, R, fR, full ? T.gOk[j] : rows_total / (T.ej * R), f.lo_ok,
                                           f.hi_ok, full ? &fnp : nullptr, INV && T.bt2 >= 0, sy, rm, str);
      if (sy.tid() == 0 && j < 8) PTRACE_IF(trace_k >= 0, trace_k, 8 + j);
      continue;
    }
    if (T.bt2 >= 0 && j == T.bj + 1) {              // second blocked axis
      fused_axis_block<INV, W, NT, SY, RM>(sm, RS, T.bt2, R, fR,
                                           full ? T.gOk[j] : rows_total / (((1 << T.bt2) + 1) * R), f.lo2_ok,
                                           f.hi2_ok, full ? &fnp : nullptr, false, sy, rm, str);
      if (sy.tid() == 0 && j < 8) PTRACE_IF(trace_k >= 0, trace_k, 8 + j);
      continue;
    }
    const int n = (T.bj == j) ? T.ej : (1 << l) - 1;
    hs.on = blocked && INV && j < T.bj;             // nodal block ends stay as loaded
#ifdef SGH_WARP_ROWS   // experiment (off): inlining it costs spills elsewhere in k_fused (C5 117 vs 130)
    if (W == 1 && !INV && R == 1 && !hs.on && warp_rows_dispatch(sm, rows_total / n, l)) {
      __syncthreads();                              // the next axis reads other rows
      continue;
    }
#endif
    const int Ok = full ? T.gOk[j] : rows_total / (n * R);
    if (R == 1 && !PAD) fused_axis<INV, W, true, NT, SY>(sm, RS, l, R, fR, Ok, hs, full ? &fnp : nullptr, sy);
    else fused_axis<INV, W, false, NT, SY, RM>(sm, RS, l, R, fR, Ok, hs, full ? &fnp : nullptr, sy, rm, str);
    if (sy.tid() == 0 && j < 8) PTRACE_IF(trace_k >= 0, trace_k, 8 + j);
  }
}

// all axes of the group on a staged tile, then the store
template <bool INV, int W>
__device__ __forceinline__ void fused_compute_store(const Task &T, const FusedTile &f, double *sm) {
  constexpr int RS = (W == 1) ? 1 : W + 1;
  const int P = T.P;
  const int units = f.units, wc = f.wc;
  const int64_t S = T.S;
  double *gbase = f.g;
  const int rows_total = units * P;
  fused_compute<INV, W>(T, f, sm);
#if defined(SGH_DEBUG_NOMEMORY) || defined(SGH_DEBUG_NOSTORE)
  return;                                         // timing experiments: compute only / no store
#endif
  if (T.bj >= 0) {
    if (W == 1) fused_segments<true>(T, f, sm);
    else fused_rows_special<(W == 1 ? 8 : W), true>(T, f, sm);
    return;
  }
  if (W == 1) {
    if (SGH_BULK_STORE) {
      bulk_fence_barrier();
      if (threadIdx.x == 0) {
        bulk_store_range(gbase, sm, rows_total);
        bulk_commit();
      }
    } else {
      for (int e = threadIdx.x; e < rows_total; e += FT<1>::v) __stcg(gbase + e, sm[e]);
    }
  } else {
    constexpr int RPI = (W >= 32) ? 1 : 32 / W;   // rows per warp instruction
    constexpr int CPL = (W >= 32) ? W / 32 : 1;   // columns per lane
    constexpr int STEP = RPI * (FT<W>::v / 32);
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
#define FUSED_MINB 3   // resident CTAs per SM the FUSED register budget is sized for (W > 1)
#endif
#ifndef FUSED_MINB_W1
#define FUSED_MINB_W1 3  // the same for the W == 1 kernels
#endif
#ifndef FUSED_MINB2
#define FUSED_MINB2 2  // the same for the two-stage (double-buffered) variant
#endif
// Tile assignment: cyclic (CTA c takes tiles c, c + grid, ...), which
// interleaves cheap and expensive tiles across CTAs.  The contiguous variant
// (-DSGH_FUSED_CONTIGUOUS: CTA c takes [c per, (c+1) per), so a task's
// descriptor is staged once per CTA) measured C5 95.9 vs 129.8 Gpoints/s: tile
// costs vary by task and contiguous ranges leave CTAs imbalanced.  The SMEM
// descriptor is re-staged only when the task changes.
template <bool INV, int W, int STAGES>
__global__ void __launch_bounds__(FT<W>::v, (STAGES == 1 ? (W == 1 ? FUSED_MINB_W1 : FUSED_MINB) : FUSED_MINB2)) k_fused(const __grid_constant__ Src src) {
  extern __shared__ __align__(16) double smem[];
  __shared__ Task s_task[2];                      // descriptors of the two in-flight tiles
#ifndef SGH_FUSED_CONTIGUOUS
  int64_t q = blockIdx.x;
  const int64_t qstep = gridDim.x, qend = src.total_tiles;
#else
  const int64_t per = (src.total_tiles + gridDim.x - 1) / gridDim.x;
  int64_t q = int64_t(blockIdx.x) * per;
  const int64_t qstep = 1, qend = min(src.total_tiles, q + per);
#endif
  if (q >= qend) return;
  int idx = -1, staged = -2;
  auto stage_task = [&](Task *dst, const Task *from) {
    const uint64_t *a = reinterpret_cast<const uint64_t *>(from);
    uint64_t *b = reinterpret_cast<uint64_t *>(dst);
    for (int i = threadIdx.x; i < (int)(sizeof(Task) / 8); i += FT<W>::v) b[i] = a[i];
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
  staged = idx;
  int slot = 0;                                   // s_task slot of the current tile (STAGES == 1)
  for (int k = 0;; ++k) {
    double *cur = smem + (STAGES == 2 ? (k & 1) * src.stage_doubles : 0);
    const int64_t qn = q + qstep;
    const bool more = qn < qend;
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
    // STAGES == 1: fetch the NEXT tile's task descriptor into the other slot
    // now (cp.async), so the next tile's geometry is read from SMEM instead of
    // a chain of global loads on the critical path (C5: every tile of a CTA is
    // a different task)
    int64_t qln = 0;
    bool newtask = false;
    if (STAGES == 1 && more) {
      Tn = ref(qn, qln);
      newtask = (idx != staged);
      if (newtask) {
        const uint64_t *a = reinterpret_cast<const uint64_t *>(Tn);
        uint64_t *b = reinterpret_cast<uint64_t *>(&s_task[slot ^ 1]);
        for (int i = threadIdx.x; i < (int)(sizeof(Task) / 8); i += FT<W>::v)
          cp_async8(reinterpret_cast<double *>(b + i), reinterpret_cast<const double *>(a + i));
        cp_async_commit();
      }
    }
    fused_compute_store<INV, W>(s_task[STAGES == 2 ? (k & 1) : slot], fc, cur + fc.par);
#ifndef SGH_DEBUG_NOSTOREWAIT   // timing experiment only (races: results wrong)
    if (W == 1 && SGH_BULK_STORE && threadIdx.x == 0) bulk_wait_read();   // bulk stores have read the stage
#endif
    if (STAGES == 1 && newtask) cp_async_wait<0>();
    __syncthreads();                              // the stage is free for the next load
    if (!more) break;
    q = qn;
    if (STAGES == 1) {                            // single stage: load the next tile now
      if (newtask) {
        slot ^= 1;
        staged = idx;
      }
      const Task &TS = s_task[slot];
      fn = fused_tile<W>(TS, qln);
      fused_issue<W>(TS, fn, smem);
      cp_async_commit();
    }
    Tc = Tn;
    fc = fn;
  }
  if (W == 1 && SGH_BULK_STORE && threadIdx.x == 0) bulk_wait_all();
}

// ============================================= PIPELINED FUSED W == 1 (k_fpipe)
// The same tiles as k_fused<W = 1> (whole poles of a run of axes, or a run
// with one / two BLOCKED axes; contiguous global runs), run by a
// warp-specialised persistent CTA, one per SM, over a ring of NS SMEM stages
// (and NS + 3 descriptor slots):
//   warp 1        descriptors: per tile, finds its task (prefix table) and
//                 copies the task descriptor and the tile geometry into a
//                 slot, up to NS + 3 tiles ahead (slot freed by the storer), so
//                 these dependent global loads never sit on the load path;
//   warp 0        producer: per tile, waits for its descriptor and a free
//                 stage and issues the tile's loads -- one cp.async.bulk (TMA
//                 bulk copy, SASS UBLKCP) per contiguous run into the 16-byte
//                 aligned body, completing on the stage's `full` mbarrier by
//                 transaction count, plus 8-byte cp.async for the odd end
//                 elements of runs at an 8-mod-16 phase
//                 (cp.async.mbarrier.arrive.noinc);
//   warps 2+G..   consumers (CFG::groups groups of CFG::cwarps warps, group g
//                 takes tiles g, g + G, ..): wait for `full`, run the group's
//                 axes in SMEM (fused_compute: the oracle's operation order,
//                 bitwise), fence the generic-proxy writes for the async proxy
//                 and arrive on `computed`;
//   warps 2..1+G  storers, one per consumer group (group g's tiles): wait for
//                 `computed`, issue the bulk stores of the
//                 tile's written runs (cp.async.bulk shared -> global) and its
//                 8-byte ends, waits until the copies have READ the stage and
//                 arrives on `empty` (and frees the descriptor slot).
// So the loads of tile k+1.. and the stores of tile k-1 stream while tile k is
// transformed: the engine keeps HBM busy, the SM's issue slots go to the
// transform.  Tasks whose SMEM phase does not follow the global one
// (`aligned == 0`, lattice views with 8-byte copies) stay on k_fused.
// The ring holds as many stages as fit the SM's shared memory (chosen per
// launch from the group's largest tile: 3 stages of the 8192-point tiles,
// more for smaller tiles), at most kPipeMaxStages.  (A ring of variable-size
// tiles, each taking only the space it needs -- up to 6 C5 tiles in flight
// instead of 3 -- measured slower: C5 155.9 vs 163, C4 270.8 vs 278.)
constexpr int kPipeMaxStages = 6;
#ifndef SGH_PIPE_MINW
#define SGH_PIPE_MINW 999
#endif
#ifndef SGH_PIPE_MINRUN
#define SGH_PIPE_MINRUN 128
#endif
constexpr int kPipeMinRun = SGH_PIPE_MINRUN;        // W == 1 tiles whose runs are shorter stay on k_fused
constexpr int kPipeMinW = SGH_PIPE_MINW;            // W > 1 column tiles this wide or wider run on k_fpipe

#ifndef SGH_WAIT_HINT_NS
#define SGH_WAIT_HINT_NS 20000
#endif
#ifndef SGH_WAIT_SLEEP_NS
#define SGH_WAIT_SLEEP_NS 0
#endif
constexpr int kPipeDescAhead = 3;                    // descriptor slots beyond the stages
constexpr int kPipeMaxDesc = kPipeMaxStages + kPipeDescAhead;
// Consumer configuration <groups, warps per group>: one task per launch (a
// single big grid, every tile alike: C4's two-blocked tiles) -> one group of 8
// warps (C4 281.7 vs 273.4 Gpoints/s with 2 x 6); a batched launch (every
// tile a different task, short barrier phases: C5) -> two groups of 6 warps
// that transform two tiles at once (C5 157.1 vs 147.9).
template <int G, int CW>
struct PipeCfg {
  static constexpr int groups = G;
  static constexpr int cwarps = CW;
  static constexpr int ct = 32 * CW;              // threads per consumer group
  static constexpr int roles = 2 + G;           // producer, descriptors, one storer per group
  static constexpr int threads = 32 * roles + G * 32 * CW;
};
#ifndef SGH_PIPE_BG
#define SGH_PIPE_BG 2
#endif
#ifndef SGH_PIPE_BW
#define SGH_PIPE_BW 6
#endif
#ifndef SGH_PIPE_SW
#define SGH_PIPE_SW 8
#endif
using PipeSingle = PipeCfg<1, SGH_PIPE_SW>;
using PipeBatched = PipeCfg<SGH_PIPE_BG, SGH_PIPE_BW>;

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mb_init(uint64_t *b, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(b)), "r"(count) : "memory");
}
// The waiting warp sleeps in hardware until the phase completes or the time
// hint (ns) runs out, instead of re-issuing try_wait (a spinning consumer
// takes issue slots from the other consumer group on its SM sub-partitions).
__device__ __forceinline__ void mb_wait(uint64_t *b, uint32_t parity) {
  uint32_t done;
#if SGH_WAIT_SLEEP_NS > 0
  int sleep_ns = 32;
#endif
  for (;;) {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(done)
        : "r"(smem_u32(b)), "r"(parity), "n"(SGH_WAIT_HINT_NS)
        : "memory");
    if (done) break;
#if SGH_WAIT_SLEEP_NS > 0
    __nanosleep(sleep_ns);                         // back off: fewer issue slots taken while waiting
    if (sleep_ns < SGH_WAIT_SLEEP_NS) sleep_ns *= 2;
#endif
  }
}
__device__ __forceinline__ void mb_arrive(uint64_t *b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mb_expect_tx(uint64_t *b, uint32_t bytes) {
  asm volatile("mbarrier.expect_tx.relaxed.cta.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
// one arrival, triggered when all of this thread's earlier cp.async copies have landed
__device__ __forceinline__ void mb_arrive_cpasync(uint64_t *b) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];\n" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void bulk_load(double *sdst, const double *gsrc, uint32_t bytes, uint64_t *bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
          smem_u32(sdst)),
      "l"(gsrc), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// Contiguous runs of a W == 1 tile, for the loads (every existing row) or the
// stores (the rows the tile writes; fused_segments).  Run i (i < count) covers
// SMEM [lo(i), lo(i) + len) of the stage and global [g(i), g(i) + len).
struct PipeRuns {
  double *g0;
  int64_t Gj, Gn;
  int A, ej, y0, z0, nyw, len, count, sy, sz, ez;
  int64_t OSu;
  __device__ __forceinline__ PipeRuns(const Task &T, const FusedTile &f, bool store) {
    sy = sz = 0;
    ez = 1;
    OSu = 0;
    if (T.bj < 0) {                                 // dense: one range of R units
      g0 = f.g;
      Gj = Gn = 0;
      A = ej = 1;
      y0 = z0 = 0;
      nyw = 1;
      len = f.units * T.P;
      count = 1;
      return;
    }
    const bool blocked = T.bt < T.gl[T.bj];
    A = T.A;
    ej = T.ej;
    y0 = (store && blocked) ? 1 : f.ylo;
    const int y1 = (store && blocked) ? ej - 2 : f.yhi;
    const int ny = y1 - y0 + 1;
    z0 = 0;
    ez = T.P / (A * ej);
    OSu = f.units > 1 ? T.OS : 0;                   // units (lattice views, R > 1) stack along z
    int nz = ez * f.units;
    if (T.bt2 >= 0) {
      z0 = store ? 1 : f.zlo;
      nz = (store ? nz - 2 : f.zhi) - z0 + 1;
    }
    Gj = T.Gj;
    Gn = T.Gnext;
    g0 = f.g;
    sy = T.sy;
    sz = T.sz;
    const bool dense_y = (Gj == (int64_t)A) && sy == 0;
    len = dense_y ? ny * A : A;
    nyw = dense_y ? 1 : ny;
    count = (ny > 0 && nz > 0) ? nz * nyw : 0;
  }
  __device__ __forceinline__ int lo(int i) const {
    const int z = i / nyw, yy = i - z * nyw;
    return sy > 0 ? (z0 + z) * sz + (y0 + yy) * sy : ((z0 + z) * ej + y0 + yy) * A;
  }
  __device__ __forceinline__ double *g(int i) const {
    const int z = i / nyw, yy = i - z * nyw;
    const int zz = z0 + z;
    if (OSu == 0) return g0 + (int64_t)(y0 + yy) * Gj + (int64_t)zz * Gn;
    const int u = zz / ez;
    return g0 + (int64_t)u * OSu + (int64_t)(y0 + yy) * Gj + (int64_t)(zz - u * ez) * Gn;
  }
};

// Runs of a W > 1 column tile: every tile row is one run of wc doubles
// (SMEM row r at r (W + 1), odd stride: its 8-byte phase follows the global
// row's, as in fused_load_rows).  Dense: rows r = 0..P-1 at g + r S.  With a
// special axis: row r = x + A (y + ej z) at g + x S + y Gj + z Gnext, loaded
// if y is a grid row, stored if y is a row the tile writes (fused_rows_special).
template <int W>
struct PipeRunsW {
  double *g0;
  int64_t S, Gj, Gn;
  int A, ej, y0, ny, len, count;
  FDiv fA;
  bool special;
  __device__ __forceinline__ PipeRunsW(const Task &T, const FusedTile &f, bool store) {
    g0 = f.g;
    S = T.S;
    len = f.wc;
    special = T.bj >= 0;
    if (!special) {
      count = T.P;
      A = 1;
      ej = 1;
      y0 = 0;
      ny = 1;
      Gj = Gn = 0;
      return;
    }
    const bool blocked = T.bt < T.gl[T.bj];
    A = T.A;
    ej = T.ej;
    fA = T.fA;
    Gj = T.Gj;
    Gn = T.Gnext;
    y0 = (store && blocked) ? 1 : f.ylo;
    const int y1 = (store && blocked) ? ej - 2 : f.yhi;
    ny = y1 - y0 + 1;
    const int nz = T.P / (A * ej);
    count = (ny > 0) ? A * ny * nz : 0;
  }
  // run i -> (x, y, z): x fastest, then the existing / written rows y, then z
  __device__ __forceinline__ void xyz(int i, int &x, int &y, int &z) const {
    const int q = (int)fdiv((uint32_t)i, fA);
    x = i - q * A;
    z = q / ny;
    y = y0 + (q - z * ny);
  }
  __device__ __forceinline__ int lo(int i) const {
    if (!special) return i * (W + 1);
    int x, y, z;
    xyz(i, x, y, z);
    return (x + A * (y + ej * z)) * (W + 1);
  }
  __device__ __forceinline__ double *g(int i) const {
    if (!special) return g0 + (int64_t)i * S;
    int x, y, z;
    xyz(i, x, y, z);
    return g0 + (int64_t)x * S + (int64_t)y * Gj + (int64_t)z * Gn;
  }
};

// Task owning tile q (the last t with prefix[t] <= q), searching forward from
// idx (prefix[idx] <= q) with the whole warp: 32 probes per round trip at
// stride 1, 32, 1024, .. (expanding while all probes are <= q, then refining).
// The prefix is non-decreasing, so the probes that are <= q form a prefix of
// the lanes.
__device__ __forceinline__ int warp_find_task(const Src &src, int idx, int64_t q, int lane) {
  int step = 1;
  bool expanding = true;
  for (;;) {
    const int64_t p = (int64_t)idx + 1 + (int64_t)lane * step;
    const bool le = p < src.ntasks && __ldg(&src.prefix[p]) <= q;
    const int cnt = __popc(__ballot_sync(0xffffffffu, le));
    if (cnt == 32 && expanding) {                 // the answer is further on
      idx += 1 + 31 * step;                       // the last probe, <= q
      if (step < (1 << 20)) step *= 32;
      continue;
    }
    if (cnt > 0) idx += 1 + (cnt - 1) * step;     // the last probe <= q
    if (step == 1) return idx;                    // the next position is > q (or the end)
    expanding = false;
    step /= 32;                                   // the answer lies in (idx, idx + 32 step)
  }
}

template <bool INV, class CFG, int W>
__global__ void __launch_bounds__(CFG::threads, 1) k_fpipe(const __grid_constant__ Src src) {
  using Runs = typename std::conditional<W == 1, PipeRuns, PipeRunsW<W>>::type;
  extern __shared__ __align__(128) double pipe_smem[];
  // `computed` is a ring per consumer group (its j-th tile: slot j % NS), so
  // each storer waits for the phases of its barriers strictly in order (two
  // storers on one barrier could wait for a phase two ahead of the current
  // one, which the parity test cannot tell from the previous one)
  // `full` and `computed` are rings per consumer group, indexed by the group's
  // own tile count j (slot j % NS): each barrier's phases then belong to ONE
  // group's tiles, which that group (and its storer) waits for strictly in
  // order.  (With the stage's barrier shared by the groups, group A could
  // wait for its tile k while the stage's previous tile k - NS -- the other
  // group's, whose copies may still be landing -- had not completed its
  // phase: the parity test reads that incomplete phase as done.)
  __shared__ __align__(8) uint64_t bar_full[CFG::groups][kPipeMaxStages], bar_computed[CFG::groups][kPipeMaxStages],
      bar_empty[kPipeMaxStages], bar_dfull[kPipeMaxDesc], bar_dfree[kPipeMaxDesc];
  __shared__ __align__(16) Task s_task[kPipeMaxDesc];   // descriptor slot of tile k: k % ND
  __shared__ FusedTile s_tile[kPipeMaxDesc];
  const int NS = src.nstages;                     // stage of tile k: k % NS
  const int ND = NS + kPipeDescAhead;             // descriptor slots
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < NS; ++s) {
      for (int g = 0; g < CFG::groups; ++g) mb_init(&bar_full[g][s], 32);   // one (cp.async) arrival per producer lane
      for (int g = 0; g < CFG::groups; ++g) mb_init(&bar_computed[g][s], 1);   // the group's leader
      mb_init(&bar_empty[s], 1);                    // the storer's lane 0
    }
    for (int s = 0; s < ND; ++s) {
      mb_init(&bar_dfull[s], 32);                   // every lane of the descriptor warp
      mb_init(&bar_dfree[s], 1);                    // the storer's lane 0 (the slot's last reader)
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  const int64_t total = src.total_tiles;
  const int64_t q0 = blockIdx.x, qstep = gridDim.x;
  const int sd = src.stage_doubles;
#ifdef SGH_PIPE_TRACE
  const bool trace_on = total >= g_ptrace_min;
#endif
  if (warp == 1) {
    // ---------------------------------------------------------- descriptors
    // Looks up the task of each tile (a chain of dependent global loads: the
    // tile's task in the prefix table, then its descriptor) and publishes the
    // descriptor and the tile geometry in a slot, up to ND tiles ahead of the
    // storer, so the producer never waits for those loads.
    constexpr int kTW = (int)(sizeof(Task) / 8);
    static_assert(kTW <= 96, "Task descriptor must fit 3 words per lane");
    int idx = 0;
    int64_t q = q0;
    for (int k = 0; q < total; ++k, q += qstep) {
      const int ds = k % ND;
      const int rr = k / ND;
      int64_t ql;
      const uint64_t *a;
      if (src.tasks) {
        idx = warp_find_task(src, idx, q, lane);
        ql = q - __ldg(&src.prefix[idx]);
        a = reinterpret_cast<const uint64_t *>(&src.tasks[idx]);
      } else {
        ql = q;
        a = reinterpret_cast<const uint64_t *>(&src.single);
      }
      uint64_t dreg[3];
#pragma unroll
      for (int u = 0; u < 3; ++u) dreg[u] = (lane + 32 * u < kTW) ? a[lane + 32 * u] : 0;
      if (rr > 0) mb_wait(&bar_dfree[ds], (rr - 1) & 1);
      uint64_t *b = reinterpret_cast<uint64_t *>(&s_task[ds]);
#pragma unroll
      for (int u = 0; u < 3; ++u)
        if (lane + 32 * u < kTW) b[lane + 32 * u] = dreg[u];
      __syncwarp();
      const FusedTile f = fused_tile<W>(s_task[ds], ql);
      if (lane == 0) s_tile[ds] = f;
      __syncwarp();
      if (lane == 0) PTRACE(k, 0);
#ifdef SGH_PIPE_TRACE
      if (lane == 0 && trace_on && k < kTraceTiles && blockIdx.x < 160) {
        unsigned long long *w = &g_ptrace[((size_t)blockIdx.x * kTraceTiles + k) * 24 + 16];
        const Task &TT = s_task[ds];
        unsigned long long lv = 0;
        for (int j = 0; j < TT.m && j < 8; ++j) lv |= (unsigned long long)(uint8_t)TT.gl[j] << (8 * j);
        w[0] = TT.m; w[1] = lv; w[2] = (unsigned long long)(long long)TT.bj; w[3] = (unsigned long long)(long long)TT.bt;
        w[4] = (unsigned long long)(long long)TT.bt2; w[5] = TT.P; w[6] = f.units; w[7] = TT.skipmask;
      }
#endif
      mb_arrive(&bar_dfull[ds]);
    }
  } else if (warp == 0) {
    // ------------------------------------------------------------ producer
    int64_t q = q0;
    for (int k = 0; q < total; ++k, q += qstep) {
      const int s = k % NS;
      const int r = k / NS;
      const int ds = k % ND;
      mb_wait(&bar_dfull[ds], (k / ND) & 1);
      uint64_t *const fb = &bar_full[k % CFG::groups][(k / CFG::groups) % NS];   // the consuming group's ring
      const Task &T = s_task[ds];
      const FusedTile f = s_tile[ds];
      double *const sbase = pipe_smem + (size_t)s * sd;   // stage start; tile data from f.par
      const Runs runs(T, f, false);
      // one bulk copy (copy engine) per run; bytes first: expect_tx before the copies
      uint32_t tx = 0;
      for (int i = lane; i < runs.count; i += 32) tx += (uint32_t)((runs.len - phase8(runs.g(i))) >> 1) * 16u;
      if (r > 0) mb_wait(&bar_empty[s], (r - 1) & 1);
      // only now is the stage's previous tile consumed, i.e. the previous phase
      // of this `full` barrier complete: the expected bytes count for THIS tile
      if (tx) mb_expect_tx(fb, tx);
      if (lane == 0) PTRACE(k, 1);
      for (int i = lane; i < runs.count; i += 32) {
        double *sp = sbase + f.par + runs.lo(i);
        const double *gp = runs.g(i);
        const int len = runs.len;
        const int head = phase8(gp);
        const int pairs = (len - head) >> 1;
        const int last = head + 2 * pairs;
        if (head) cp_async8(sp, gp);
        if (last < len) cp_async8(sp + last, gp + last);
        if (pairs > 0) bulk_load(sp + head, gp + head, (uint32_t)pairs * 16u, fb);
      }
      mb_arrive_cpasync(fb);
      if (lane == 0) PTRACE(k, 2);
    }
    cp_async_wait<0>();                            // no cp.async outstanding when the warp exits
  } else if (warp < CFG::roles) {
    // ------------------------------------------------------------- storers
    // storer g stores the tiles of consumer group g (k = g, g + G, ..), so a
    // group's finished tile never waits behind the other group's
    const int g = warp - 2;
    int64_t q = q0 + (int64_t)g * qstep;
    for (int k = g; q < total; k += CFG::groups, q += CFG::groups * qstep) {
      const int s = k % NS;
      const int ds = k % ND;
      const int j = k / CFG::groups;                // the group's j-th tile
      mb_wait(&bar_computed[g][j % NS], (j / NS) & 1);
      const Task &T = s_task[ds];
      const FusedTile f = s_tile[ds];
      const double *const sbase = pipe_smem + (size_t)s * sd;
      const Runs runs(T, f, true);
      for (int i = lane; i < runs.count; i += 32) {
        const double *sp = sbase + f.par + runs.lo(i);
        double *gp = runs.g(i);
        const int len = runs.len;
        const int head = phase8(gp);
        const int pairs = (len - head) >> 1;
        const int last = head + 2 * pairs;
        if (head) __stcg(gp, sp[0]);
        if (last < len) __stcg(gp + last, sp[last]);
        if (pairs > 0)
          asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;\n" ::"l"(gp + head),
                       "r"(smem_u32(sp + head)), "r"(pairs * 16)
                       : "memory");
      }
      bulk_commit();
      if (lane == 0) PTRACE(k, 6);
      bulk_wait_read();                             // this lane's copies have read the stage
      __syncwarp();
      if (lane == 0) mb_arrive(&bar_empty[s]);
      if (lane == 0) {
        PTRACE(k, 7);
        mb_arrive(&bar_dfree[ds]);
      }
    }
    bulk_wait_all();
  } else {
    // ----------------------------------------------------------- consumers
    constexpr int kPipeCT = CFG::ct;
    constexpr int kPipeGroups = CFG::groups;
    const int g = (warp - CFG::roles) / CFG::cwarps;
    const GroupSync<kPipeCT> sy{(int)threadIdx.x - 32 * CFG::roles - g * kPipeCT, 1 + g};
    int64_t q = q0 + (int64_t)g * qstep;
    for (int k = g; q < total; k += kPipeGroups, q += kPipeGroups * qstep) {
      const int s = k % NS;
      if (sy.tid() == 0) PTRACE(k, 3);
      const int jg = k / kPipeGroups;                // the group's jg-th tile
      mb_wait(&bar_full[g][jg % NS], (jg / NS) & 1);
      if (sy.tid() == 0) PTRACE(k, 4);
      const Task &T = s_task[k % ND];
      const FusedTile f = s_tile[k % ND];
#ifdef SGH_PIPE_TRACE
      const int tk = trace_on ? k : -1;
#else
      const int tk = -1;
#endif
      fused_compute<INV, W, kPipeCT, GroupSync<kPipeCT>>(T, f, pipe_smem + (size_t)s * sd + f.par, sy, tk);
      asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");   // SMEM results -> the bulk stores
      sy.bar();
      if (sy.tid() == 0) {
        PTRACE(k, 5);
        mb_arrive(&bar_computed[g][(k / CFG::groups) % NS]);
      }
    }
  }
}

// W == 1 FUSED tasks the pipelined kernel runs: dense ranges, or runs whose
// SMEM 8-byte phase follows the global one (bulk copies need equal 16-byte phases)
// (runs shorter than kPipeMinRun doubles -- e.g. C3's 33-point blocks of the
// contiguous axis, 225 runs per tile -- make the copy engine slow: one bulk
// copy per short run measured 0.26 of the copy peak on C3 vs 0.49 on k_fused's
// LDGSTS from all threads; W > 1 column tiles, one run per 128-1024 B row,
// likewise: C5 146 vs 167.  Loading short runs with 16-byte cp.async from the
// producer warp instead was slower still (C3 0.11, C5 101-145): one warp
// cannot issue a tile's worth of small copies in time.  Both stay on k_fused.)
bool pipe_task(const Task &t, bool batched) {
  if (t.kind != KIND_FUSED || (t.bj >= 0 && !t.aligned)) return false;
  // padded lattice views: on k_fpipe in single-grid calls (C2: 130 vs 125
  // Gpoints/s -- and the blocked tiles launched before them ran at 0.70 vs
  // 0.62 of the peak when the next kernel was k_fpipe rather than k_fused),
  // on k_fused in grouped launches over several grids (C5: 175.0 vs 165.8)
  static const bool pad_pipe = tuning_env("SGH_PAD_PIPE") != nullptr;   // experiment
  static const int pad_pipe_min_p =
      tuning_env("SGH_PAD_PIPE_MIN_P") ? atoi(tuning_env("SGH_PAD_PIPE_MIN_P")) : (1 << 30);   // experiment
  if (t.sy > 0 && batched && !pad_pipe && t.P < pad_pipe_min_p) return false;
  if (t.W > 1) return t.W >= kPipeMinW;
  if (t.bj < 0) return true;                      // dense: one range per tile
  const int64_t run = (t.Gj == t.A) ? int64_t(t.A) * t.ej : t.A;
  return run >= kPipeMinRun;
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
          HIER_UPDATE(x, i - s >= 1, v[c][i - s - 1], i + s <= n, v[c][i + s - 1]);
          p[c][(i - 1) * PS] = x;
        }
      } else {
#pragma unroll
        for (int lam = 2; lam <= L; ++lam) {
          const int s = 1 << (L - lam);
#pragma unroll
          for (int i = s; i <= n; i += 2 * s) {
            double x = v[c][i - 1];
            if (i - s >= 1) x = hadd(x, v[c][i - s - 1]);
            if (i + s <= n) x = hadd(x, v[c][i + s - 1]);
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
constexpr int kProfKindPipe = 7;                 // sgh_launch_record.kind of k_fpipe launches

// the k_fpipe instance for a tile width
template <class CFG>
static KernelFn fpipe_for(int w, bool inv) {
  switch (w) {
    case 1: return inv ? k_fpipe<true, CFG, 1> : k_fpipe<false, CFG, 1>;
    case 8: return inv ? k_fpipe<true, CFG, 8> : k_fpipe<false, CFG, 8>;
    case 16: return inv ? k_fpipe<true, CFG, 16> : k_fpipe<false, CFG, 16>;
    case 32: return inv ? k_fpipe<true, CFG, 32> : k_fpipe<false, CFG, 32>;
    case 64: return inv ? k_fpipe<true, CFG, 64> : k_fpipe<false, CFG, 64>;
    case 128: return inv ? k_fpipe<true, CFG, 128> : k_fpipe<false, CFG, 128>;
    default: return nullptr;
  }
}

// FUSED pipeline depth: 1 (default) or 2 stages (tuning override SGH_FUSED_STAGES)
int fused_stages() {
  static int st = -1;
  if (st < 0) {
    const char *e = tuning_env("SGH_FUSED_STAGES");
    st = (e && atoi(e) == 2) ? 2 : 1;
  }
  return st;
}

static KernelFn kernel_for(int kind, int l, int w, bool inv, int stages = -1) {
  if (stages < 0) stages = fused_stages();
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
      if (stages == 2) {
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
    case KIND_FLAT_SLABS: {                       // +1 phase shift, + 1 pad per 32 (INV, S < 32)
      const size_t e = size_t(t.R) * size_t(n * t.S);
      return (e + e / 32 + 2) * 8;
    }
    case KIND_FLAT_BLOCKS: {
      const size_t e = size_t((int64_t(std::max(1, t.R)) << t.t) + 1) * size_t(t.S);
      return (e + e / 32 + 2) * 8;
    }
    case KIND_STRIDED: return size_t((int64_t(1) << t.t) + 1) * size_t(t.W + 2) * 8;
    case KIND_FUSED:
      if (t.W == 1 && t.sy > 0) return (size_t(t.R) * size_t(t.P / (t.A * t.ej)) * size_t(t.sz) + 2) * 8;   // padded
      return t.W == 1 ? (size_t(t.R) * size_t(t.P) + 2) * 8 : (size_t(t.P) * size_t(t.W + 1) + 2) * 8;
    default: return 0;
  }
}

// resident CTAs on the whole device for a kernel instance and smem size (cached)
static int resident_ctas(KernelFn fn, size_t smem, int threads = kThreads) {
  int dev = 0;
  cudaGetDevice(&dev);
  struct Entry { KernelFn fn; int dev; size_t smem; int ctas; };
  static Entry cache[256];
  static int ncache = 0;
  static std::mutex mu;                           // calls may come from several host threads
  std::lock_guard<std::mutex> lk(mu);
  for (int i = 0; i < ncache; ++i)
    if (cache[i].fn == fn && cache[i].dev == dev && cache[i].smem == smem) return cache[i].ctas;
  // Opt in to large dynamic shared memory (FUSED / STRIDED tiles up to ~70 KB):
  // the default limit of 48 KB covers static + dynamic shared memory, so the
  // opt-in is needed as soon as both together exceed it; the opt-in maximum is
  // the device's per-block limit minus the kernel's static shared memory.
  cudaFuncAttributes fa;
  size_t stat = 0;
  if (cudaFuncGetAttributes(&fa, fn) == cudaSuccess) stat = fa.sharedSizeBytes;
  if (smem + stat > 48 * 1024) {
    int optin = 0;
    cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(optin - (int)stat));
  }
  int ctas = 1;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&ctas, fn, threads, smem) != cudaSuccess || ctas < 1) ctas = 1;
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int total = ctas * sms;
  if (ncache < 256) cache[ncache++] = Entry{fn, dev, smem, total};
  return total;
}

// stages of k_fpipe's ring for a stage size: all that fit the per-block
// shared memory next to the kernel's static part, 2 .. kPipeMaxStages
static int pipe_stages(KernelFn fn, size_t stage_bytes) {
  int dev = 0, optin = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  cudaFuncAttributes fa;
  size_t stat = 0;
  if (cudaFuncGetAttributes(&fa, fn) == cudaSuccess) stat = fa.sharedSizeBytes;
  const size_t avail = size_t(optin) > stat + 1024 ? size_t(optin) - stat - 1024 : 0;
  const int n = stage_bytes ? int(avail / stage_bytes) : kPipeMaxStages;
  return std::max(2, std::min(kPipeMaxStages, n));
}

// Launch one task (single grid).  Returns the CUDA error of the launch.
cudaError_t launch_single(const Task &task, bool inv, cudaStream_t stream) {
  const bool pipe = pipe_task(task, false);
  KernelFn fn = pipe ? fpipe_for<PipeSingle>(task.W, inv) : kernel_for(task.kind, task.l, task.W, inv);
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
    if (pipe) src.nstages = pipe_stages(fn, size_t(src.stage_doubles) * 8);
    smem = size_t(pipe ? src.nstages : fused_stages()) * src.stage_doubles * 8;
  }
  const int nt = pipe ? PipeSingle::threads : task.kind == KIND_FUSED ? (task.W == 1 ? FT<1>::v : FT<8>::v) : kThreads;
  const int64_t cap = resident_ctas(fn, smem, nt);
  const int64_t grid = task.tiles < cap ? task.tiles : cap;
  if (grid <= 0) return cudaSuccess;
  ProfToken tok = prof_begin(stream);
  fn<<<(unsigned)grid, nt, smem, stream>>>(src);
  cudaError_t e = cudaGetLastError();
  prof_end(tok, pipe ? kProfKindPipe : task.kind, task.kind == KIND_FUSED || task.kind == KIND_STRIDED ? task.W : task.l,
           inv, 16.0 * task_points(task), stream, task_variant(task));
  return e;
}

// Launch a group of tasks of one kernel instance from a device task table;
// smem = max task_smem over the group.
cudaError_t launch_table(int kind, int l, int w, bool inv, const Task *d_tasks, const int64_t *d_prefix,
                         int32_t ntasks, int64_t total_tiles, size_t smem, double points, cudaStream_t stream,
                         int variant, bool pipe) {
  // experiment: groups of small W == 1 tiles on the double-buffered k_fused
  static const size_t small2 = tuning_env("SGH_SMALL_STAGES2") ? (size_t)atol(tuning_env("SGH_SMALL_STAGES2")) : 0;
  const int stages = (kind == KIND_FUSED && !pipe && w == 1 && smem <= small2) ? 2 : fused_stages();
  KernelFn fn = pipe ? fpipe_for<PipeBatched>(w, inv) : kernel_for(kind, l, w, inv, stages);
  if (!fn) return cudaErrorInvalidValue;
  Src src{};
  src.tasks = d_tasks;
  src.prefix = d_prefix;
  src.ntasks = ntasks;
  src.total_tiles = total_tiles;
  if (kind == KIND_FUSED) {
    src.stage_doubles = (int32_t)((smem + 15) / 16 * 2);
    if (pipe) src.nstages = pipe_stages(fn, size_t(src.stage_doubles) * 8);
    smem = size_t(pipe ? src.nstages : stages) * src.stage_doubles * 8;
  }
  const int nt = pipe ? PipeBatched::threads : kind == KIND_FUSED ? (w == 1 ? FT<1>::v : FT<8>::v) : kThreads;
  const int64_t cap = resident_ctas(fn, smem, nt);
  const int64_t grid = total_tiles < cap ? total_tiles : cap;
  if (grid <= 0) return cudaSuccess;
  ProfToken tok = prof_begin(stream);
  fn<<<(unsigned)grid, nt, smem, stream>>>(src);
  cudaError_t e = cudaGetLastError();
  prof_end(tok, pipe ? kProfKindPipe : kind, kind == KIND_FUSED || kind == KIND_STRIDED ? w : l, inv, 16.0 * points,
           stream, variant);
  return e;
}

}  // namespace sgh

#ifdef SGH_PIPE_TRACE
// diagnostic build only: out == NULL -> arm tracing for launches with >= min_tiles
// tiles; else copy the trace (160 CTAs x kTraceTiles x 24 words) out.
extern "C" int64_t sgh_debug_pipe_trace(int64_t min_tiles, unsigned long long *out, int64_t cap) {
  const int64_t n = 160 * sgh::kTraceTiles * 24;
  if (!out) {
    long long m = min_tiles;
    cudaMemcpyToSymbol(sgh::g_ptrace_min, &m, sizeof m);
    return n;
  }
  cudaDeviceSynchronize();
  cudaMemcpyFromSymbol(out, sgh::g_ptrace, sizeof(unsigned long long) * (size_t)std::min(n, cap));
  return n;
}
#endif
