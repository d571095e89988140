// sgh_combi.cu -- the communication phase of the combination technique that the
// hierarchization exists for ("the combination technique
// ... linear combination of the solutions on the anisotropic full grids",
// P:77 "all combination grids are hierarchized in parallel ... communication",
// P:86-88 hierarchical surpluses of nested grids).
//
// The sparse grid of level sum n is the set of hierarchical subspaces W_lam,
// lam_k >= 1, |lam|_1 <= n.  A combination grid l holds exactly the subspaces
// lam <= l; its point i (1-based per axis) is the point j of W_lam with
// lam_k = l_k - tz(i_k), j_k = i_k >> (tz(i_k) + 1)  (predecessor rule).
//
// SG LAYOUT (include/sgh.h): subspaces by level sum s ascending, then
// lexicographically ascending in (lam_1..lam_d); inside W_lam the
// 2^{lam_k - 1} points per axis row-major with j_1 fastest.  All subspaces of
// level sum s have 2^{s-d} points, so
//   offset(lam) = sum_{s'<s} C(s'-1, d-1) 2^{s'-d} + rank_s(lam) 2^{s-d},
//   rank_s(lam) = sum_k [ C(rem_k - 1, d-k-1) - C(rem_k - lam_k, d-k-1) ],
// rem_k = s - lam_1 - .. - lam_{k-1} (the compositions of rem_k into d - k parts
// whose first part is < lam_k, by the hockey-stick identity).
//
// gather:  sparse(lam, j) = sum over the grids g holding W_lam, in the given
//          grid order, of coeff_g * alpha_g(point) -- a PULL per sparse point,
//          accumulated sequentially from +0.0 with explicit __dmul_rn /
//          __dadd_rn (no FMA), so the result is bitwise the oracle's
//          "for g in order: sparse += coeff_g * alpha_g".
// scatter: every grid point gets its sparse value (data movement only).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>
#include <map>
#include <mutex>
#include <vector>

#include "../../include/sgh.h"
#include "sgh_common.cuh"
#include "sgh_plan.hpp"

namespace sgh {

constexpr int kCombiMaxN = 62;     // level sums up to 62 (binomial table rows)
constexpr int kCombiPts = 1024;    // points per work item

__constant__ int64_t c_binom[kCombiMaxN + 2][SGH_MAX_D + 1];

struct CombiGrid {
  double *grid;
  double coeff;
  int64_t N;
  int8_t l[SGH_MAX_D];
  FDiv fn[SGH_MAX_D];              // division by n_k = 2^{l_k} - 1 (scatter: unflatten)
  int32_t str[SGH_MAX_D];          // row strides prod_{m<k} n_m (gather; N < 2^31)
};

// gather work unit: a FAMILY = all subspaces (lam_1, lam') with the same tail
// lam' = (lam_2..lam_d), lam_1 = 1..L, L = n - |lam'|.  In every grid holding
// them, the points of one tail index j' lie in ONE x_1 row, the point of W_lam
// with index j_1 at i_1 = (2 j_1 + 1) 2^{l_1 - lam_1}, i.e. at position
// I = (2 j_1 + 1) 2^{L - lam_1} of the family's finest row.  A tile holds all
// lam_1 of 2^mlog rows (L <= kFamB) or of the positions [c 2^kFamB,
// (c+1) 2^kFamB) of one row (L > kFamB), so every grid sector a tile reads is
// used by the tile's own warps while it is in L1, instead of by subspaces
// processed far apart (one pull per subspace read 6x the grid bytes on C5).
constexpr int kFamB = 14;
struct CombiFam {
  int32_t sub0;                    // fam_subs[sub0 + lam_1 - 1] = index of subspace (lam_1, lam')
  int32_t L;                       // largest lam_1
  int32_t rlog;                    // log2 of the tail index count (rows)
  int32_t mlog;                    // L <= kFamB: log2 rows per tile
  int32_t thr;                     // family tiles do lam_1 = thr..L (>= 32 points per tile each); the
                                   // coarser subspaces go to per-subspace tiles (k_gather_sub)
  int8_t lam[SGH_MAX_D];           // lam[1..d-1] = lam'
};

struct CombiSub {                  // one subspace W_lam of the sparse grid
  int64_t off;                     // its sparse offset (SG layout)
  int64_t c0;                      // its contributing grids: contrib[c0 .. c0+nc)   (built on the device)
  int32_t nc;
  int32_t npts;                    // 2^{|lam|-d}
  int8_t lam[SGH_MAX_D];
};

struct CombiArgs {
  const CombiGrid *grids;
  CombiSub *subs;
  const CombiFam *fams;            // gather: families (items), their subspace lists
  const int32_t *fam_subs;
  int32_t nsubs;
  int32_t *contrib;                // grid indices, grouped per subspace, in grid order
  const int64_t *prefix;           // tile prefix over families (gather) or grids (scatter), items + 1 entries
  int32_t items;                   // families (gather) or grids (scatter)
  int32_t num_grids;
  int64_t tiles;
  const int32_t *csubs;            // gather: the coarse subspaces (per-subspace tiles of kCombiPts points)
  const int64_t *cprefix;          //   and their tile prefix (ncsubs + 1 entries)
  int32_t ncsubs;
  int64_t ctiles;
  int64_t sbase[kCombiMaxN + 2];   // offset of the first subspace of level sum s
  double *sparse;
  int32_t d, n;
};

// binom / sbase: the tables staged in SMEM (lanes index them with different
// values; constant-bank reads would serialise)
template <int D>
__device__ __forceinline__ int64_t sg_offset(const int *lam, const int64_t (*binom)[SGH_MAX_D + 1],
                                             const int64_t *sbase) {
  int s = 0;
#pragma unroll
  for (int k = 0; k < D; ++k) s += lam[k];
  int64_t rank = 0;
  int rem = s;
#pragma unroll
  for (int k = 0; k < D - 1; ++k) {
    const int m = D - k - 1;
    rank += binom[rem - 1][m] - binom[rem - lam[k]][m];
    rem -= lam[k];
  }
  return sbase[s] + (rank << (s - D));
}

// owner item of tile q (tiles of a CTA increase): galloping search from the cursor
__device__ __forceinline__ int combi_item_in(const int64_t *prefix, int items, int idx, int64_t q) {
  if (idx < 0) {
    int lo = 0, hi = items - 1;
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (__ldg(&prefix[mid]) <= q) lo = mid; else hi = mid - 1;
    }
    return lo;
  }
  if (idx + 1 >= items || __ldg(&prefix[idx + 1]) > q) return idx;
  int lo = idx + 1, step = 1, hi = lo + 1;
  while (hi < items && __ldg(&prefix[hi]) <= q) {
    lo = hi;
    step <<= 1;
    hi = lo + step;
  }
  if (hi > items) hi = items;
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if (__ldg(&prefix[mid]) <= q) lo = mid; else hi = mid;
  }
  return lo;
}
__device__ __forceinline__ int combi_item(const CombiArgs &A, int idx, int64_t q) {
  return combi_item_in(A.prefix, A.items, idx, q);
}

// one warp per subspace: count (fill = false) or list (fill = true) the grids
// holding it, in grid order (ballot + popc keeps the order)
template <bool FILL>
__global__ void __launch_bounds__(kThreads) k_contrib(const __grid_constant__ CombiArgs A) {
  const int lane = threadIdx.x & 31;
  for (int sidx = (blockIdx.x * kThreads + threadIdx.x) >> 5; sidx < A.nsubs;
       sidx += (gridDim.x * kThreads) >> 5) {
    CombiSub &S = A.subs[sidx];
    int64_t at = FILL ? S.c0 : 0;
    int cnt = 0;
    for (int g0 = 0; g0 < A.num_grids; g0 += 32) {
      const int g = g0 + lane;
      bool holds = g < A.num_grids;
      for (int k = 0; k < A.d && holds; ++k) holds = S.lam[k] <= A.grids[g].l[k];
      const unsigned m = __ballot_sync(0xffffffffu, holds);
      if (FILL && holds) A.contrib[at + __popc(m & ((1u << lane) - 1))] = g;
      at += __popc(m);
      cnt += __popc(m);
    }
    if (!FILL && lane == 0) S.nc = cnt;
  }
}

// exclusive scan of nc into c0 (one CTA; a few thousand subspaces)
__global__ void __launch_bounds__(kThreads) k_contrib_scan(const __grid_constant__ CombiArgs A) {
  __shared__ int64_t part[kThreads];
  const int per = (A.nsubs + kThreads - 1) / kThreads;
  const int b = threadIdx.x * per, e = min(A.nsubs, b + per);
  int64_t acc = 0;
  for (int i = b; i < e; ++i) acc += A.subs[i].nc;
  part[threadIdx.x] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    int64_t run = 0;
    for (int t = 0; t < kThreads; ++t) {
      const int64_t v = part[t];
      part[t] = run;
      run += v;
    }
  }
  __syncthreads();
  acc = part[threadIdx.x];
  for (int i = b; i < e; ++i) {
    A.subs[i].c0 = acc;
    acc += A.subs[i].nc;
  }
}

// the coarse subspaces (lam_1 < thr of their family): per-subspace tiles of
// kCombiPts points, kCombiPts / kThreads points per thread, contributing grids
// staged in SMEM in batches of kGBatch (base, coefficient, shift l_k - lam_k,
// stride), K loads in flight per grid; sums in grid order as above
constexpr int kGBatch = 64;
template <int D>
struct GatherCon {
  const double *grid;
  double coeff;
  int32_t str[D];
  int8_t sh[D];
};
template <int D>
__global__ void __launch_bounds__(kThreads) k_gather_sub(const __grid_constant__ CombiArgs A) {
  __shared__ CombiSub s_sub;
  __shared__ GatherCon<D> s_con[kGBatch];
  constexpr int K = kCombiPts / kThreads;
  int idx = -1, cur = -1;
  for (int64_t q = blockIdx.x; q < A.ctiles; q += gridDim.x) {
    idx = combi_item_in(A.cprefix, A.ncsubs, idx, q);
    if (idx != cur) {
      __syncthreads();
      if (threadIdx.x == 0) s_sub = A.subs[__ldg(&A.csubs[idx])];
      __syncthreads();
      cur = idx;
    }
    const int nc = s_sub.nc;
    const int64_t c0 = s_sub.c0;
    const int p0 = (int)(q - __ldg(&A.cprefix[idx])) * kCombiPts;
    const int np = min(kCombiPts, s_sub.npts - p0);
    int jj[K][D];                                  // 2 j_k + 1 per point
#pragma unroll
    for (int u = 0; u < K; ++u) {
      int rest = p0 + threadIdx.x + u * kThreads;
#pragma unroll
      for (int k = 0; k < D; ++k) {               // j_1 fastest
        const int b = s_sub.lam[k] - 1;
        jj[u][k] = 2 * (rest & ((1 << b) - 1)) + 1;
        rest >>= b;
      }
    }
    double sum[K];
#pragma unroll
    for (int u = 0; u < K; ++u) sum[u] = 0.0;
    for (int cb = 0; cb < nc; cb += kGBatch) {
      const int nb = min(kGBatch, nc - cb);
      __syncthreads();                             // previous batch consumed
      if (threadIdx.x < nb) {
        const CombiGrid &G = A.grids[__ldg(&A.contrib[c0 + cb + threadIdx.x])];
        GatherCon<D> c;
        c.grid = G.grid;
        c.coeff = G.coeff;
#pragma unroll
        for (int k = 0; k < D; ++k) {
          c.str[k] = G.str[k];
          c.sh[k] = (int8_t)(G.l[k] - s_sub.lam[k]);
        }
        s_con[threadIdx.x] = c;
      }
      __syncthreads();
      for (int c = 0; c < nb; ++c) {               // grid order (deterministic)
        const GatherCon<D> &C = s_con[c];
        double v[K];
#pragma unroll
        for (int u = 0; u < K; ++u) {
          int gi = 0;
#pragma unroll
          for (int k = 0; k < D; ++k) gi += ((jj[u][k] << C.sh[k]) - 1) * C.str[k];
          v[u] = (threadIdx.x + u * kThreads < np) ? __ldg(C.grid + gi) : 0.0;
        }
#pragma unroll
        for (int u = 0; u < K; ++u) sum[u] = __dadd_rn(sum[u], __dmul_rn(C.coeff, v[u]));
      }
    }
#pragma unroll
    for (int u = 0; u < K; ++u) {
      const int qq = threadIdx.x + u * kThreads;
      if (qq < np) A.sparse[s_sub.off + p0 + qq] = sum[u];
    }
  }
}

// one family tile (see CombiFam): warps take 32-point chunks of its lam_1
// groups round robin (fine groups first), so a warp's lanes share one
// subspace and loop over its contributing grids together; every point sums
// its grids strictly in grid order from +0.0 with explicit __dmul_rn /
// __dadd_rn (bitwise the oracle's sequential sum), four grids' loads in flight
// No CTA barriers: descriptors are read through L1, so a warp stuck on a
// coarse point's long grid list does not hold the others back.
template <int D>
__global__ void __launch_bounds__(kThreads) k_gather(const __grid_constant__ CombiArgs A) {
  constexpr int NW = kThreads / 32;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int idx = -1;
  for (int64_t q = blockIdx.x; q < A.tiles; q += gridDim.x) {
    idx = combi_item(A, idx, q);
    const CombiFam &F = A.fams[idx];
    const int L = F.L, mlog = F.mlog, sub0 = F.sub0;
    int lamt[D];                                   // the tail lam_2..lam_d (lamt[0] unused)
#pragma unroll
    for (int k = 1; k < D; ++k) lamt[k] = F.lam[k];
    const int64_t ql = q - __ldg(&A.prefix[idx]);
    const bool rowtile = L <= kFamB;
    const int lo = rowtile ? 1 : L - kFamB + 1;   // coarsest lam_1 with more than the chunk's first point
    const int J0 = rowtile ? (int)(ql << mlog) : (int)(ql >> (L - kFamB));
    const int c = rowtile ? 0 : (int)(ql & ((int64_t(1) << (L - kFamB)) - 1));
    int kch = 0;                                   // warp chunks before this group
    for (int lam1 = L; lam1 >= F.thr; --lam1) {   // (thr > lo: the chunk's coarse points are elsewhere)
      const int lamg = lam1;
      const int cnt = rowtile ? (1 << (lam1 - 1 + mlog)) : (1 << (lam1 - lo));
      const int j1base = rowtile ? 0 : (int)((int64_t(c) << kFamB) >> (L - lam1 + 1));
      const int nch = (cnt + 31) >> 5;
      int ch = (warp - kch) % NW;
      if (ch < 0) ch += NW;
      kch += nch;
      if (ch >= nch) continue;
      const CombiSub &S = A.subs[__ldg(&A.fam_subs[sub0 + lamg - 1])];
      const int nc = S.nc;
      const int32_t *cl = A.contrib + S.c0;
      const int64_t soff = S.off;
      for (; ch < nch; ch += NW) {
        const int t = ch * 32 + lane;
        const bool valid = t < cnt;
        const int j1 = j1base + (t & ((1 << (lamg - 1)) - 1));
        const int jrow = J0 + (t >> (lamg - 1));
        int jj[D], lam[D];
        jj[0] = 2 * j1 + 1;
        lam[0] = lamg;
        int rest = jrow;
#pragma unroll
        for (int k = 1; k < D; ++k) {              // j_2 fastest
          const int b = lamt[k] - 1;
          jj[k] = 2 * (rest & ((1 << b) - 1)) + 1;
          rest >>= b;
          lam[k] = lamt[k];
        }
        // descriptors of 32 contributors at a time, one per lane (off the
        // per-grid critical path), broadcast with shuffles; 8 grids' loads in flight
        double sum = 0.0;
        for (int cb = 0; cb < nc; cb += 32) {
          const int nb = min(32, nc - cb);
          const double *my_grid = nullptr;
          double my_coeff = 0.0;
          int my_sh[D] = {}, my_str[D] = {};
          if (lane < nb) {
            const CombiGrid &G = A.grids[__ldg(cl + cb + lane)];
            my_grid = G.grid;
            my_coeff = G.coeff;
#pragma unroll
            for (int k = 0; k < D; ++k) {
              my_sh[k] = G.l[k] - lam[k];
              my_str[k] = G.str[k];
            }
          }
          for (int c8 = 0; c8 < nb; c8 += 8) {
            double w[8], v[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) {
              const int src = c8 + u;              // (src >= nb: the shuffles read lanes left idle)
              const double *gp = (const double *)__shfl_sync(0xffffffffu, (unsigned long long)my_grid, src & 31);
              w[u] = __shfl_sync(0xffffffffu, my_coeff, src & 31);
              int gi = 0;
#pragma unroll
              for (int k = 0; k < D; ++k)
                gi += ((jj[k] << __shfl_sync(0xffffffffu, my_sh[k], src & 31)) - 1) *
                      __shfl_sync(0xffffffffu, my_str[k], src & 31);
              v[u] = (valid && src < nb) ? __ldg(gp + gi) : 0.0;
            }
#pragma unroll
            for (int u = 0; u < 8; ++u)            // grid order (deterministic)
              if (c8 + u < nb) sum = __dadd_rn(sum, __dmul_rn(w[u], v[u]));
          }
        }
        if (valid) A.sparse[soff + j1 + (int64_t(jrow) << (lamg - 1))] = sum;
      }
    }
  }
}

// thread per grid point, in grid order (coalesced writes).  Measured: four
// points per thread with their loads issued first, descriptor in registers
// and contiguous tile ranges per CTA was slower on C5 (30.2 vs 27.0 ms)
template <int D>
__global__ void __launch_bounds__(kThreads) k_scatter(const __grid_constant__ CombiArgs A) {
  __shared__ int64_t s_binom[kCombiMaxN + 2][SGH_MAX_D + 1];
  __shared__ int64_t s_sbase[kCombiMaxN + 2];
  for (int i = threadIdx.x; i < (kCombiMaxN + 2) * (SGH_MAX_D + 1); i += kThreads)
    (&s_binom[0][0])[i] = (&c_binom[0][0])[i];
  for (int i = threadIdx.x; i < kCombiMaxN + 2; i += kThreads) s_sbase[i] = A.sbase[i];
  __syncthreads();
  int idx = -1;
  for (int64_t q = blockIdx.x; q < A.tiles; q += gridDim.x) {
    idx = combi_item(A, idx, q);
    const CombiGrid &G = A.grids[idx];
    const int64_t p0 = (q - __ldg(&A.prefix[idx])) * kCombiPts;
    const int np = (int)min((int64_t)kCombiPts, G.N - p0);
    for (int qq = threadIdx.x; qq < np; qq += kThreads) {
      uint32_t rest = (uint32_t)(p0 + qq);       // N < 2^31 per grid (checked on the host)
      int lam[D];
      int64_t in = 0;
      int sh = 0;
#pragma unroll
      for (int k = 0; k < D; ++k) {               // x_1 fastest
        const int lk = G.l[k];
        const uint32_t nk = (1u << lk) - 1;
        const uint32_t qk = (k == D - 1) ? 0u : fdiv(rest, G.fn[k]);
        const uint32_t i = rest - qk * nk + 1;    // 1-based
        rest = qk;
        const int t = __ffs(i) - 1;
        lam[k] = lk - t;
        in += int64_t(i >> (t + 1)) << sh;
        sh += lam[k] - 1;
      }
      G.grid[p0 + qq] = __ldg(A.sparse + sg_offset<D>(lam, s_binom, s_sbase) + in);
    }
  }
}

// ------------------------------------------------------------------ host
static void init_binom() {
  static std::once_flag once;
  static int64_t tab[kCombiMaxN + 2][SGH_MAX_D + 1];
  std::call_once(once, [] {
    for (int a = 0; a < kCombiMaxN + 2; ++a)
      for (int b = 0; b <= SGH_MAX_D; ++b) tab[a][b] = (b == 0) ? 1 : (a == 0 ? 0 : tab[a - 1][b - 1] + tab[a - 1][b]);
  });
  int dev = 0;
  cudaGetDevice(&dev);
  static std::mutex mu;
  static std::vector<int> done;
  std::lock_guard<std::mutex> lk(mu);
  if (std::find(done.begin(), done.end(), dev) != done.end()) return;
  cudaMemcpyToSymbol(c_binom, tab, sizeof tab);
  done.push_back(dev);
}

static int64_t binom_host(int a, int b) {
  if (b < 0 || a < b) return 0;
  int64_t r = 1;
  for (int i = 1; i <= b; ++i) r = r * (a - b + i) / i;
  return r;
}

// offsets of the level-sum blocks; returns total points, -1 if invalid
static int64_t sparse_bases(int d, int n, int64_t *sbase) {
  if (d < 1 || d > SGH_MAX_D || n < d || n > kCombiMaxN) return -1;
  int64_t acc = 0;
  for (int s = 0; s <= n + 1 && s < kCombiMaxN + 2; ++s) {
    if (sbase) sbase[s] = acc;
    if (s >= d && s <= n) {
      const int64_t cnt = binom_host(s - 1, d - 1);
      if (s - d > 40 || cnt > (int64_t(1) << 40)) return -1;
      acc += cnt << (s - d);
    }
  }
  return acc;
}

// lexicographic successor of a composition of s into d positive parts
static bool next_composition(int *lam, int d) {
  int tail = lam[d - 1];                           // sum of positions k+1 .. d-1
  for (int k = d - 2; k >= 0; --k) {
    if (tail > d - 1 - k) {                        // position k can take 1 more
      lam[k] += 1;
      const int r = tail - 1;                      // remaining for positions k+1..d-1
      for (int q = k + 1; q < d - 1; ++q) lam[q] = 1;
      lam[d - 1] = r - (d - 2 - k);
      return true;
    }
    tail += lam[k];
  }
  return false;
}

struct CombiPlan {
  std::vector<CombiGrid> grids;
  std::vector<CombiSub> subs;
  std::vector<int64_t> prefix;
  std::vector<CombiFam> fams;
  std::vector<int32_t> fam_subs;
  std::vector<int32_t> csubs;      // coarse subspaces (per-subspace tiles)
  std::vector<int64_t> cprefix;
  int64_t sbase[kCombiMaxN + 2];
  int64_t M = 0;
  int64_t ncontrib = 0;            // sum_g prod_k l_k: every (grid, subspace it holds) pair
  // workspace: [grids][subs][prefix][fams][fam_subs][contrib], each 256-byte aligned
  static size_t al(size_t b) { return (b + 255) / 256 * 256; }
  size_t off_subs() const { return al(grids.size() * sizeof(CombiGrid)); }
  size_t off_prefix() const { return off_subs() + al(subs.size() * sizeof(CombiSub)); }
  size_t off_fams() const { return off_prefix() + al(prefix.size() * 8); }
  size_t off_fam_subs() const { return off_fams() + al(fams.size() * sizeof(CombiFam)); }
  size_t off_csubs() const { return off_fam_subs() + al(fam_subs.size() * 4); }
  size_t off_cprefix() const { return off_csubs() + al(csubs.size() * 4); }
  size_t off_contrib() const { return off_cprefix() + al(cprefix.size() * 8); }
  size_t bytes() const { return off_contrib() + size_t(ncontrib) * 4 + 16; }
};

static sgh_status build_combi_plan(double *const *grids, const int32_t *levels, const double *coeffs, int32_t d,
                                   int64_t num_grids, int32_t n, bool gather, CombiPlan &P) {
  P.M = sparse_bases(d, n, P.sbase);
  if (P.M < 0) return invalid("unsupported (d, n) for the sparse grid (d <= 16, n <= 62)");
  if (num_grids >= (int64_t(1) << 31)) return invalid("too many grids");
  P.grids.resize(num_grids);
  P.ncontrib = 0;
  for (int64_t g = 0; g < num_grids; ++g) {
    int64_t N = 0;
    sgh_status st = validate_levels(levels + g * d, d, &N);
    if (st != SGH_OK) return st;
    int sum = 0;
    int64_t nsub = 1;
    for (int k = 0; k < d; ++k) {
      sum += levels[g * d + k];
      nsub *= levels[g * d + k];
    }
    if (sum > n) return invalid("a grid's level sum exceeds the sparse grid's n");
    if (N >= (int64_t(1) << 31)) return invalid("grid too large for gather/scatter (N >= 2^31)");
    if (grids && !grids[g]) return invalid("grids[g] is NULL");
    P.ncontrib += nsub;
    CombiGrid &G = P.grids[g];
    std::memset(&G, 0, sizeof G);
    G.grid = grids ? grids[g] : nullptr;
    G.coeff = coeffs ? coeffs[g] : 0.0;
    G.N = N;
    int32_t rs = 1;
    for (int k = 0; k < d; ++k) {
      G.l[k] = (int8_t)levels[g * d + k];
      G.fn[k] = make_fdiv((uint32_t)((1u << levels[g * d + k]) - 1));
      G.str[k] = rs;
      rs *= (int32_t)((1u << levels[g * d + k]) - 1);
    }
  }
  int64_t acc = 0;
  if (!gather) {
    P.ncontrib = 0;
    for (int64_t g = 0; g < num_grids; ++g) {
      P.prefix.push_back(acc);
      acc += (P.grids[g].N + kCombiPts - 1) / kCombiPts;
    }
    P.prefix.push_back(acc);
    return SGH_OK;
  }
  if (n - d > 30) return invalid("gather: subspaces of more than 2^30 points (n - d > 30)");
  std::vector<int> lam(d);
  std::map<std::vector<int8_t>, int32_t> where;    // subspace index by lam
  for (int s = d; s <= n; ++s) {                   // subspaces in SG order
    for (int k = 0; k < d - 1; ++k) lam[k] = 1;
    lam[d - 1] = s - (d - 1);
    int64_t off = P.sbase[s];
    do {
      CombiSub S;
      std::memset(&S, 0, sizeof S);
      S.off = off;
      S.npts = 1 << (s - d);
      for (int k = 0; k < d; ++k) S.lam[k] = (int8_t)lam[k];
      if (P.subs.size() >= (size_t(1) << 30)) return invalid("too many subspaces");
      where[std::vector<int8_t>(S.lam, S.lam + d)] = (int32_t)P.subs.size();
      P.subs.push_back(S);
      off += S.npts;
    } while (next_composition(lam.data(), d));
  }
  // families: tails lam' (compositions of s' into d - 1 parts), coarse tails first
  std::vector<int> tail(std::max(d - 1, 1));
  int64_t cacc = 0;
  for (int sp = d - 1; sp <= n - 1; ++sp) {
    if (d > 1) {
      for (int k = 0; k < d - 2; ++k) tail[k] = 1;
      tail[d - 2] = sp - (d - 2);
    }
    do {
      CombiFam F;
      std::memset(&F, 0, sizeof F);
      F.L = n - sp;
      F.rlog = sp - (d - 1);
      F.mlog = (F.L <= kFamB) ? std::min(F.rlog, kFamB - F.L) : 0;
      // lam_1 groups with >= 32 points per tile: 2^{lam_1 - 1 + mlog} (row tiles), 2^{lam_1 - lo} (chunks)
      F.thr = (F.L <= kFamB) ? std::max(1, 6 - F.mlog) : F.L - kFamB + 6;
      F.sub0 = (int32_t)P.fam_subs.size();
      std::vector<int8_t> key(d);
      for (int k = 1; k < d; ++k) key[k] = F.lam[k] = (int8_t)tail[k - 1];
      for (int l1 = 1; l1 <= F.L; ++l1) {
        key[0] = (int8_t)l1;
        const int32_t si = where.at(key);
        P.fam_subs.push_back(si);
        if (l1 < F.thr) {                          // coarse: a per-subspace tile list
          P.csubs.push_back(si);
          P.cprefix.push_back(cacc);
          cacc += (P.subs[si].npts + kCombiPts - 1) / kCombiPts;
        }
      }
      if (F.thr <= F.L) {                          // the family has fine groups
        P.fams.push_back(F);
        P.prefix.push_back(acc);
        acc += (F.L <= kFamB) ? (int64_t(1) << (F.rlog - F.mlog)) : (int64_t(1) << F.rlog) << (F.L - kFamB);
      }
    } while (d > 1 && next_composition(tail.data(), d - 1));
    if (d == 1) break;                             // one family, empty tail
  }
  P.prefix.push_back(acc);
  P.cprefix.push_back(cacc);
  return SGH_OK;
}

// persistent grids: exactly the CTAs that are resident at once (a second
// wave of a cyclic tile loop would start late and leave a long tail)
template <typename KernelFn>
static int64_t resident_grid(KernelFn fn, int64_t tiles, int sms) {
  int per = 1;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, fn, kThreads, 0) != cudaSuccess || per < 1) per = 1;
  return std::max<int64_t>(1, std::min<int64_t>(tiles, int64_t(sms) * per));
}

static sgh_status run_combi(double *const *grids, const int32_t *levels, const double *coeffs, int32_t d,
                            int64_t num_grids, int32_t n, double *sparse, void *workspace, size_t ws_bytes,
                            cudaStream_t s, bool gather) {
  if (num_grids < 0) return invalid("num_grids < 0");
  if (!levels || (num_grids > 0 && !grids) || !sparse || (gather && num_grids > 0 && !coeffs))
    return invalid("NULL argument");
  if (num_grids == 0 && !gather) return SGH_OK;
  CombiPlan P;
  sgh_status st = build_combi_plan(grids, levels, coeffs, d, num_grids, n, gather, P);
  if (st != SGH_OK) return st;
  const size_t need = P.bytes();
  if (!workspace || ws_bytes < need || (reinterpret_cast<uintptr_t>(workspace) & 15)) {
    set_error("workspace missing, misaligned or smaller than sgh_combi_workspace_bytes()");
    return SGH_ERR_WORKSPACE;
  }
  init_binom();
  const size_t up = P.off_contrib();               // tables uploaded; contrib is built on the device
  std::vector<unsigned char> host(up, 0);
  if (!P.grids.empty()) std::memcpy(host.data(), P.grids.data(), P.grids.size() * sizeof(CombiGrid));
  if (!P.subs.empty()) std::memcpy(host.data() + P.off_subs(), P.subs.data(), P.subs.size() * sizeof(CombiSub));
  std::memcpy(host.data() + P.off_prefix(), P.prefix.data(), P.prefix.size() * 8);
  if (!P.fams.empty()) std::memcpy(host.data() + P.off_fams(), P.fams.data(), P.fams.size() * sizeof(CombiFam));
  if (!P.fam_subs.empty()) std::memcpy(host.data() + P.off_fam_subs(), P.fam_subs.data(), P.fam_subs.size() * 4);
  if (!P.csubs.empty()) std::memcpy(host.data() + P.off_csubs(), P.csubs.data(), P.csubs.size() * 4);
  if (!P.cprefix.empty()) std::memcpy(host.data() + P.off_cprefix(), P.cprefix.data(), P.cprefix.size() * 8);
  if ((st = staged_upload(workspace, host.data(), up, s)) != SGH_OK) return st;
  unsigned char *ws = static_cast<unsigned char *>(workspace);
  CombiArgs A;
  std::memset(&A, 0, sizeof A);
  A.grids = reinterpret_cast<const CombiGrid *>(ws);
  A.subs = reinterpret_cast<CombiSub *>(ws + P.off_subs());
  A.prefix = reinterpret_cast<const int64_t *>(ws + P.off_prefix());
  A.contrib = reinterpret_cast<int32_t *>(ws + P.off_contrib());
  A.fams = reinterpret_cast<const CombiFam *>(ws + P.off_fams());
  A.fam_subs = reinterpret_cast<const int32_t *>(ws + P.off_fam_subs());
  A.nsubs = (int32_t)P.subs.size();
  A.csubs = reinterpret_cast<const int32_t *>(ws + P.off_csubs());
  A.cprefix = reinterpret_cast<const int64_t *>(ws + P.off_cprefix());
  A.ncsubs = (int32_t)P.csubs.size();
  A.ctiles = P.cprefix.empty() ? 0 : P.cprefix.back();
  A.items = gather ? (int32_t)P.fams.size() : (int32_t)P.grids.size();
  A.num_grids = (int32_t)num_grids;
  A.tiles = P.prefix.back();
  std::memcpy(A.sbase, P.sbase, sizeof A.sbase);
  A.sparse = sparse;
  A.d = d;
  A.n = n;
  if (gather ? A.nsubs == 0 : (A.items == 0 || A.tiles == 0)) return SGH_OK;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaError_t e = cudaSuccess;
  if (gather) {                                    // contributor lists, on the device
    const int64_t warps_grid = std::min<int64_t>((A.nsubs + 7) / 8, int64_t(sms) * 8);
    k_contrib<false><<<(unsigned)warps_grid, kThreads, 0, s>>>(A);
    k_contrib_scan<<<1, kThreads, 0, s>>>(A);
    k_contrib<true><<<(unsigned)warps_grid, kThreads, 0, s>>>(A);
    if ((e = cudaGetLastError()) != cudaSuccess) return cuda_fail(e, "contributor lists");
    count_launch(3);
  }
  const bool fam = gather && A.tiles > 0, sub = gather && A.ctiles > 0;
  ProfToken tok = prof_begin(s);
  switch (d) {
#define SGH_COMBI_CASE(DD)                                                                               \
  case DD:                                                                                               \
    if (fam) k_gather<DD><<<(unsigned)resident_grid(k_gather<DD>, A.tiles, sms), kThreads, 0, s>>>(A);   \
    if (sub)                                                                                             \
      k_gather_sub<DD><<<(unsigned)resident_grid(k_gather_sub<DD>, A.ctiles, sms), kThreads, 0, s>>>(A); \
    if (!gather) k_scatter<DD><<<(unsigned)resident_grid(k_scatter<DD>, A.tiles, sms), kThreads, 0, s>>>(A); \
    break;
    SGH_COMBI_CASE(1) SGH_COMBI_CASE(2) SGH_COMBI_CASE(3) SGH_COMBI_CASE(4) SGH_COMBI_CASE(5)
    SGH_COMBI_CASE(6) SGH_COMBI_CASE(7) SGH_COMBI_CASE(8) SGH_COMBI_CASE(9) SGH_COMBI_CASE(10)
    SGH_COMBI_CASE(11) SGH_COMBI_CASE(12) SGH_COMBI_CASE(13) SGH_COMBI_CASE(14) SGH_COMBI_CASE(15)
    SGH_COMBI_CASE(16)
#undef SGH_COMBI_CASE
    default: return invalid("d out of range");
  }
  e = cudaGetLastError();
  double pts = 0;
  for (const CombiGrid &G : P.grids) pts += double(G.N);
  prof_end(tok, gather ? 5 : 6, 0, false, 8.0 * pts + 8.0 * double(P.M), s);
  if (e != cudaSuccess) return cuda_fail(e, gather ? "gather launch" : "scatter launch");
  count_launch(gather ? int(fam) + int(sub) : 1);
  return SGH_OK;
}

}  // namespace sgh

using namespace sgh;

extern "C" {

int64_t sgh_sparse_num_points(int32_t d, int32_t n) { return sparse_bases(d, n, nullptr); }

size_t sgh_combi_workspace_bytes(const int32_t *levels, int32_t d, int64_t num_grids, int32_t n, uint32_t flags) {
  if (!levels || num_grids < 0) return 0;
  CombiPlan P;
  const bool gather = (flags & SGH_FLAG_SCATTER) == 0;
  if (build_combi_plan(nullptr, levels, nullptr, d, num_grids, n, gather, P) != SGH_OK) return 0;
  return P.bytes();
}

sgh_status sgh_gather(const double *const *grids, const int32_t *levels, const double *coeffs, int32_t d,
                      int64_t num_grids, int32_t n, double *sparse, void *workspace, size_t ws_bytes, void *stream) {
  return run_combi(const_cast<double *const *>(grids), levels, coeffs, d, num_grids, n, sparse, workspace, ws_bytes,
                   static_cast<cudaStream_t>(stream), true);
}

sgh_status sgh_scatter(double *const *grids, const int32_t *levels, int32_t d, int64_t num_grids, int32_t n,
                       const double *sparse, void *workspace, size_t ws_bytes, void *stream) {
  return run_combi(grids, levels, nullptr, d, num_grids, n, const_cast<double *>(sparse), workspace, ws_bytes,
                   static_cast<cudaStream_t>(stream), false);
}

}  // extern "C"
