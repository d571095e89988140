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
  int32_t *contrib;                // grid indices, grouped per subspace, in grid order
  const int64_t *prefix;           // tile prefix over subs (gather) or grids (scatter), items + 1 entries
  int32_t items;                   // subspaces (gather) or grids (scatter)
  int32_t num_grids;
  int64_t tiles;
  int64_t sbase[kCombiMaxN + 2];   // offset of the first subspace of level sum s
  double *sparse;
  int32_t d, n;
  int32_t accumulate;              // gather: sums start from the values in sparse (SGH_FLAG_ACCUMULATE)
  int32_t x1_bfs;                  // gather: the grids' x_1 rows are in BFS order (SGH_FLAG_X1_BFS)
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
__device__ __forceinline__ int combi_item(const CombiArgs &A, int idx, int64_t q) {
  if (idx < 0) {
    int lo = 0, hi = A.items - 1;
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (__ldg(&A.prefix[mid]) <= q) lo = mid; else hi = mid - 1;
    }
    return lo;
  }
  if (idx + 1 >= A.items || __ldg(&A.prefix[idx + 1]) > q) return idx;
  int lo = idx + 1, step = 1, hi = lo + 1;
  while (hi < A.items && __ldg(&A.prefix[hi]) <= q) {
    lo = hi;
    step <<= 1;
    hi = lo + step;
  }
  if (hi > A.items) hi = A.items;
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if (__ldg(&A.prefix[mid]) <= q) lo = mid; else hi = mid;
  }
  return lo;
}

// one warp per subspace: count (fill = false) or list (fill = true) the grids
// holding it, in grid order (ballot + popc keeps the order)
template <bool FILL>
__global__ void __launch_bounds__(kThreads) k_contrib(const __grid_constant__ CombiArgs A) {
  const int lane = threadIdx.x & 31;
  for (int sidx = (blockIdx.x * kThreads + threadIdx.x) >> 5; sidx < A.items;
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
  const int per = (A.items + kThreads - 1) / kThreads;
  const int b = threadIdx.x * per, e = min(A.items, b + per);
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

// thread per sparse point of a subspace chunk (kCombiPts points per tile),
// kCombiPts / kThreads points per thread; the contributing grids are staged in
// SMEM in batches of kGBatch (base, coefficient, shift l_k - lam_k, stride:
// grid index = sum_k (((2 j_k + 1) << sh_k) - 1) str_k), so no descriptor load
// sits on the per-grid critical path and every thread has K independent loads
// in flight per grid.  Each point accumulates its grids strictly in grid order
// from +0.0 with explicit __dmul_rn / __dadd_rn: bitwise the oracle's
// "for g in order: sparse += coeff_g * alpha_g".  (C5: 37.2 vs 39.8 ms for a
// thread per point reading the descriptors through L1.)
constexpr int kGBatch = 64;
template <int D>
struct GatherCon {
  const double *grid;
  double coeff;
  int32_t str[D];
  int8_t sh[D];
};
template <int D>
__global__ void __launch_bounds__(kThreads) k_gather(const __grid_constant__ CombiArgs A) {
  __shared__ CombiSub s_sub;
  __shared__ GatherCon<D> s_con[kGBatch];
  constexpr int K = kCombiPts / kThreads;
  int idx = -1, cur = -1;
  for (int64_t q = blockIdx.x; q < A.tiles; q += gridDim.x) {
    idx = combi_item(A, idx, q);
    if (idx != cur) {
      __syncthreads();
      if (threadIdx.x == 0) s_sub = A.subs[idx];
      __syncthreads();
      cur = idx;
    }
    const int nc = s_sub.nc;
    const int64_t c0 = s_sub.c0;
    const bool bfs = A.x1_bfs != 0;
    const int x1base = (1 << (s_sub.lam[0] - 1)) - 1;     // BFS x_1 rows: level lam_1 starts here
    const int p0 = (int)(q - __ldg(&A.prefix[idx])) * kCombiPts;
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
    double sum[K];                                 // +0.0, or the running sum of earlier grids
#pragma unroll
    for (int u = 0; u < K; ++u) {
      const int qq = threadIdx.x + u * kThreads;
      sum[u] = (A.accumulate && qq < np) ? A.sparse[s_sub.off + p0 + qq] : 0.0;
    }
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
          for (int k = 0; k < D; ++k) {
            if (k == 0 && bfs) gi += x1base + (jj[u][0] >> 1);   // BFS row: level block, then j_1
            else gi += ((jj[u][k] << C.sh[k]) - 1) * C.str[k];
          }
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
  int64_t sbase[kCombiMaxN + 2];
  int64_t M = 0;
  int64_t ncontrib = 0;            // sum_g prod_k l_k: every (grid, subspace it holds) pair
  // workspace: [grids][subs][prefix][contrib], each 256-byte aligned
  size_t off_subs() const { return (grids.size() * sizeof(CombiGrid) + 255) / 256 * 256; }
  size_t off_prefix() const { return off_subs() + (subs.size() * sizeof(CombiSub) + 255) / 256 * 256; }
  size_t off_contrib() const { return off_prefix() + (prefix.size() * 8 + 255) / 256 * 256; }
  size_t bytes() const { return off_contrib() + size_t(ncontrib) * 4 + 16; }
};

static sgh_status build_combi_plan(double *const *grids, const int32_t *levels, const double *coeffs, int32_t d,
                                   int64_t num_grids, int32_t n, bool gather, CombiPlan &P, int64_t sub_begin = 0,
                                   int64_t sub_end = INT64_MAX) {
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
  // a subspace has 2^{s-d} points, indexed in int32 by the gather kernel; no
  // grid can hold a larger one anyway (N < 2^31 per grid)
  if (n - d > 30) return invalid("gather: subspaces of more than 2^30 points (n - d > 30)");
  {                                                // refuse before listing: C(n, d) can be ~1e14
    const int64_t total = binom_host(n, d);
    const int64_t cnt = std::min(sub_end, total) - std::max<int64_t>(sub_begin, 0);
    if (cnt >= (int64_t(1) << 31)) {
      set_error("gather: too many subspaces in the requested range (>= 2^31)");
      return SGH_ERR_CAPACITY;
    }
  }
  std::vector<int> lam(d);
  int64_t si = 0;                                  // subspace index in SG order
  for (int s = d; s <= n && si < sub_end; ++s) {   // subspaces in SG order
    const int64_t cnt = binom_host(s - 1, d - 1);
    if (si + cnt <= sub_begin) {                   // level sum entirely before the range
      si += cnt;
      continue;
    }
    for (int k = 0; k < d - 1; ++k) lam[k] = 1;
    lam[d - 1] = s - (d - 1);
    int64_t off = P.sbase[s];
    do {
      const bool in = si >= sub_begin && si < sub_end;
      ++si;
      if (!in) {
        off += int64_t(1) << (s - d);
        continue;
      }
      CombiSub S;
      std::memset(&S, 0, sizeof S);
      S.off = off;
      S.npts = 1 << (s - d);
      for (int k = 0; k < d; ++k) S.lam[k] = (int8_t)lam[k];
      P.subs.push_back(S);
      P.prefix.push_back(acc);
      acc += (S.npts + kCombiPts - 1) / kCombiPts;
      off += S.npts;
    } while (next_composition(lam.data(), d));
  }
  P.prefix.push_back(acc);
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
                            cudaStream_t s, bool gather, int64_t sub_begin = 0, int64_t sub_end = INT64_MAX,
                            uint32_t flags = 0) {
  if (num_grids < 0) return invalid("num_grids < 0");
  if (!levels || (num_grids > 0 && !grids) || !sparse || (gather && num_grids > 0 && !coeffs))
    return invalid("NULL argument");
  if (num_grids == 0 && !gather) return SGH_OK;
  if (flags & ~uint32_t(SGH_FLAG_ACCUMULATE | SGH_FLAG_X1_BFS)) return invalid("unknown gather flags");
  CombiPlan P;
  sgh_status st = build_combi_plan(grids, levels, coeffs, d, num_grids, n, gather, P, sub_begin, sub_end);
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
  if ((st = staged_upload(workspace, host.data(), up, s)) != SGH_OK) return st;
  unsigned char *ws = static_cast<unsigned char *>(workspace);
  CombiArgs A;
  std::memset(&A, 0, sizeof A);
  A.grids = reinterpret_cast<const CombiGrid *>(ws);
  A.subs = reinterpret_cast<CombiSub *>(ws + P.off_subs());
  A.prefix = reinterpret_cast<const int64_t *>(ws + P.off_prefix());
  A.contrib = reinterpret_cast<int32_t *>(ws + P.off_contrib());
  A.items = gather ? (int32_t)P.subs.size() : (int32_t)P.grids.size();
  A.num_grids = (int32_t)num_grids;
  A.tiles = P.prefix.back();
  std::memcpy(A.sbase, P.sbase, sizeof A.sbase);
  A.sparse = sparse;
  A.d = d;
  A.n = n;
  A.accumulate = (flags & SGH_FLAG_ACCUMULATE) ? 1 : 0;
  A.x1_bfs = (flags & SGH_FLAG_X1_BFS) ? 1 : 0;
  if (A.items == 0 || A.tiles == 0) return SGH_OK;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaError_t e = cudaSuccess;
  if (gather) {                                    // contributor lists, on the device
    const int64_t warps_grid = std::min<int64_t>((A.items + 7) / 8, int64_t(sms) * 8);
    k_contrib<false><<<(unsigned)warps_grid, kThreads, 0, s>>>(A);
    k_contrib_scan<<<1, kThreads, 0, s>>>(A);
    k_contrib<true><<<(unsigned)warps_grid, kThreads, 0, s>>>(A);
    if ((e = cudaGetLastError()) != cudaSuccess) return cuda_fail(e, "contributor lists");
    count_launch(3);
  }
  ProfToken tok = prof_begin(s);
  switch (d) {
#define SGH_COMBI_CASE(DD)                                                                              \
  case DD:                                                                                              \
    if (gather) k_gather<DD><<<(unsigned)resident_grid(k_gather<DD>, A.tiles, sms), kThreads, 0, s>>>(A); \
    else k_scatter<DD><<<(unsigned)resident_grid(k_scatter<DD>, A.tiles, sms), kThreads, 0, s>>>(A);     \
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
  count_launch();
  return SGH_OK;
}

// ------------------------------------------------ x_1 rows in BFS order
// The gather reads grid g's point (j_1, ..) of W_lam at x_1 index
// (2 j_1 + 1) 2^{l_1 - lam_1}: consecutive sparse points are 2^{l_1-lam_1+1}
// doubles apart, one useful double per 32-byte sector for every lam_1 < l_1
// (DRAM reads ~6x the surpluses).  Permuting every x_1 row into BFS order --
// level 1 first, then level 2, .., each level's points by j_1 (P:232-233,
// Fig. fig:hierDehier: the paper's BFS layout) -- makes those reads
// contiguous runs; the sums are unchanged (the same values, added in the
// same order).  Natural 1-based index i (level lam = l_1 - tz(i),
// j = i >> (tz(i) + 1)) goes to BFS position 2^{lam-1} - 1 + j.
constexpr int kPermBatch = 96;     // grids per launch (kernel parameter table)
constexpr int kPermSeg = 4096;     // points per tile: R whole rows (l_1 <= 12) or a 2^12 row segment
struct PermGrid {
  const double *src;
  double *dst;
  int64_t rows;                    // N / n_1
  int32_t l1, R;                   // R rows per tile (l_1 <= 12)
  FDiv fn1;                        // division by n_1
};
struct PermArgs {
  PermGrid g[kPermBatch];
  int64_t prefix[kPermBatch + 1];  // tiles
  int32_t ng;
};

__global__ void __launch_bounds__(kThreads) k_x1_bfs(const __grid_constant__ PermArgs A) {
  __shared__ double s[kPermSeg];
  int gi = 0;
  const int64_t total = A.prefix[A.ng];
  for (int64_t q = blockIdx.x; q < total; q += gridDim.x) {
    while (A.prefix[gi + 1] <= q) ++gi;            // tiles of a CTA only increase
    const PermGrid &G = A.g[gi];
    const int64_t lq = q - A.prefix[gi];
    const int l1 = G.l1;
    const int n1 = (1 << l1) - 1;
    __syncthreads();                               // the previous tile's reads of s are done
    if (l1 <= 12) {                                // R whole rows: one contiguous range
      const int64_t r0 = lq * G.R;
      const int nr = (int)min((int64_t)G.R, G.rows - r0);
      const double *src = G.src + r0 * n1;
      double *dst = G.dst + r0 * n1;
      const int cnt = nr * n1;
      for (int e = threadIdx.x; e < cnt; e += kThreads) s[e] = __ldcs(src + e);
      __syncthreads();
      for (int o = threadIdx.x; o < cnt; o += kThreads) {
        const int row = (int)fdiv((uint32_t)o, G.fn1);
        const int p = o - row * n1;                // BFS position
        const int lam = 32 - __clz(p + 1);         // level: positions 2^{lam-1}-1 .. 2^lam-2
        const int j = p + 1 - (1 << (lam - 1));
        const int i = (2 * j + 1) << (l1 - lam);   // natural 1-based index
        dst[o] = s[row * n1 + i - 1];
      }
    } else {                                       // one aligned 2^12-index segment of one row
      const int sh = l1 - 12;
      const int64_t row = lq >> sh;
      const int S0 = (int)(lq & ((1 << sh) - 1)) << 12;
      const double *src = G.src + row * n1;
      double *dst = G.dst + row * n1;
      for (int k = threadIdx.x; k < kPermSeg; k += kThreads) {
        const int i = S0 + k;
        if (i >= 1 && i <= n1) s[k] = __ldcs(src + i - 1);
      }
      __syncthreads();
      // levels with tz(i) = t < 12: 2^{11-t} points S0 + 2^t (2m + 1), at the
      // contiguous BFS positions 2^{l1-t-1} - 1 + (S0 >> (t+1)) + m
      for (int o = threadIdx.x; o < kPermSeg - 1; o += kThreads) {
        const int t = 11 - (31 - __clz(kPermSeg - 1 - o));   // run t covers o in [4096 - 2^{12-t}, 4096 - 2^{11-t})
        const int m = o - (kPermSeg - (kPermSeg >> t));
        const int i = S0 + (1 << t) * (2 * m + 1);
        dst[((1 << (l1 - t - 1)) - 1) + (S0 >> (t + 1)) + m] = s[i - S0];
      }
      if (threadIdx.x == 0 && S0 > 0) {            // the segment's first index: a coarser level
        const int t = __ffs(S0) - 1;
        dst[((1 << (l1 - t - 1)) - 1) + (S0 >> (t + 1))] = s[0];
      }
    }
  }
}

static sgh_status permute_x1_bfs(const double *const *src, double *const *dst, const int32_t *levels, int32_t d,
                                 int64_t num_grids, cudaStream_t s) {
  if (num_grids < 0) return invalid("num_grids < 0");
  if (num_grids > 0 && (!src || !dst || !levels)) return invalid("NULL argument");
  for (int64_t b = 0; b < num_grids; b += kPermBatch) {
    PermArgs A;
    std::memset(&A, 0, sizeof A);
    A.ng = (int32_t)std::min<int64_t>(kPermBatch, num_grids - b);
    int64_t acc = 0;
    for (int k = 0; k < A.ng; ++k) {
      const int64_t g = b + k;
      int64_t N = 0;
      sgh_status st = validate_levels(levels + g * d, d, &N);
      if (st != SGH_OK) return st;
      if (!src[g] || !dst[g]) return invalid("grid pointer is NULL");
      if (src[g] == dst[g]) return invalid("the permutation is out of place (src == dst)");
      PermGrid &P = A.g[k];
      P.src = src[g];
      P.dst = dst[g];
      P.l1 = levels[g * d];
      const int64_t n1 = (int64_t(1) << P.l1) - 1;
      P.rows = N / n1;
      P.R = P.l1 <= 12 ? (kPermSeg >> P.l1) : 1;
      P.fn1 = make_fdiv((uint32_t)n1);
      A.prefix[k] = acc;
      acc += P.l1 <= 12 ? (P.rows + P.R - 1) / P.R : (P.rows << (P.l1 - 12));
    }
    A.prefix[A.ng] = acc;
    if (acc == 0) continue;
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int64_t grid = std::min<int64_t>(acc, int64_t(sms) * 6);
    k_x1_bfs<<<(unsigned)grid, kThreads, 0, s>>>(A);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_fail(e, "x1 BFS permutation");
    count_launch();
  }
  return SGH_OK;
}

}  // namespace sgh

using namespace sgh;

extern "C" {

int64_t sgh_sparse_num_points(int32_t d, int32_t n) { return sparse_bases(d, n, nullptr); }

int64_t sgh_sparse_num_subspaces(int32_t d, int32_t n) {
  if (sparse_bases(d, n, nullptr) < 0) return -1;
  return binom_host(n, d);                         // sum_{s=d}^{n} C(s-1, d-1)
}

int64_t sgh_sparse_subspace_offset(int32_t d, int32_t n, int64_t index) {
  int64_t sbase[kCombiMaxN + 2];
  if (sparse_bases(d, n, sbase) < 0 || index < 0 || index > binom_host(n, d)) return -1;
  int64_t first = 0;                               // index of the first subspace of level sum s
  for (int s = d; s <= n; ++s) {
    const int64_t cnt = binom_host(s - 1, d - 1);
    if (index < first + cnt) return sbase[s] + ((index - first) << (s - d));
    first += cnt;
  }
  return sbase[n + 1];                             // index == count: the total
}

size_t sgh_combi_workspace_bytes(const int32_t *levels, int32_t d, int64_t num_grids, int32_t n, uint32_t flags) {
  return guarded_value<size_t>(0, [&]() -> size_t {
  if (!levels || num_grids < 0) return 0;
  CombiPlan P;
  const bool gather = (flags & SGH_FLAG_SCATTER) == 0;
  if (build_combi_plan(nullptr, levels, nullptr, d, num_grids, n, gather, P) != SGH_OK) return 0;
  return P.bytes();
});
}

sgh_status sgh_gather(const double *const *grids, const int32_t *levels, const double *coeffs, int32_t d,
                      int64_t num_grids, int32_t n, double *sparse, void *workspace, size_t ws_bytes, void *stream) {
  return guarded([&]() -> sgh_status {
  return run_combi(const_cast<double *const *>(grids), levels, coeffs, d, num_grids, n, sparse, workspace, ws_bytes,
                   static_cast<cudaStream_t>(stream), true);
});
}

sgh_status sgh_gather_ex(const double *const *grids, const int32_t *levels, const double *coeffs, int32_t d,
                         int64_t num_grids, int32_t n, double *sparse, int64_t sub_begin, int64_t sub_end,
                         uint32_t flags, void *workspace, size_t ws_bytes, void *stream) {
  return guarded([&]() -> sgh_status {
  const int64_t nsub = sgh_sparse_num_subspaces(d, n);
  if (nsub < 0) return invalid("unsupported (d, n) for the sparse grid");
  if (sub_begin < 0 || sub_end < sub_begin || sub_end > nsub) return invalid("subspace range out of bounds");
  if (sub_begin == sub_end) return SGH_OK;
  return run_combi(const_cast<double *const *>(grids), levels, coeffs, d, num_grids, n, sparse, workspace, ws_bytes,
                   static_cast<cudaStream_t>(stream), true, sub_begin, sub_end, flags);
});
}

sgh_status sgh_permute_x1_bfs(const double *const *src, double *const *dst, const int32_t *levels, int32_t d,
                              int64_t num_grids, void *stream) {
  return guarded([&]() -> sgh_status {
  return permute_x1_bfs(src, dst, levels, d, num_grids, static_cast<cudaStream_t>(stream));
});
}

sgh_status sgh_scatter(double *const *grids, const int32_t *levels, int32_t d, int64_t num_grids, int32_t n,
                       const double *sparse, void *workspace, size_t ws_bytes, void *stream) {
  return guarded([&]() -> sgh_status {
  return run_combi(grids, levels, nullptr, d, num_grids, n, const_cast<double *>(sparse), workspace, ws_bytes,
                   static_cast<cudaStream_t>(stream), false);
});
}

}  // extern "C"
