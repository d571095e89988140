// sgh_capi.cu -- the extern "C" surface of libsgh (include/sgh.h): argument
// validation, the per-axis planner, single-grid and batched drivers, fill and
// digest utilities.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <tuple>
#include <vector>

#include "../../include/sgh.h"
#include "sgh_common.cuh"
#include "sgh_plan.hpp"

namespace sgh {

uint64_t host_splitmix_finalise(uint64_t z);
int64_t util_chunks(int64_t n);
cudaError_t launch_fill(const FillItem *d_items, const int64_t *d_prefix, int nitems, const FillItem &single,
                        int64_t total_chunks, cudaStream_t st);
cudaError_t launch_digest(const FillItem *d_items, const int64_t *d_prefix, int nitems, const FillItem &single,
                          int64_t total_chunks, unsigned long long *d_out, cudaStream_t st);

// ------------------------------------------------------------ bookkeeping
static thread_local std::string g_last_error;
static std::atomic<uint64_t> g_launches{0};

void set_error(const std::string &msg) { g_last_error = msg; }
void count_launch(uint64_t k) { g_launches.fetch_add(k, std::memory_order_relaxed); }

sgh_status cuda_fail(cudaError_t e, const char *where) {
  set_error(std::string(where) + ": " + cudaGetErrorName(e) + " (" + cudaGetErrorString(e) + ")");
  return SGH_ERR_CUDA;
}

sgh_status invalid(const char *msg) {
  set_error(msg);
  return SGH_ERR_INVALID_ARGUMENT;
}

// levels: d in [1, SGH_MAX_D], l_k >= 1 -> INVALID; l_k > SGH_MAX_LEVEL or N*8 overflow -> CAPACITY
sgh_status validate_levels(const int32_t *levels, int32_t d, int64_t *N_out) {
  if (!levels) return invalid("levels is NULL");
  if (d < 1 || d > SGH_MAX_D) return invalid("d out of range [1, SGH_MAX_D]");
  int64_t N = 1;
  for (int k = 0; k < d; ++k) {
    if (levels[k] < 1) return invalid("level < 1");
    if (levels[k] > SGH_MAX_LEVEL) {
      set_error("level > SGH_MAX_LEVEL");
      return SGH_ERR_CAPACITY;
    }
    const int64_t nk = (int64_t(1) << levels[k]) - 1;
    if (N > (INT64_MAX / 8) / nk) {
      set_error("grid size overflows int64 bytes");
      return SGH_ERR_CAPACITY;
    }
    N *= nk;
  }
  if (N_out) *N_out = N;
  return SGH_OK;
}

// ---------------------------------------------------------------- planner
static int floor_log2(int64_t x) {
  int r = -1;
  while (x) { ++r; x >>= 1; }
  return r;
}

void plan_view(double *grid, int64_t O, int64_t OS, int64_t PS, int64_t S, int64_t base, int l,
               std::vector<Task> &phases) {
  if (l <= 1 || O <= 0 || S <= 0) return;
  const int64_t n = (int64_t(1) << l) - 1;
  Task t;
  std::memset(&t, 0, sizeof t);
  t.bt2 = -1;
  t.grid = grid;
  t.O = O;
  t.OS = OS;
  t.PS = PS;
  t.S = S;
  t.base = base;
  t.l = l;
  const bool contiguous_slabs = (PS == S) && (OS == n * S);
  if (contiguous_slabs && S < kFlatMaxS) {
    t.fS = make_fdiv((uint32_t)S);
    if (n * S <= kFlatT) {                               // whole slabs per tile
      t.kind = KIND_FLAT_SLABS;
      t.t = l;
      t.R = (int32_t)(kFlatT / (n * S));
      t.tiles = (O + t.R - 1) / t.R;
      t.fNS = make_fdiv((uint32_t)(n * S));
      phases.push_back(t);
      return;
    }
    const int tb = floor_log2(kFlatT / S);               // 2^tb * S <= kFlatT < 2^l * S
    t.kind = KIND_FLAT_BLOCKS;
    t.t = tb;
    t.rlog = l - tb;
    t.tiles = O << (l - tb);
    phases.push_back(t);
    plan_view(grid, O, OS, PS << tb, S, base + ((int64_t(1) << tb) - 1) * PS, l - tb, phases);
    return;
  }
  if (l <= kRegMaxL) {
    t.kind = KIND_REG;
    t.t = l;
    const int64_t cols_per_tile = int64_t(kThreads) * std::max(1, 16 / (int)n);   // RegCfg<L>::CPT
    t.tiles = (O * S + cols_per_tile - 1) / cols_per_tile;
    phases.push_back(t);
    return;
  }
  // tile width: as wide as the columns allow (long contiguous row segments keep
  // DRAM pages open), rows = 2^t + 1 within the SMEM budget
  static int wpref = -1;
  if (wpref < 0) {
    const char *e = tuning_env("SGH_STRIDED_W");  // tuning experiment override
    wpref = e ? atoi(e) : 256;
    if (wpref != 32 && wpref != 64 && wpref != 128 && wpref != 256) wpref = 128;
  }
  static int64_t tile_budget = -1;
  if (tile_budget < 0) {
    const char *e = tuning_env("SGH_STRIDED_TILE");  // tuning experiment override (doubles)
    tile_budget = e ? atoll(e) : kStridedTileDoubles;
    if (tile_budget < 1024 || tile_budget > 13000) tile_budget = kStridedTileDoubles;
  }
  auto tmax_of = [&](int w) {
    int tm = 0;
    while (((int64_t(1) << (tm + 1)) + 1) * (w + 2) <= tile_budget) ++tm;
    return tm;
  };
  int W = wpref;
  while (W > 32 && S <= W / 2 + W / 4) W >>= 1;
  // Prefer a width whose tile holds the whole pole (no coarse-lattice phase;
  // l - t == 1 leaves only the root, which has no update) as long as rows stay
  // >= 512 B; otherwise the widest tile and a lattice phase.
  for (int w = W; w >= 64; w >>= 1)
    if (tmax_of(w) >= l - 1) {
      W = w;
      break;
    }
  const int tb = std::min(l, tmax_of(W));   // l - tb == 1: the lattice is the root alone (no phase)
  t.kind = KIND_STRIDED;
  t.W = W;
  t.t = tb;
  t.rlog = l - tb;
  t.ncb = (S + W - 1) / W;
  t.tiles = (O << (l - tb)) * t.ncb;
  phases.push_back(t);
  if (tb < l) plan_view(grid, O, OS, PS << tb, S, base + ((int64_t(1) << tb) - 1) * PS, l - tb, phases);
}

// Outer multiplier of the planner (1 = a whole grid).  The sharded paths plan
// a row shard of x_d as `rows` consecutive (d-1)-dimensional grids: every
// planned view's outer count O (units beyond its axis group, dense at stride
// OS with O * OS = the grid's extent) is multiplied by it, which extends the
// view over the stacked copies.  Two-blocked plans (whose outer index is split,
// O1 / OS2) are not used while it is set.  Thread-local: set it only through
// plan_grid_rows.
static thread_local int64_t g_outer_mult = 1;

void plan_axis(double *grid, const int32_t *levels, int d, int k, std::vector<Task> &phases, int64_t rows_last) {
  int64_t S = 1, O = g_outer_mult;
  for (int j = 0; j < k; ++j) S *= (int64_t(1) << levels[j]) - 1;
  for (int j = k + 1; j < d; ++j) O *= (j == d - 1 && rows_last >= 0) ? rows_last : (int64_t(1) << levels[j]) - 1;
  const int64_t n = (int64_t(1) << levels[k]) - 1;
  plan_view(grid, O, n * S, S, S, 0, levels[k], phases);
}

// Whole-pole multi-axis group [a, b).  Returns false if the
// group's tile does not fit the FUSED budget.
static int fused_budget() {
  static int T = -1;
  if (T < 0) {
    const char *e = tuning_env("SGH_FUSED_T");  // tuning experiment override
    T = e ? atoi(e) : kFusedT;
    if (T < 1024 || T > 14336) T = kFusedT;
  }
  return T;
}

// W == 1 (contiguous) FUSED tile budget (kFusedT1); SGH_FUSED_T1 overrides
// (experiments with smaller W == 1 CTAs, sgh_kernels.cu FT<1>)
static int fused_budget_w1() {
  static int T = -1;
  if (T < 0) {
    const char *e = tuning_env("SGH_FUSED_T1");
    T = e ? atoi(e) : kFusedT1;
    if (T < 1024 || T > 14336) T = kFusedT1;
  }
  return T;
}

static int fused_wmax() {
  static int wmax = -1;
  if (wmax < 0) {
    const char *e = tuning_env("SGH_FUSED_W");  // tuning experiment override (8..128)
    wmax = e ? atoi(e) : 128;
    if (wmax != 8 && wmax != 16 && wmax != 32 && wmax != 64 && wmax != 128) wmax = 128;
  }
  return wmax;
}

// per-axis constants of a full FUSED tile (Task::gOk, Task::fNP)
static void finish_fused(Task &t) {
  const int64_t rows = int64_t(t.P) * (t.W == 1 ? t.R : 1);   // R units per W == 1 tile (dense, lattice views)
  const int Wc = t.W == 1 ? 1 : t.W;
  for (int j = 0; j < t.m; ++j) {
    int64_t e = (int64_t(1) << t.gl[j]) - 1;
    if (t.bj >= 0 && j == t.bj) e = t.ej;
    if (t.bj >= 0 && t.bt2 >= 0 && j == t.bj + 1) e = (int64_t(1) << t.bt2) + 1;
    const int64_t ok = rows / (e * t.gR[j]);
    t.gOk[j] = (int32_t)ok;
    const int64_t np = ok * t.gR[j] * Wc;
    t.fNP[j] = make_fdiv((uint32_t)std::max<int64_t>(1, np));
  }
}

// PADDED SMEM layout (Task::sy / sz) for W == 1 special-axis tasks whose tile
// rows do not keep the global 8-byte phase in the dense layout (coarse-lattice
// views: Gj even, A odd): rows of the special axis at an SMEM pitch sy of
// Gj's parity, rows after it at a pitch sz of Gnext's parity, so every run
// starts at its global phase and the task loads / stores with 16-byte and
// bulk copies (`aligned`).  Runs of one element (A == 1) keep 8-byte copies.
static void pad_layout(Task &t) {
  t.sy = t.sz = 0;
  if (t.kind != KIND_FUSED || t.W != 1 || t.bj < 0 || t.aligned || t.A <= 1) return;
  static const bool no_pad = tuning_env("SGH_NO_PAD") != nullptr;   // experiment
  if (no_pad) return;
  const int64_t sy = t.A + ((t.A ^ t.Gj) & 1);
  const int64_t ez = t.P / (int64_t(t.A) * t.ej);
  int64_t sz = sy * t.ej;
  if (ez > 1 && ((sz ^ t.Gnext) & 1)) ++sz;
  // one row after the special axis: its pitch is free -- give it the parity of
  // the outer stride OS, so R > 1 units per tile stack at their global phase
  if (ez == 1 && ((sz ^ t.OS) & 1)) ++sz;
  if (ez * sz + 2 > int64_t(kFusedT1) + kFusedT1 / 8) return;   // the SMEM stage: keep 8-byte copies
  t.sy = (int32_t)sy;
  t.sz = (int32_t)sz;
  t.aligned = 1;
}

static bool plan_fused_group(double *grid, const int32_t *levels, int d, int a, int b, Task &t) {
  const int64_t kFusedT = fused_budget();
  int64_t Sa = 1, P = 1, O = g_outer_mult;
  int busy = 0;
  for (int k = 0; k < a; ++k) Sa *= (int64_t(1) << levels[k]) - 1;
  for (int k = a; k < b; ++k) {
    P *= (int64_t(1) << levels[k]) - 1;
    busy += levels[k] > 1;
  }
  for (int k = b; k < d; ++k) O *= (int64_t(1) << levels[k]) - 1;
  if (busy < 2 || b - a > 16) return false;
  std::memset(&t, 0, sizeof t);
  t.bt2 = -1;
  t.grid = grid;
  t.kind = KIND_FUSED;
  t.bj = -1;
  t.m = b - a;
  t.P = (int32_t)std::min<int64_t>(P, INT32_MAX);
  int64_t R = 1;
  for (int k = a; k < b; ++k) {
    t.gl[k - a] = (int8_t)levels[k];
    t.gR[k - a] = (int32_t)R;
    t.fR[k - a] = make_fdiv((uint32_t)R);
    R *= (int64_t(1) << levels[k]) - 1;
  }
  t.base = 0;
  t.S = Sa;
  t.O = O;
  t.l = levels[a];
  if (Sa == 1) {
    const int t1 = fused_budget_w1();
    if (P > t1) return false;
    t.W = 1;
    t.R = (int32_t)(std::max<int64_t>(t1, P) / P);
    t.OS = P;
    t.tiles = (O + t.R - 1) / t.R;
    finish_fused(t);
    return true;
  }
  // widest tile that fits: long contiguous row segments keep DRAM efficient
  int W = 8;
  while (W < fused_wmax() && W < Sa) W <<= 1;
  while (W > 8 && P * (W + 1) > kFusedT + kFusedT / 16) W >>= 1;
  if (P * (W + 1) > kFusedT + kFusedT / 16) return false;
  t.W = W;
  t.R = 1;
  t.OS = P * Sa;
  t.ncb = (Sa + W - 1) / W;
  t.tiles = O * t.ncb;
  finish_fused(t);
  return true;
}

// BLOCKED group [a, b) with special axis j (a <= j < b), column width W (1: the
// group starts at a unit-stride axis).  The other axes of the group hold whole
// poles; axis j is viewed as a pole of level lj at global stride Gj from
// `base`.  While its whole poles do not fit a tile, the tile holds aligned
// blocks of 2^bt points + their end points (the largest bt that fits) and
// writes the blocks' fine points; the coarse lattice {i : 2^bt | i} of axis j
// (level lj - bt, stride 2^bt Gj) is the next view.
// Phases come out in hierarchization order (block tiles, then the lattice
// views); dehierarchization runs them reversed, which requires that no axis
// after j in the group is transformed (the block ends must be final values
// when a block tile reads them).  Returns false if no block of >= 4 points fits.
static bool plan_blocked_group(double *grid, const int32_t *levels, int d, int a, int b, int j, int W,
                               std::vector<Task> &phases, bool inv = false) {
  const int64_t budget = W == 1 ? fused_budget_w1() + fused_budget_w1() / 16 : fused_budget() + fused_budget() / 16;
  if (b - a > 16 || b - a < 2 || levels[j] < 3) return false;
  int64_t Sa = 1, O = g_outer_mult, Prest = 1, A = 1;
  for (int k = 0; k < a; ++k) Sa *= (int64_t(1) << levels[k]) - 1;
  for (int k = b; k < d; ++k) O *= (int64_t(1) << levels[k]) - 1;
  int busy = 0;
  for (int k = a; k < b; ++k) {
    const int64_t nk = (int64_t(1) << levels[k]) - 1;
    busy += levels[k] > 1;
    if (k == j) continue;
    Prest *= nk;
    if (k < j) A *= nk;
  }
  if (busy < 2) return false;
  if ((W == 1) != (Sa == 1)) return false;
  if (W > 1 && W > 2 * Sa && W > 8) return false;
  const int64_t Wf = (W == 1) ? 1 : W + 1;
  const int64_t nj = (int64_t(1) << levels[j]) - 1;
  int64_t G = Sa;                                   // dense global stride of axis j
  for (int k = a; k < j; ++k) G *= (int64_t(1) << levels[k]) - 1;
  const int64_t Gnext = (j + 1 < b) ? G * nj : 0;
  int lj = levels[j];
  int64_t Gj = G, base = 0;
  const size_t first = phases.size();
  for (int step = 0;; ++step) {
    const int64_t nlj = (int64_t(1) << lj) - 1;
    int bt = lj;                                      // whole poles?
    if (Prest * nlj * Wf > budget) {
      bt = 0;
      while (bt + 1 < lj && Prest * ((int64_t(1) << (bt + 1)) + 1) * Wf <= budget) ++bt;
      if (bt < 2) {
        phases.resize(first);
        return false;
      }
    }
    const bool blocked = bt < lj;
    const int64_t ej = blocked ? (int64_t(1) << bt) + 1 : nlj;
    Task t;
    std::memset(&t, 0, sizeof t);
    t.bt2 = -1;
    t.grid = grid;
    t.kind = KIND_FUSED;
    t.m = b - a;
    int64_t R = 1;
    for (int k = a; k < b; ++k) {
      t.gl[k - a] = (int8_t)(k == j ? lj : levels[k]);
      t.gR[k - a] = (int32_t)R;
      t.fR[k - a] = make_fdiv((uint32_t)R);
      R *= (k == j) ? ej : (int64_t(1) << levels[k]) - 1;
    }
    t.P = (int32_t)R;
    t.S = Sa;
    t.O = O;
    t.OS = Prest * nj * Sa;                           // the group's dense extent
    t.base = base;
    t.l = levels[a];
    t.W = W;
    t.R = 1;
    t.bj = j - a;
    t.bt = blocked ? bt : lj;
    t.nb_log = blocked ? lj - bt : 0;
    t.A = (int32_t)A;
    t.ej = (int32_t)ej;
    t.fA = make_fdiv((uint32_t)A);
    t.fE = make_fdiv((uint32_t)ej);
    t.Gj = Gj;
    t.Gnext = Gnext;
    // 16-byte copies need the global 8-byte phase of every tile row (element)
    // to follow the SMEM one: rows x + A (y + ej z) at x S + y Gj + z Gnext with
    // S, A odd (products of odd extents) -> Gj odd and Gnext = ej (mod 2).
    t.aligned = ((Gj & 1) == (A & 1)) && (Gnext == 0 || (Gnext & 1) == ((A * ej) & 1));
    pad_layout(t);
    t.ncb = (W > 1) ? (Sa + W - 1) / W : 1;
    t.tiles = (O << t.nb_log) * t.ncb;
    if (lj <= 1 && busy - (levels[j] > 1) == 0) break;   // nothing left to transform
    if (lj == 1 && b - a == 2 && j == a && Sa == 1 && !inv) {
      // a single lattice point along j and ONE other group axis k: the phase
      // is a plain pole view along k (REG / STRIDED kernels: one thread per
      // column) instead of one FUSED tile per unit (C3's (1, 4) lattice of
      // isolated elements: 3,375 tiles of 15 points)
      const int k = (j == a) ? a + 1 : a;
      int64_t Gk = Sa;
      for (int q = a; q < k; ++q) Gk *= (int64_t(1) << levels[q]) - 1;
      if (levels[k] > 1) plan_view(grid, O, t.OS, Gk, Sa, base, levels[k], phases);
      break;
    }
    const int64_t foot = t.sy > 0 ? int64_t(t.P / (t.A * t.ej)) * t.sz : t.P;   // SMEM pitch of a unit
    // (units stack in SMEM at `foot`, in global memory at OS: with 16-byte
    // copies both must have the same 8-byte parity)
    if (!blocked && W == 1 && O > 1 && (!t.aligned || ((foot ^ t.OS) & 1) == 0)) {
      // a coarse-lattice view: R consecutive outer units per tile, as many as
      // the tile budget holds (small lattice tiles are latency-bound)
      const int64_t R = std::min<int64_t>(O, std::max<int64_t>(1, budget / std::max<int64_t>(1, foot)));
      t.R = (int32_t)R;
      t.tiles = (O + R - 1) / R;
    }
    finish_fused(t);
    phases.push_back(t);
    if (!blocked) break;
    base += ((int64_t(1) << bt) - 1) * Gj;            // first lattice point i = 2^bt
    Gj <<= bt;
    lj -= bt;
  }
  return phases.size() > first;
}

// Dehierarchization of a blocked group whose axes after the blocked one (local
// index jb) are transformed too.  The oracle applies D_a, .., D_{b-1} (the
// per-axis inverses) in ascending order, each coarse -> fine.  A block tile's
// D_jb reads the block ends, which must then hold D_a..D_jb but not yet
// D_{jb+1}..: so every lattice phase T_m (m >= 1; hierarchization order
// T_0 = the block tiles, T_1.. the lattice views) is split into T_m^A (axes
// <= jb, run before the tiles, coarse lattices first) and T_m^B (axes > jb,
// run after them).  Execution T_k^A .. T_1^A, T_0, T_1^B .. T_k^B: every point
// sees its axes in ascending order, and D_jb of every level reads final coarser
// ends.  Emitted reversed (the runner reverses dehierarchization phase lists).
static void split_inverse_lattice(std::vector<Task> &bp, int jb) {
  if (bp.size() < 2) return;
  uint32_t upto = 0, after = 0;
  for (int k = 0; k < bp[0].m; ++k) (k <= jb ? upto : after) |= 1u << k;
  std::vector<Task> out;
  for (size_t m = bp.size() - 1; m >= 1; --m) {     // T_k^B .. T_1^B
    Task t = bp[m];
    t.skipmask |= upto;
    out.push_back(t);
  }
  out.push_back(bp[0]);                             // T_0
  for (size_t m = 1; m < bp.size(); ++m) {          // T_1^A .. T_k^A
    Task t = bp[m];
    t.skipmask |= after;
    out.push_back(t);
  }
  bp.swap(out);
}

// Only the FINE part of a pole view w.r.t. block level tb (the points with
// tz(i) < tb, each written from its aligned 2^tb block + end points): one
// FLAT_BLOCKS or STRIDED phase, no lattice.  Returns false if no tile fits.
bool plan_view_fine(double *grid, int64_t O, int64_t OS, int64_t PS, int64_t S, int64_t base, int l, int tb,
                    std::vector<Task> &phases) {
  if (l <= 1 || O <= 0 || S <= 0 || tb < 1 || tb >= l) return false;
  Task t;
  std::memset(&t, 0, sizeof t);
  t.bt2 = -1;
  t.grid = grid;
  t.O = O;
  t.OS = OS;
  t.PS = PS;
  t.S = S;
  t.base = base;
  t.l = l;
  t.t = tb;
  t.rlog = l - tb;
  if (PS == S && S < kFlatMaxS && (int64_t(1) << tb) * S <= kFlatT) {
    t.kind = KIND_FLAT_BLOCKS;
    t.fS = make_fdiv((uint32_t)S);
    // consecutive blocks per tile while they fit the FLAT budget (small tb:
    // the two-blocked cross phases, C4's 256-point blocks of single rows)
    int nbl = 0;
    while (nbl < l - tb && (int64_t(2) << (tb + nbl)) * S <= kFlatT) ++nbl;
    t.R = 1 << nbl;
    t.tiles = O << (l - tb - nbl);
    phases.push_back(t);
    return true;
  }
  int W = 256;
  while (W > 32 && S <= W / 2 + W / 4) W >>= 1;
  while (W > 32 && ((int64_t(1) << tb) + 1) * (W + 2) > kStridedTileDoubles) W >>= 1;
  if (((int64_t(1) << tb) + 1) * (W + 2) > kStridedTileDoubles) return false;
  t.kind = KIND_STRIDED;
  t.W = W;
  t.ncb = (S + W - 1) / W;
  t.tiles = (O << (l - tb)) * t.ncb;
  phases.push_back(t);
  return true;
}

// TWO-BLOCKED group (the block scheme for C4): a grid whose only
// non-trivial axes are a and a + 1 (a the unit-stride one).  Hierarchization
// only.  Phases, in order (no phase reads a value an earlier one wrote unless
// it needs exactly that value):
//   0  FUSED tiles of (2^t1 + 1) x (2^t2 + 1) points: the fine-a & fine-b points
//      (axis a fine part, then axis b fine part, both in SMEM);
//   1  fine-a part on the coarse-b rows (reads original coarse-a ends);
//   2  FUSED tiles over the coarse-a columns x one b-block (+ end rows): the
//      whole a-lattice of each row, then the fine-b part; writes the fine-b
//      rows (the end rows are only a halo here);
//   3  the a-lattice on the coarse-b rows (points coarse along both axes),
//      after phases 1 and 2 have read their original values;
//   4  the coarse-b lattice over all columns (level l_b - t2, stride 2^t2 n_a).
// Phases 1-4 move ~2^-t1 + 2^-t2 of the points.  Bitwise equal to Alg. 1: every
// point receives the same operations in the same order (axis a, then b).
// Dehierarchization (inv): the oracle applies H_a^-1 to every point, then
// H_b^-1, each coarse -> fine.  Execution order: (1) the a-lattice of every
// row, (2) the fine-a part of the coarse-b rows, (3) the b-lattice of the
// coarse-b rows -- the coarse-b rows are now final -- (4) the tiles: H_a^-1 on
// their fine-b rows (a-ends: the coarse-a points of those rows, a-inverted by
// (1), not yet b-inverted), then H_b^-1 on the fine-a columns with the final
// b-end rows, written fine along both axes; the tile must not touch its b-end
// rows; (5) the fine-b part of the coarse-a columns (task 2 without its a
// transform).  Every point sees the oracle's operations in its order:
// bitwise.  Phases are emitted so that the runner's reversal for
// dehierarchization yields this order.
static bool plan_two_blocked(double *grid, const int32_t *levels, int d, int a, int t1, int t2,
                             std::vector<Task> &phases, bool inv = false) {
  if (a + 1 >= d) return false;
  for (int k = 0; k < d; ++k)
    if (k != a && k != a + 1 && levels[k] != 1) return false;
  const int la = levels[a], lb = levels[a + 1];
  if (t1 < 2 || t2 < 2 || t1 >= la || t2 >= lb) return false;
  const int64_t na = (int64_t(1) << la) - 1, nb = (int64_t(1) << lb) - 1;
  const int64_t e1 = (int64_t(1) << t1) + 1, e2 = (int64_t(1) << t2) + 1;
  if (e1 * e2 > fused_budget_w1() + fused_budget_w1() / 16) return false;
  const size_t first = phases.size();
  Task t;
  std::memset(&t, 0, sizeof t);
  t.grid = grid;
  t.kind = KIND_FUSED;
  t.m = 2;
  t.gl[0] = (int8_t)la;
  t.gl[1] = (int8_t)lb;
  t.gR[0] = 1;
  t.gR[1] = (int32_t)e1;
  t.fR[0] = make_fdiv(1);
  t.fR[1] = make_fdiv((uint32_t)e1);
  t.P = (int32_t)(e1 * e2);
  t.S = 1;
  t.O = 1;
  t.OS = na * nb;
  t.l = la;
  t.W = 1;
  t.R = 1;
  t.bj = 0;
  t.bt = t1;
  t.nb_log = la - t1;
  t.A = 1;
  t.ej = (int32_t)e1;
  t.fA = make_fdiv(1);
  t.fE = make_fdiv((uint32_t)e1);
  t.Gj = 1;
  t.Gnext = na;
  t.aligned = 1;                                     // Gj = 1, Gnext = n_a and e1 odd
  t.bt2 = t2;
  t.nb2_log = lb - t2;
  t.ncb = 1;
  t.tiles = int64_t(1) << (t.nb_log + t.nb2_log);
  finish_fused(t);
  const int64_t s1 = int64_t(1) << t1, s2 = int64_t(1) << t2;
  const int64_t nla = (int64_t(1) << (la - t1)) - 1;   // coarse-a columns
  if (nla * e2 > fused_budget_w1() + fused_budget_w1() / 16) return false;
  // 2: the coarse-a columns in b-blocks: the whole a-lattice of every row of the
  //    block (its end rows only as halo, not written), then the fine-b part
  Task c = t;
  c.gl[0] = (int8_t)(la - t1);
  c.gR[1] = (int32_t)nla;
  c.fR[1] = make_fdiv((uint32_t)nla);
  c.P = (int32_t)(nla * e2);
  c.base = s1 - 1;
  c.bt = la - t1;                                    // whole lattice poles (not blocked)
  c.nb_log = 0;
  c.ej = (int32_t)nla;
  c.fE = make_fdiv((uint32_t)nla);
  c.Gj = s1;
  c.aligned = 0;
  c.tiles = int64_t(1) << c.nb2_log;
  finish_fused(c);
  bool ok;
  if (!inv) {
    phases.push_back(t);
    // 1: fine-a part on the coarse-b rows
    ok = plan_view_fine(grid, (int64_t(1) << (lb - t2)) - 1, s2 * na, 1, 1, (s2 - 1) * na, la, t1, phases);
    phases.push_back(c);
    // 3: the a-lattice on the coarse-b rows (the points coarse along both axes)
    plan_view(grid, (int64_t(1) << (lb - t2)) - 1, s2 * na, s1, 1, (s2 - 1) * na + s1 - 1, la - t1, phases);
    // 4: the coarse-b lattice over all columns
    plan_view(grid, 1, 0, s2 * na, na, (s2 - 1) * na, lb - t2, phases);
  } else {                                           // emitted reversed (see above)
    Task c5 = c;
    c5.skipmask = 1u;                                // (5) fine-b of the coarse-a columns only
    phases.push_back(c5);
    phases.push_back(t);                             // (4)
    plan_view(grid, 1, 0, s2 * na, na, (s2 - 1) * na, lb - t2, phases);                           // (3)
    ok = plan_view_fine(grid, (int64_t(1) << (lb - t2)) - 1, s2 * na, 1, 1, (s2 - 1) * na, la, t1, phases);  // (2)
    // (1) the a-lattice: of the coarse-b rows as a view, of the fine-b rows as
    //     task 2's tiles without their b transform (they store the fine-b rows)
    plan_view(grid, (int64_t(1) << (lb - t2)) - 1, s2 * na, s1, 1, (s2 - 1) * na + s1 - 1, la - t1, phases);
    Task c1 = c;
    c1.skipmask = 2u;
    phases.push_back(c1);
  }
  if (!ok) phases.resize(first);
  return ok;
}

static double kind_bw(const Task &t);

// ------------------------------------------- PREFIX TWO-BLOCKED plans (hier)
// Grids with >= 3 non-trivial axes (trivial axes squeezed out: same layout):
// the last two axes a, b are cut into aligned blocks, the axes before them
// (the prefix, P0 points) stay whole poles, and ONE pass of box tiles
// (P0 x (2^ta + 1) x (2^tb + 1) points) writes every point that is fine along
// both (the SURVEY 8(a) a4 block scheme with the prefix axes carried along).
// The rest is partitioned by the set C of blocked axes a point is coarse along;
// class C's tiles hold the coarse lattice (stride 2^t) along the axes in C and
// the same blocks + ends along the others, run the prefix axes, then a, then b
// (the oracle's order: bitwise), and write only the class's points.
// Class C reads original values of the classes containing C only, so running
// the classes by increasing C (main, {a}, {b}, {a,b}) is in-place safe
// (SURVEY H2).  A class whose lattice does not fit a tile is itself a box
// problem with the other axis restricted to its fine points (solve_box,
// recursive).  Hierarchization only: the inverse would need the block ends
// half-transformed (cf. split_inverse_lattice).
struct BoxAxis {
  int l;            // level of the view (n = 2^l - 1 points)
  int64_t G, base;  // global stride of its points and offset of its first point
  int f;            // only points with tz(i) < f are written (f == l: all)
  int T = -1;       // restricted to the aligned super-block r of level T (T == l or < 0: the whole pole;
  int64_t r = 0;    //   halo-sharded plans: the points of one rank's row shard)
};
struct BoxCtx {
  double *grid;
  int np;           // prefix axes (whole poles)
  int8_t pl[16];    // their levels
  int64_t P0;       // their points (odd)
  int64_t budget;   // tile points
  int64_t N;        // grid points
};

static Task box_task(const BoxCtx &c, const BoxAxis &a, int ta, const BoxAxis &b, int tb) {
  Task t;
  std::memset(&t, 0, sizeof t);
  t.grid = c.grid;
  t.kind = KIND_FUSED;
  t.m = c.np + 2;
  int64_t R = 1;
  for (int j = 0; j < c.np; ++j) {
    t.gl[j] = c.pl[j];
    t.gR[j] = (int32_t)R;
    t.fR[j] = make_fdiv((uint32_t)R);
    R *= (int64_t(1) << c.pl[j]) - 1;
  }
  const bool ba = ta < a.l, bb = tb < b.l;
  const int64_t ea = ba ? (int64_t(1) << ta) + 1 : (int64_t(1) << a.l) - 1;
  const int64_t eb = bb ? (int64_t(1) << tb) + 1 : (int64_t(1) << b.l) - 1;
  t.gl[c.np] = (int8_t)a.l;
  t.gR[c.np] = (int32_t)R;
  t.fR[c.np] = make_fdiv((uint32_t)R);
  R *= ea;
  t.gl[c.np + 1] = (int8_t)b.l;
  t.gR[c.np + 1] = (int32_t)R;
  t.fR[c.np + 1] = make_fdiv((uint32_t)R);
  R *= eb;
  t.P = (int32_t)R;
  t.S = 1;
  t.O = 1;
  t.OS = c.N;
  t.base = a.base + b.base;
  t.l = t.gl[0];
  t.W = 1;
  t.R = 1;
  t.bj = c.np;
  t.bt = ba ? ta : a.l;                              // >= gl[bj]: whole (lattice) poles
  t.nb_log = ba ? a.l - ta : 0;
  t.A = (int32_t)c.P0;
  t.ej = (int32_t)ea;
  t.fA = make_fdiv((uint32_t)c.P0);
  t.fE = make_fdiv((uint32_t)ea);
  t.Gj = a.G;
  t.Gnext = b.G;
  t.bt2 = bb ? tb : -1;
  const int Tb = (b.T < 0 || b.T > b.l) ? b.l : b.T;
  t.nb2_log = bb ? Tb - tb : 0;                    // blocks of the (super-block of the) pole
  if (bb && Tb < b.l) {
    t.nb2_tot = b.l - tb;
    t.blk2_0 = b.r << (Tb - tb);
  }
  t.aligned = ((t.Gj & 1) == (t.A & 1)) && ((t.Gnext & 1) == ((int64_t(t.A) * t.ej) & 1));
  pad_layout(t);
  t.ncb = 1;
  t.tiles = int64_t(1) << (t.nb_log + t.nb2_log);
  finish_fused(t);
  return t;
}

// relative time of a phase list (1 = one pass over the grid at 1 TB/s)
static double box_cost(const BoxCtx &c, const std::vector<Task> &ph, size_t from) {
  double cost = 0;
  for (size_t i = from; i < ph.size(); ++i) {
    const double f = task_points(ph[i]) / double(c.N);
    cost += f / (i == 0 ? kind_bw(ph[i]) : 0.7 * kind_bw(ph[i])) + 0.01;
  }
  return cost;
}

// Append the phases of box problem (a, b) to `out` (execution order).  False
// if some class finds no tile that fits within `depth` levels of recursion.
static bool solve_box(const BoxCtx &c, const BoxAxis &a, const BoxAxis &b, int depth, std::vector<Task> &out,
                      bool both_blocked = false) {
  auto options = [](const BoxAxis &x) {
    std::vector<int> o;
    if (x.f < x.l) {                                 // fine-only axis: the given blocks
      o.push_back(x.f);
      if (x.T >= 0 && x.T < x.l)                     // a super-block: smaller blocks + its own lattice
        for (int t = x.f - 1; t >= 2; --t) o.push_back(t);
      return o;
    }
    o.push_back(x.l);                                // whole poles, then blocks large -> small
    for (int t = x.l - 1; t >= 2; --t) o.push_back(t);
    return o;
  };
  auto extent = [](const BoxAxis &x, int t) {
    return t < x.l ? (int64_t(1) << t) + 1 : (int64_t(1) << x.l) - 1;
  };
  double best = 1e30;
  std::vector<Task> bestv;
  for (int ta : options(a)) {
    const int64_t ea = extent(a, ta);
    if (c.P0 * ea > c.budget) continue;
    if (both_blocked && ta == a.l) continue;
    for (int tb : options(b)) {                      // the largest block of b that fits
      if (both_blocked && tb == b.l) continue;
      const int64_t eb = extent(b, tb);
      if (c.P0 * ea * eb > c.budget) continue;
      std::vector<Task> ph{box_task(c, a, ta, b, tb)};
      // a class along an axis: the points coarse w.r.t. the tile's blocks but
      // still to be written (tz < f)
      const bool ca = ta < a.f, cb = tb < b.f;
      bool ok = depth > 0 || !(ca || cb);
      auto lat = [](const BoxAxis &x, int t) {       // the coarse lattice {i : 2^t | i}
        BoxAxis y{x.l - t, x.G << t, x.base + ((int64_t(1) << t) - 1) * x.G, x.f - t};
        y.T = x.T < 0 ? -1 : x.T - t;
        y.r = x.r;
        return y;
      };
      auto fine = [](const BoxAxis &x, int t) {      // only the points fine w.r.t. blocks of level t
        BoxAxis y = x;
        y.f = t;
        return y;
      };
      const BoxAxis al = lat(a, ta), bl = lat(b, tb), af = fine(a, ta), bf = fine(b, tb);
      if (ok && ca) ok = solve_box(c, al, bf, depth - 1, ph);
      if (ok && cb) ok = solve_box(c, af, bl, depth - 1, ph);
      if (ok && ca && cb) ok = solve_box(c, al, bl, depth - 1, ph);
      if (ok) {
        const double cost = box_cost(c, ph, 0);
        if (cost < best) {
          best = cost;
          bestv.swap(ph);
        }
      }
      break;
    }
  }
  if (bestv.empty()) return false;
  out.insert(out.end(), bestv.begin(), bestv.end());
  return true;
}

// force: both blocked axes in blocks at the top level (SGH_FLAG_TWO_BLOCKED, tests)
static bool plan_prefix_two_blocked(double *grid, const int32_t *levels, int d, std::vector<Task> &phases,
                                    bool force = false) {
  int sq[SGH_MAX_D], m = 0;
  for (int k = 0; k < d; ++k)
    if (levels[k] > 1) sq[m++] = levels[k];
  if (m < 3 || sq[m - 2] < 3 || sq[m - 1] < 3) return false;
  BoxCtx c;
  c.grid = grid;
  c.np = m - 2;
  c.P0 = 1;
  for (int j = 0; j < c.np; ++j) {
    c.pl[j] = (int8_t)sq[j];
    c.P0 *= (int64_t(1) << sq[j]) - 1;
  }
  c.budget = fused_budget_w1() + fused_budget_w1() / 16;
  if (c.P0 * 25 > c.budget) return false;            // not even 5 x 5 blocks
  const int64_t na = (int64_t(1) << sq[m - 2]) - 1;
  c.N = c.P0 * na * ((int64_t(1) << sq[m - 1]) - 1);
  const BoxAxis a{sq[m - 2], c.P0, 0, sq[m - 2]};
  const BoxAxis b{sq[m - 1], c.P0 * na, 0, sq[m - 1]};
  const size_t first = phases.size();
  if (!solve_box(c, a, b, 3, phases, force)) {
    phases.resize(first);
    return false;
  }
  return true;
}

// PREFIX TWO-BLOCKED DEHIERARCHIZATION (one level, no recursion): the
// inverse needs, per axis, predecessors that are nodal along that axis and
// the earlier ones but not yet along the later ones.  With C the set of
// blocked axes a point is coarse along, the execution order
//   T^A({a,b})  D_prefix, D_a on the points coarse along both
//   {b}         the class coarse along b, all axes (its a-ends: T^A's output)
//   T^B({a,b})  D_b on the points coarse along both (now final)
//   {a}^A       D_prefix, D_a on the class coarse along a
//   main        the box tiles, all axes: prefix axes skip the a-end rows
//               ({a}^A's output) and the b-end rows (final); D_a skips the
//               b-end rows; D_b reads final b-ends
//   {a}^B       D_b on the class coarse along a (its b-ends are final)
// gives every point D_prefix, D_a, D_b in the oracle's order with the right
// predecessor states (bitwise).  Emitted reversed (the runner reverses
// dehierarchization phase lists).  Every class must fit one tile.
static bool plan_prefix_two_blocked_inv(double *grid, const int32_t *levels, int d, std::vector<Task> &phases) {
  int sq[SGH_MAX_D], m = 0;
  for (int k = 0; k < d; ++k)
    if (levels[k] > 1) sq[m++] = levels[k];
  if (m < 3 || sq[m - 2] < 3 || sq[m - 1] < 3) return false;
  BoxCtx c;
  c.grid = grid;
  c.np = m - 2;
  c.P0 = 1;
  for (int j = 0; j < c.np; ++j) {
    c.pl[j] = (int8_t)sq[j];
    c.P0 *= (int64_t(1) << sq[j]) - 1;
  }
  c.budget = fused_budget_w1() + fused_budget_w1() / 16;
  const int la = sq[m - 2], lb = sq[m - 1];
  const int64_t na = (int64_t(1) << la) - 1;
  c.N = c.P0 * na * ((int64_t(1) << lb) - 1);
  const BoxAxis a{la, c.P0, 0, la}, b{lb, c.P0 * na, 0, lb};
  auto lat = [](const BoxAxis &x, int t) {
    return BoxAxis{x.l - t, x.G << t, x.base + ((int64_t(1) << t) - 1) * x.G, x.l - t};
  };
  const uint32_t pre_a = (1u << (c.np + 1)) - 1, only_b = 1u << (c.np + 1);
  double best = 1e30;
  std::vector<Task> bestv;
  for (int ta = 2; ta < la; ++ta)
    for (int tb = 2; tb < lb; ++tb) {
      const int64_t ea = (int64_t(1) << ta) + 1, eb = (int64_t(1) << tb) + 1;
      const int64_t nla = (int64_t(1) << (la - ta)) - 1, nlb = (int64_t(1) << (lb - tb)) - 1;
      if (c.P0 * ea * eb > c.budget || c.P0 * ea * nlb > c.budget || c.P0 * nla * eb > c.budget ||
          c.P0 * nla * nlb > c.budget)
        continue;
      const BoxAxis al = lat(a, ta), bl = lat(b, tb);
      Task tAB_A = box_task(c, al, al.l, bl, bl.l);
      tAB_A.skipmask = only_b;
      Task tAB_B = box_task(c, al, al.l, bl, bl.l);
      tAB_B.skipmask = pre_a;
      BoxAxis af = a;
      af.f = ta;
      BoxAxis bf = b;
      bf.f = tb;
      Task tB = box_task(c, af, ta, bl, bl.l);
      Task tA_A = box_task(c, al, al.l, bf, tb);
      tA_A.skipmask = only_b;
      Task tA_B = box_task(c, al, al.l, bf, tb);
      tA_B.skipmask = pre_a;
      Task tM = box_task(c, a, ta, b, tb);
      std::vector<Task> ph{tA_B, tM, tA_A, tAB_B, tB, tAB_A};   // reversed execution order
      const double cost = box_cost(c, std::vector<Task>{tM, tA_A, tA_B, tB, tAB_A, tAB_B}, 0);
      if (cost < best) {
        best = cost;
        bestv.swap(ph);
      }
    }
  if (bestv.empty()) return false;
  phases.insert(phases.end(), bestv.begin(), bestv.end());
  return true;
}

// Halo-sharded hierarchization of one rank's row shard as ONE box plan
// (SURVEY 8(f) 1 with the a4 block scheme): the shard holds the aligned
// super-block r (level T) of every x_d pole, its first row and one spare halo
// row after its rows; the prefix axes and the last non-trivial axis a < d - 1
// stay whole / blocked as in plan_prefix_two_blocked, and x_d is cut into
// blocks inside the super-block (+ the super-block's own coarse lattice as
// classes).  The tiles read the shard's first row and the halo row as block
// ends: both must hold ORIGINAL values.  Writes every point of the shard whose
// x_d index is fine w.r.t. T (all rows but row 0 for r >= 1).  Hierarchization
// only.  False if no plan fits.
bool plan_shard_box(double *shard, const int32_t *levels, int d, int T, int64_t r, std::vector<Task> &phases) {
  if (d < 2 || T < 2) return false;
  int sq[SGH_MAX_D], m = 0;
  for (int k = 0; k < d - 1; ++k)
    if (levels[k] > 1) sq[m++] = levels[k];
  if (m < 1) return false;
  BoxCtx c;
  c.grid = shard;
  c.np = m - 1;
  c.P0 = 1;
  for (int j = 0; j < c.np; ++j) {
    c.pl[j] = (int8_t)sq[j];
    c.P0 *= (int64_t(1) << sq[j]) - 1;
  }
  c.budget = fused_budget_w1() + fused_budget_w1() / 16;
  if (c.P0 * 25 > c.budget) return false;
  const int64_t na = (int64_t(1) << sq[m - 1]) - 1;
  const int64_t C = c.P0 * na;
  c.N = C << T;
  const BoxAxis a{sq[m - 1], c.P0, 0, sq[m - 1]};
  const int64_t first = (r == 0) ? 1 : (r << T);    // global 1-based x_d index of shard row 0
  BoxAxis b{levels[d - 1], C, -(first - 1) * C, T};
  b.T = T;
  b.r = r;
  const size_t first_phase = phases.size();
  if (!solve_box(c, a, b, 5, phases)) {
    phases.resize(first_phase);
    return false;
  }
  return true;
}

// Estimated time per point (1 / TB/s) of a pass, from the kernels' measured
// B200 throughput (profiles/r01): wide contiguous tiles stream best, narrow
// column tiles lose DRAM efficiency.
// experiments (-DSGH_TUNING): SGH_BW_SCALE=kind:factor[,kind:factor] scales a
// kind's modelled rate (kinds 0..4; 5 = W > 1 FUSED, 6 = k_fpipe tasks)
static double bw_scale(int k) {
  static double f[8] = {-1};
  if (f[0] < 0) {
    for (double &x : f) x = 1.0;
    if (const char *e = tuning_env("SGH_BW_SCALE")) {
      int kk;
      double v;
      int used = 0;
      while (std::sscanf(e, "%d:%lf%n", &kk, &v, &used) == 2) {
        if (kk >= 0 && kk < 8) f[kk] = v;
        e += used;
        if (*e == ',') ++e;
      }
    }
  }
  return f[k];
}
static double kind_bw_raw(const Task &t);
static double kind_bw(const Task &t) {
  double bw = kind_bw_raw(t);
  if (t.kind == KIND_FUSED && pipe_task(t, true)) return bw * bw_scale(6);
  if (t.kind == KIND_FUSED && t.W > 1) return bw * bw_scale(5);
  return bw * bw_scale(t.kind);
}
static double kind_bw_raw(const Task &t) {
  switch (t.kind) {
    case KIND_FLAT_SLABS:
    case KIND_FLAT_BLOCKS: return 5.6;
    case KIND_REG: return 5.0;
    case KIND_STRIDED: return t.W >= 128 ? 4.8 : (t.W >= 64 ? 4.6 : 3.9);
    case KIND_FUSED: {
      // contiguous run length of the tile's global segments (doubles)
      int64_t run = t.W;
      if (t.W == 1) {
        run = 1 << 20;
        if (t.bj >= 0) run = (t.Gj == t.A) ? int64_t(t.A) * t.ej : t.A;
      }
// runs of 8 doubles (W = 8 column tiles): measured 2.6-2.8 TB/s on k_fused
// in C5's grouped launches (round 2; the r1 table had 2.2) -- with it
// (6,6,5,5), (7,5,5,5), (6,6,6,4) ... fuse their two trailing axes (W = 8)
// instead of two STRIDED passes: C5 1.72 -> 1.68 planned passes, same speed
#ifndef SGH_RUN8_BW
#define SGH_RUN8_BW 2.7
#endif
// ... in tiles of <= 2 axes; a W = 8 tile of many short axes spends its time in
// the barrier-separated per-axis phases: S10's (2,2,2,2,2,2) x 8 tiles ran at
// 1.75 TB/s (profiles/r02, 62.7 vs 68 Gpoints/s with the three-pass plan)
      const double run8 = t.m <= 2 ? SGH_RUN8_BW : t.m == 3 ? 2.2 : 1.75;
      double bw = run >= 256 ? 5.2 : run >= 128 ? 4.6 : run >= 64 ? 4.3 : run >= 32 ? 4.0 : run >= 16 ? 3.3
                : run >= 8 ? run8 : 2.2;
      // two blocked axes: two block transforms per tile (measured on C4's
      // 129 x 65 tiles: 2.84 TB/s with 256-thread CTAs, 3.35 TB/s with the
      // 128-thread ones -- then one round trip + cross phases beats the
      // per-axis pair FLAT_BLOCKS + STRIDED: 169.6 vs 157.7 Gpoints/s)
      if (t.bt2 >= 0 && t.bt < t.gl[t.bj]) {
        // measured (C4): 257 x 33 tiles 4.09 TB/s, 129 x 65 3.35, 257 x 17 3.3
        bw = std::min(bw, t.ej >= 257 ? 4.1 : 3.3);
        if (t.P < (fused_budget_w1() * 3) / 4) bw *= 0.85;
      }
      // (measured: dense W == 1 tiles 4.7 TB/s, blocked W == 1 tiles 3.3 TB/s;
      // feeding those rates into the model made C3 / C5 slower -- 86.2 / 130.3
      // vs 90.1 / 131.2 Gpoints/s -- so the run-length rates above are kept)
      // lattice views: 8-byte copies; single-element runs (a lattice of the
      // contiguous axis) touch one 32-byte sector per point and write partial
      // sectors (measured ~0.3 TB/s algorithmic on C3's (5,4,4) lattice)
      static const bool pad_cost_old = tuning_env("SGH_PAD_COST_OLD") != nullptr;   // experiment
      if (t.bj >= 0 && (!t.aligned || (pad_cost_old && t.sy > 0))) {
        static const double ubw = tuning_env("SGH_UNALIGNED_BW") ? atof(tuning_env("SGH_UNALIGNED_BW")) : 1.5;
        bw = std::min(bw, run <= 1 ? 0.35 : ubw);
      }
#ifndef SGH_COST_R1
      // round 2: tasks on the pipelined bulk-copy kernel k_fpipe run at its
      // measured rates (profiles/r02: C5's contiguous-run tiles 5.3 TB/s, C4's
      // 257 x 33 two-blocked tiles 5.8, C2's 255 x 33 blocked tiles 4.4);
      // W = 1 tiles with runs shorter than 128 doubles stay on k_fused (2.85)
      if (pipe_task(t, true)) {   // the cost model takes the batched (conservative) kernel
        if (t.bt2 >= 0 && t.bt < t.gl[t.bj]) bw = t.ej >= 257 ? 5.6 : 4.5;
        else bw = 5.3;
      } else if (t.W == 1 && t.aligned && run < 128) {
        bw = std::min(bw, 2.9);
      }
#endif
      if (pad_cost_old && t.sy > 0) bw = std::min(bw, 1.5);
      // padded lattice / blocked views run on k_fused in the batched launches
      // at ~1.5 TB/s (small tiles, load -> transform -> store per CTA): half
      // the run-length rate.  C5, one call: scale 1.0 175.5 Gpoints/s at 1.63
      // planned passes (dominant launch 0.77 of the peak), 0.7 175.6 (1.67,
      // 0.79), 0.5 175.6 (1.72, 0.81), 0.35 173.2 (1.76, 0.83)
      static const double pad_scale =
          tuning_env("SGH_PAD_BW_SCALE") ? atof(tuning_env("SGH_PAD_BW_SCALE")) : 0.5;   // tuning override
      if (t.sy > 0) bw *= pad_scale;
      return bw;
    }
    default: return 4.0;
  }
}

static double pass_cost(const std::vector<Task> &phases) {
  double c = 0;
  // the main phase (most points; phases[0] in hierarchization order, but not
  // in the reversed-emitted dehierarchization two-blocked list); the others
  // are charged relative to it
  size_t m0 = 0;
  for (size_t i = 1; i < phases.size(); ++i)
    if (task_points(phases[i]) > task_points(phases[m0])) m0 = i;
  const double ref = phases.empty() ? 1.0 : std::max(1.0, task_points(phases[m0]));
  for (size_t i = 0; i < phases.size(); ++i) {
    const Task &t = phases[i];
    const double bw = kind_bw(t);
    if (i == m0) {
      // (charging blocked tiles for their 2 end rows, 2 / (2^t + 1), was tried:
      // C5 150.3 vs 151.6 Gpoints/s -- not charged)
      c += 1.0 / bw;
    } else if (t.kind == KIND_FUSED) {
      // a lattice view of a blocked group: its share of the points, plus a
      // fixed per-phase cost (a few % of a pass: launch tail, small tiles)
      c += task_points(t) / ref / (0.7 * bw) + 0.01;
    } else if (t.S < 8 && t.PS != t.S) {
      // a view whose elements are isolated (one per 32-byte sector, no two in
      // a row): measured ~0.13 TB/s algorithmic (STRIDED, C4 cross phases)
      c += task_points(t) / ref / 0.15;
    } else if (task_points(t) > 0.01 * ref) {
      // a sizeable later phase of contiguous rows (e.g. the coarse-b rows of a
      // two-blocked plan): half the kernel's streaming rate
      c += task_points(t) / ref / (0.5 * bw);
    } else {
      // later phases are coarse lattices: a small fraction of the points, latency bound
      c += 2.0 * task_points(t) / ref / 1.0;
    }
  }
  return c;
}

// Passes of a whole grid (hierarchization order inside each pass).  Unless
// SGH_FLAG_PER_AXIS, a DP over consecutive axis groups picks the plan of least
// estimated time: a group is either one axis (per-axis kernels), a run of axes
// whose whole poles fit one FUSED tile, or (unless SGH_FLAG_WHOLE_POLES) a run
// with one BLOCKED axis.  The axis order stays 1..d, so the results are
// bitwise equal to the per-axis path.
void plan_grid(double *grid, const int32_t *levels, int d, uint32_t flags, std::vector<std::vector<Task>> &passes) {
  passes.clear();
  const bool fuse = (flags & SGH_FLAG_PER_AXIS) == 0;
  const bool blocked_ok = fuse && (flags & SGH_FLAG_WHOLE_POLES) == 0 && tuning_env("SGH_NO_BLOCKED") == nullptr;
  const bool inv = (flags & SGH_FLAG_DEHIERARCHIZE) != 0;
  const double kInf = 1e30;
  std::vector<double> cost(d + 1, kInf);
  std::vector<int> from(d + 1, -1);
  std::vector<std::vector<Task>> best(d + 1);      // phases of the group ending at j (fused groups)
  cost[0] = 0;
  for (int i = 0; i < d; ++i) {
    if (cost[i] >= kInf) continue;
    std::vector<Task> ph;
    plan_axis(grid, levels, d, i, ph);
    const double c1 = cost[i] + (ph.empty() ? 0.0 : pass_cost(ph));
    if (c1 < cost[i + 1]) {
      cost[i + 1] = c1;
      from[i + 1] = i;
      best[i + 1].clear();
    }
    if (!fuse) continue;
    int64_t Sa = 1;
    for (int k = 0; k < i; ++k) Sa *= (int64_t(1) << levels[k]) - 1;
    Task t;
    for (int j = i + 2; j <= d; ++j) {
      if (plan_fused_group(grid, levels, d, i, j, t)) {
        const double cj = cost[i] + pass_cost(std::vector<Task>{t});
        if (cj < cost[j] - 1e-12) {
          cost[j] = cj;
          from[j] = i;
          best[j] = std::vector<Task>{t};
        }
        continue;                                  // whole poles fit: no blocking needed
      }
      if (!blocked_ok) continue;
      for (int s = i; s < j; ++s) {
        bool later = false;                          // transformed group axes after the blocked one
        for (int k = s + 1; k < j; ++k) later |= levels[k] > 1;
        // dehierarchization with later axes runs the lattice phases twice
        // (split_inverse_lattice); not when they are single-point lattices of the
        // unit-stride axis, columns of isolated elements (C3: 77.9 vs 80.8 Gpoints/s)
        for (int W = (Sa == 1 ? 1 : fused_wmax()); W >= (Sa == 1 ? 1 : 8); W >>= 1) {
          std::vector<Task> bp;
          if (!plan_blocked_group(grid, levels, d, i, j, s, W, bp, inv)) continue;
          if (inv && later && Sa == 1 && s == i && bp.size() >= 2 && bp[1].gl[bp[1].bj] < 2) continue;
          if (inv && later) split_inverse_lattice(bp, s - i);
          const double cj = cost[i] + pass_cost(bp);
          if (cj < cost[j] - 1e-12) {
            cost[j] = cj;
            from[j] = i;
            best[j] = bp;
          }
        }
      }
    }
  }
  // two-blocked plan (grids with exactly two adjacent non-trivial axes)
  if (blocked_ok && g_outer_mult == 1) {
    std::vector<Task> bestp;
    // SGH_FLAG_TWO_BLOCKED: take a two-blocked plan whenever one exists (tests)
    double bc = (flags & SGH_FLAG_TWO_BLOCKED) ? 1e30 : cost[d];
    // SGH_TWO_BLOCKED_T=t1,t2 (experiments): only that pair of block levels
    int ft1 = -1, ft2 = -1;
    if (const char *e = tuning_env("SGH_TWO_BLOCKED_T")) std::sscanf(e, "%d,%d", &ft1, &ft2);
    for (int a = 0; a + 1 < d; ++a)
      for (int t1 = 2; t1 < levels[a]; ++t1)
        for (int t2 = 2; t2 < levels[a + 1]; ++t2) {
          if (ft1 >= 0 && (t1 != ft1 || t2 != ft2)) continue;
          std::vector<Task> ph;
          if (!plan_two_blocked(grid, levels, d, a, t1, t2, ph, inv)) continue;
          const double c = pass_cost(ph);
          if (c < bc - 1e-12) {
            bc = c;
            bestp = ph;
          }
        }
    // prefix two-blocked plan (hierarchization, >= 3 non-trivial axes)
    static const bool no_ptb = tuning_env("SGH_NO_PTB") != nullptr;   // experiment
    if (g_outer_mult == 1 && !no_ptb) {
      std::vector<Task> ph;
      if (inv ? plan_prefix_two_blocked_inv(grid, levels, d, ph)
              : plan_prefix_two_blocked(grid, levels, d, ph, (flags & SGH_FLAG_TWO_BLOCKED) != 0)) {
        const double c = pass_cost(ph);
        if (c < bc - 1e-12) {
          bc = c;
          bestp = ph;
        }
      }
    }
    if (!bestp.empty()) {
      passes.push_back(std::move(bestp));
      return;
    }
  }
  std::vector<int> ends;
  for (int j = d; j > 0; j = from[j]) ends.push_back(j);
  std::reverse(ends.begin(), ends.end());
  for (int j : ends) {
    const int i = from[j];
    std::vector<Task> phases;
    if (j - i == 1 && best[j].empty()) plan_axis(grid, levels, d, i, phases);
    else phases = best[j];
    if (!phases.empty()) passes.push_back(std::move(phases));
  }
}

// plan_grid over `outer` stacked copies of the grid (a row shard of a
// (d+1)-dimensional grid: rows of its last axis, each one d-dimensional grid)
void plan_grid_rows(double *grid, const int32_t *levels, int d, int64_t outer, uint32_t flags,
                    std::vector<std::vector<Task>> &passes) {
  struct Reset {
    ~Reset() { g_outer_mult = 1; }
  } reset;
  g_outer_mult = outer < 1 ? 1 : outer;
  plan_grid(grid, levels, d, flags, passes);
}

// A single grid's coarse-lattice views keep >= 2 tiles per SM of a B200: the
// R units per tile that fill the tiles of a batched launch (many grids) would
// leave SMs idle in a launch of one grid's lattice (C2: 64 tiles of 4 units).
static void single_grid_units(std::vector<std::vector<Task>> &passes) {
  constexpr int64_t kMinTiles = 2 * 148;
  for (auto &ph : passes)
    for (Task &t : ph) {
      if (t.kind != KIND_FUSED || t.W != 1 || t.bj < 0 || t.R <= 1) continue;
      const int64_t R = std::max<int64_t>(1, std::min<int64_t>(t.R, t.O / kMinTiles));
      if (R == t.R) continue;
      t.R = (int32_t)R;
      t.tiles = (t.O + R - 1) / R;
      finish_fused(t);
    }
}

// ------------------------------------------------- pinned staging ring
// Task tables are staged in pinned host memory and copied asynchronously into
// the caller's workspace.  A slot is reused only after its copy has completed.
struct StagingSlot {
  void *host = nullptr;
  size_t cap = 0;
  cudaEvent_t done = nullptr;
  bool pending = false;
};
struct StagingRing {
  StagingSlot slot[4];
  int next = 0;
};
static std::mutex g_ring_mu;
static std::map<int, StagingRing> g_rings;

// copy `bytes` from `src` to device `dst` on `stream` via a pinned slot
sgh_status staged_upload(void *dst, const void *src, size_t bytes, cudaStream_t stream) {
  if (bytes == 0) return SGH_OK;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return cuda_fail(e, "cudaGetDevice");
  std::lock_guard<std::mutex> lk(g_ring_mu);
  StagingRing &ring = g_rings[dev];
  StagingSlot &s = ring.slot[ring.next];
  ring.next = (ring.next + 1) % 4;
  if (s.pending) {
    e = cudaEventSynchronize(s.done);
    if (e != cudaSuccess) return cuda_fail(e, "cudaEventSynchronize(staging)");
    s.pending = false;
  }
  if (!s.done) {
    e = cudaEventCreateWithFlags(&s.done, cudaEventDisableTiming);
    if (e != cudaSuccess) return cuda_fail(e, "cudaEventCreate");
  }
  if (s.cap < bytes) {
    // grow every slot at once (geometrically) so steady-state calls never
    // allocate pinned memory (cudaHostAlloc synchronises and takes ms)
    size_t cap = std::max(bytes * 2, size_t(4) << 20);
    for (StagingSlot &o : ring.slot) {
      if (o.cap >= cap) continue;
      if (o.pending) {
        e = cudaEventSynchronize(o.done);
        if (e != cudaSuccess) return cuda_fail(e, "cudaEventSynchronize(staging)");
        o.pending = false;
      }
      if (o.host) cudaFreeHost(o.host);
      o.host = nullptr;
      o.cap = 0;
      e = cudaHostAlloc(&o.host, cap, cudaHostAllocDefault);
      if (e != cudaSuccess) return cuda_fail(e, "cudaHostAlloc(staging)");
      o.cap = cap;
    }
  }
  std::memcpy(s.host, src, bytes);
  e = cudaMemcpyAsync(dst, s.host, bytes, cudaMemcpyHostToDevice, stream);
  if (e != cudaSuccess) return cuda_fail(e, "cudaMemcpyAsync(task table)");
  e = cudaEventRecord(s.done, stream);
  if (e != cudaSuccess) return cuda_fail(e, "cudaEventRecord(staging)");
  s.pending = true;
  return SGH_OK;
}

// ---------------------------------------------------------- single grid
static sgh_status transform_single(double *grid, const int32_t *levels, int32_t d, const int32_t *axis_order,
                                   uint32_t axis_mask, uint32_t flags, void *stream) {
  int64_t N = 0;
  sgh_status st = validate_levels(levels, d, &N);
  if (st != SGH_OK) return st;
  if (!grid) return invalid("grid is NULL");
  int order[SGH_MAX_D];
  if (axis_order) {
    bool seen[SGH_MAX_D] = {false};
    for (int k = 0; k < d; ++k) {
      if (axis_order[k] < 0 || axis_order[k] >= d || seen[axis_order[k]]) return invalid("axis_order is not a permutation");
      seen[axis_order[k]] = true;
      order[k] = axis_order[k];
    }
  } else {
    for (int k = 0; k < d; ++k) order[k] = k;
  }
  const bool all_axes = (axis_mask == 0) || ((axis_mask & ((d >= 32) ? 0xffffffffu : ((1u << d) - 1))) ==
                                             ((d >= 32) ? 0xffffffffu : ((1u << d) - 1)));
  if (axis_mask == 0) axis_mask = 0xffffffffu;
  if (flags & ~kKnownFlags) return invalid("unknown flags");
  const bool inv = (flags & SGH_FLAG_DEHIERARCHIZE) != 0;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (!axis_order && all_axes) {
    std::vector<std::vector<Task>> passes;
    plan_grid(grid, levels, d, flags, passes);
    single_grid_units(passes);
    for (auto &phases : passes) {
      if (inv) std::reverse(phases.begin(), phases.end());   // coarse lattice first (H2)
      for (const Task &t : phases) {
        cudaError_t e = launch_single(t, inv, s);
        if (e != cudaSuccess) return cuda_fail(e, pipe_task(t) ? "kernel launch (k_fpipe)" : "kernel launch");
        count_launch();
      }
    }
    return SGH_OK;
  }
  std::vector<Task> phases;
  for (int kk = 0; kk < d; ++kk) {
    const int k = order[kk];
    if (!((axis_mask >> k) & 1u)) continue;
    phases.clear();
    plan_axis(grid, levels, d, k, phases);
    if (inv) std::reverse(phases.begin(), phases.end());   // coarse lattice first (H2)
    for (const Task &t : phases) {
      cudaError_t e = launch_single(t, inv, s);
      if (e != cudaSuccess) return cuda_fail(e, "kernel launch");
      count_launch();
    }
  }
  return SGH_OK;
}

// -------------------------------------------------------------- batched
struct Segment {
  int kind, l, w;
  size_t task_off;    // index of first task in the table
  size_t prefix_off;  // index of first prefix entry
  int32_t ntasks;
  int64_t tiles;
  size_t smem;        // max dynamic shared memory over the segment's tasks
  double points;      // points the segment transforms (profiling)
  int variant;        // task_variant of its tasks (3: mixed blocked / lattice)
  bool pipe;          // runs on k_fpipe (pipe_task)
  int stage;          // (round, phase) index: segments of one stage touch disjoint grids
};

struct BatchedPlan {
  std::vector<Task> tasks;
  std::vector<int64_t> prefix;
  std::vector<Segment> segs;
  std::vector<unsigned char> image;   // the device table image (built once per cached plan)
  void *resident_ws = nullptr;        // the workspace this plan's table was last uploaded to
  // the plan's launches captured into a CUDA graph for `graph_ws` on `graph_dev`
  cudaGraphExec_t gexec = nullptr;
  void *graph_ws = nullptr;
  int graph_dev = -1;
  std::mutex graph_mu;
  ~BatchedPlan() {
    if (gexec) cudaGraphExecDestroy(gexec);
  }
  size_t table_bytes() const {
    return (tasks.size() * sizeof(Task) + 255) / 256 * 256 + prefix.size() * sizeof(int64_t);
  }
};

static void build_batched_plan(double *const *grids, const int32_t *levels, int32_t d, int64_t num_grids,
                               uint32_t flags, BatchedPlan &P) {
  const bool inv = (flags & SGH_FLAG_DEHIERARCHIZE) != 0;
  std::vector<std::vector<std::vector<Task>>> all(num_grids);
  size_t rounds = 0;
  for (int64_t g = 0; g < num_grids; ++g) {
    plan_grid(grids ? grids[g] : nullptr, levels + g * d, d, flags, all[g]);
    if (num_grids == 1) single_grid_units(all[g]);
    rounds = std::max(rounds, all[g].size());
  }
  std::vector<std::vector<Task>> per(num_grids);
  int stage = 0;
  for (size_t k = 0; k < rounds; ++k) {
    size_t maxp = 0;
    for (int64_t g = 0; g < num_grids; ++g) {
      per[g].clear();
      if (k < all[g].size()) per[g] = all[g][k];
      if (inv) std::reverse(per[g].begin(), per[g].end());
      maxp = std::max(maxp, per[g].size());
    }
    for (size_t j = 0; j < maxp; ++j, ++stage) {
      // group phase j of all grids by kernel instance (kind, and l for REG)
      // SGH_SPLIT_VARIANTS=1 (profiling): dense / blocked / lattice FUSED tasks in separate launches
      static const bool split = tuning_env("SGH_SPLIT_VARIANTS") != nullptr;
      std::map<std::tuple<int, int, int, int>, std::vector<const Task *>> groups;
      for (int64_t g = 0; g < num_grids; ++g)
        if (j < per[g].size()) {
          const Task &t = per[g][j];
          groups[{t.kind, t.kind == KIND_REG ? t.l : 0, (t.kind == KIND_STRIDED || t.kind == KIND_FUSED) ? t.W : 0,
                  (split ? task_variant(t) : 0) * 2 + (pipe_task(t, num_grids > 1) ? 1 : 0)}]
              .push_back(&t);
        }
      for (auto &kv : groups) {
        Segment sg;
        sg.kind = std::get<0>(kv.first);
        sg.l = std::get<1>(kv.first);
        sg.w = std::get<2>(kv.first);
        sg.task_off = P.tasks.size();
        sg.prefix_off = P.prefix.size();
        sg.ntasks = (int32_t)kv.second.size();
        sg.pipe = (std::get<3>(kv.first) & 1) != 0;
        sg.stage = stage;
        int64_t acc = 0;
        sg.smem = 0;
        sg.points = 0;
        sg.variant = -1;
        for (const Task *t : kv.second) {
          const int v = task_variant(*t);
          sg.variant = (sg.variant < 0 || sg.variant == v) ? v : 3;
          sg.smem = std::max(sg.smem, task_smem(*t));
          sg.points += task_points(*t);
          P.tasks.push_back(*t);
          P.prefix.push_back(acc);
          acc += t->tiles;
        }
        P.prefix.push_back(acc);
        sg.tiles = acc;
        P.segs.push_back(sg);
      }
    }
  }
}

size_t batched_table_bytes(double *const *grids, const int32_t *levels, int32_t d, int64_t num_grids,
                           uint32_t flags) {
  // the size depends on the levels and flags only: cached (the e2e host path
  // asks for every transfer chunk on every call)
  static std::mutex mu;
  static std::map<std::pair<std::vector<int32_t>, uint32_t>, size_t> memo;
  auto key = std::make_pair(std::vector<int32_t>(levels, levels + num_grids * d), (flags & kPlanFlags) | (uint32_t(d) << 24));
  {
    std::lock_guard<std::mutex> lk(mu);
    auto it = memo.find(key);
    if (it != memo.end()) return it->second;
  }
  BatchedPlan P;
  build_batched_plan(grids, levels, d, num_grids, flags & kPlanFlags, P);
  const size_t b = P.segs.empty() ? 0 : P.table_bytes();
  std::lock_guard<std::mutex> lk(mu);
  if (memo.size() > 4096) memo.clear();
  memo.emplace(std::move(key), b);
  return b;
}

static sgh_status validate_batch(double *const *grids, const int32_t *levels, int32_t d, int64_t num_grids,
                                 bool need_grids) {
  if (num_grids < 0) return invalid("num_grids < 0");
  if (num_grids == 0) return SGH_OK;
  if (!levels) return invalid("levels is NULL");
  if (need_grids && !grids) return invalid("grids is NULL");
  for (int64_t g = 0; g < num_grids; ++g) {
    sgh_status st = validate_levels(levels + g * d, d, nullptr);
    if (st != SGH_OK) return st;
    if (need_grids && !grids[g]) return invalid("grids[g] is NULL");
  }
  return SGH_OK;
}

#ifndef SGH_CONCURRENT
#define SGH_CONCURRENT 0
#endif
constexpr bool kConcurrent = SGH_CONCURRENT != 0;

// library-owned streams and events for the concurrent launch of a stage's
// segments (per device, created once)
struct ConcStreams {
  static constexpr size_t kN = 4;
  cudaStream_t st[kN] = {};
  cudaEvent_t fork = nullptr, join[kN] = {};
};
static std::mutex g_conc_mu;
static std::map<int, ConcStreams> g_conc;

#ifndef SGH_GRAPHS
#define SGH_GRAPHS 1
#endif
constexpr bool kGraphs = SGH_GRAPHS != 0;
static std::map<int, cudaStream_t> g_capture;

// a private stream per device to capture a plan's launches on
static sgh_status capture_stream(cudaStream_t &out) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return cuda_fail(e, "cudaGetDevice");
  std::lock_guard<std::mutex> lk(g_conc_mu);
  cudaStream_t &c = g_capture[dev];
  if (!c && (e = cudaStreamCreateWithFlags(&c, cudaStreamNonBlocking)) != cudaSuccess) return cuda_fail(e, "stream");
  out = c;
  return SGH_OK;
}

static sgh_status conc_streams(ConcStreams *&out) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return cuda_fail(e, "cudaGetDevice");
  std::lock_guard<std::mutex> lk(g_conc_mu);
  ConcStreams &c = g_conc[dev];
  if (!c.fork) {
    for (size_t i = 0; i < ConcStreams::kN; ++i) {
      if ((e = cudaStreamCreateWithFlags(&c.st[i], cudaStreamNonBlocking)) != cudaSuccess) return cuda_fail(e, "stream");
      if ((e = cudaEventCreateWithFlags(&c.join[i], cudaEventDisableTiming)) != cudaSuccess) return cuda_fail(e, "event");
    }
    if ((e = cudaEventCreateWithFlags(&c.fork, cudaEventDisableTiming)) != cudaSuccess) return cuda_fail(e, "event");
  }
  out = &c;
  return SGH_OK;
}

sgh_status run_batched(double *const *grids, const int32_t *levels, int32_t d, int64_t num_grids,
                              uint32_t flags, void *workspace, size_t ws_bytes, cudaStream_t s) {
  if (flags & ~kKnownFlags) return invalid("unknown flags");
  sgh_status st = validate_batch(grids, levels, d, num_grids, true);
  if (st != SGH_OK) return st;
  if (num_grids == 0) return SGH_OK;
  const bool inv = (flags & SGH_FLAG_DEHIERARCHIZE) != 0;
  // Plan cache: the combination grids are transformed every iteration of the
  // combination technique with the same pointers and levels, and planning
  // 4,255 grids takes tens of ms of host time -- reuse the plan.  The table is
  // uploaded on every call unless SGH_FLAG_TABLE_RESIDENT says the workspace
  // still holds it.  Up to kCacheMax plans (the e2e host path runs one plan
  // per transfer chunk: ~640 for C5).
  const uint32_t pflags = flags & kPlanFlags;
  constexpr size_t kCacheMax = 2048;
  struct CacheEntry {
    std::vector<int32_t> levels;
    std::vector<double *> grids;
    uint32_t flags;
    int32_t d;
    std::shared_ptr<BatchedPlan> plan;
  };
  static std::mutex cache_mu;
  static std::vector<CacheEntry> cache;            // most recent last, at most 4
  std::shared_ptr<BatchedPlan> plan;
  {
    std::lock_guard<std::mutex> lk(cache_mu);
    for (size_t i = 0; i < cache.size(); ++i) {
      const CacheEntry &c = cache[i];
      if (c.flags == pflags && c.d == d && c.grids.size() == size_t(num_grids) &&
          std::equal(c.grids.begin(), c.grids.end(), grids) &&
          std::equal(c.levels.begin(), c.levels.end(), levels)) {
        plan = c.plan;
        break;
      }
    }
  }
  if (!plan) {
    plan = std::make_shared<BatchedPlan>();
    build_batched_plan(grids, levels, d, num_grids, pflags, *plan);
    CacheEntry c;
    c.levels.assign(levels, levels + num_grids * d);
    c.grids.assign(grids, grids + num_grids);
    c.flags = pflags;
    c.d = d;
    c.plan = plan;
    std::lock_guard<std::mutex> lk(cache_mu);
    cache.push_back(std::move(c));
    if (cache.size() > kCacheMax) cache.erase(cache.begin());
  }
  const BatchedPlan &P = *plan;
  if (P.segs.empty()) return SGH_OK;
  const size_t bytes = P.table_bytes();
  if (!workspace || ws_bytes < bytes || (reinterpret_cast<uintptr_t>(workspace) & 15)) {
    set_error("workspace missing, misaligned or smaller than sgh_batched_workspace_bytes()");
    return SGH_ERR_WORKSPACE;
  }
  const size_t prefix_base = (P.tasks.size() * sizeof(Task) + 255) / 256 * 256;
  if (plan->image.size() != bytes) {
    std::vector<unsigned char> &host = plan->image;
    host.assign(bytes, 0);
    std::memcpy(host.data(), P.tasks.data(), P.tasks.size() * sizeof(Task));
    std::memcpy(host.data() + prefix_base, P.prefix.data(), P.prefix.size() * sizeof(int64_t));
  }
  bool uploaded = false;
  if (!((flags & SGH_FLAG_TABLE_RESIDENT) && plan->resident_ws == workspace)) {
    st = staged_upload(workspace, plan->image.data(), bytes, s);
    if (st != SGH_OK) return st;
    plan->resident_ws = workspace;
    uploaded = true;
  }
  const Task *d_tasks = reinterpret_cast<const Task *>(workspace);
  const int64_t *d_prefix = reinterpret_cast<const int64_t *>(static_cast<unsigned char *>(workspace) + prefix_base);
  auto launch_all = [&](cudaStream_t s) -> sgh_status {
    // The segments of one (round, phase) stage touch disjoint grids: with
    // kConcurrent (-DSGH_CONCURRENT=1), a stage's launches go to library
    // streams forked from and joined back into `s`, so one kernel's tail
    // overlaps the next ones.  Measured slower on C5 (169.2 vs 170-171, dehier
    // 152.9 vs 155.0: the overlapping kernels compete), so off by default.
    ConcStreams *cs = nullptr;
    if (kConcurrent && (st = conc_streams(cs)) != SGH_OK) return st;
    for (size_t a = 0; a < P.segs.size();) {
      size_t b = a + 1;
      while (b < P.segs.size() && P.segs[b].stage == P.segs[a].stage) ++b;
      const bool fork = kConcurrent && b - a > 1;
      if (fork) {
        cudaEventRecord(cs->fork, s);
        for (size_t i = 0; i < b - a && i < ConcStreams::kN; ++i) cudaStreamWaitEvent(cs->st[i], cs->fork, 0);
      }
      for (size_t i = a; i < b; ++i) {
        const Segment &sg = P.segs[i];
        cudaStream_t ls = fork ? cs->st[(i - a) % ConcStreams::kN] : s;
        cudaError_t e = launch_table(sg.kind, sg.l, sg.w, inv, d_tasks + sg.task_off, d_prefix + sg.prefix_off,
                                     sg.ntasks, sg.tiles, sg.smem, sg.points, ls, sg.variant, sg.pipe);
        if (e != cudaSuccess) {
          char where[160];
          std::snprintf(where, sizeof where, "grouped kernel launch (kind %d, W %d, l %d, variant %d, %s, %d tasks)",
                        sg.kind, sg.w, sg.l, sg.variant, sg.pipe ? "k_fpipe" : "k_fused/per-axis", sg.ntasks);
          return cuda_fail(e, where);
        }
        count_launch();
      }
      if (fork) {
        for (size_t i = 0; i < b - a && i < ConcStreams::kN; ++i) {
          cudaEventRecord(cs->join[i], cs->st[i]);
          cudaStreamWaitEvent(s, cs->join[i], 0);
        }
      }
      a = b;
    }
    return SGH_OK;
  };
  // CUDA graph replay (kGraphs): a repeated call on a resident table (the
  // combination technique's every iteration; bench.py's timed steps) replays
  // the plan's ~36 launches as one graph instead of launching them from the
  // host one by one.  The first resident call captures them (on a private
  // stream: capture is not allowed on the legacy default stream) and launches
  // the graph; later ones only launch it.  Not while per-launch profiling is
  // on (those launches carry events).
  if (kGraphs && !prof_active() && (flags & SGH_FLAG_TABLE_RESIDENT) && !uploaded) {
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return cuda_fail(e, "cudaGetDevice");
    std::lock_guard<std::mutex> lk(plan->graph_mu);
    if (!(plan->gexec && plan->graph_ws == workspace && plan->graph_dev == dev)) {
      cudaStream_t cap = nullptr;
      if ((st = capture_stream(cap)) != SGH_OK) return st;
      if ((e = cudaStreamBeginCapture(cap, cudaStreamCaptureModeRelaxed)) != cudaSuccess)
        return cuda_fail(e, "cudaStreamBeginCapture");
      sgh_status lst = launch_all(cap);
      cudaGraph_t g = nullptr;
      e = cudaStreamEndCapture(cap, &g);
      if (lst != SGH_OK) {
        if (g) cudaGraphDestroy(g);
        return lst;
      }
      if (e != cudaSuccess) return cuda_fail(e, "cudaStreamEndCapture");
      cudaGraphExec_t x = nullptr;
      e = cudaGraphInstantiate(&x, g, 0);
      cudaGraphDestroy(g);
      if (e != cudaSuccess) return cuda_fail(e, "cudaGraphInstantiate");
      if (plan->gexec) cudaGraphExecDestroy(plan->gexec);
      plan->gexec = x;
      plan->graph_ws = workspace;
      plan->graph_dev = dev;
    } else {
      count_launch(P.segs.size());
    }
    if ((e = cudaGraphLaunch(plan->gexec, s)) != cudaSuccess) return cuda_fail(e, "cudaGraphLaunch");
    return SGH_OK;
  }
  return launch_all(s);
}

// per-device scratch for single-grid digests (allocated once, not in a hot call)
static std::mutex g_scratch_mu;
static std::map<int, unsigned long long *> g_digest_scratch;

}  // namespace sgh

using namespace sgh;

extern "C" {

int64_t sgh_num_points(const int32_t *levels, int32_t d) {
  int64_t N = 0;
  if (validate_levels(levels, d, &N) != SGH_OK) return -1;
  return N;
}

sgh_status sgh_hierarchize(double *grid, const int32_t *levels, int32_t d, void *stream) {
  return guarded([&]() -> sgh_status {
  return transform_single(grid, levels, d, nullptr, 0u, SGH_FLAG_NONE, stream);
});
}

sgh_status sgh_dehierarchize(double *grid, const int32_t *levels, int32_t d, void *stream) {
  return guarded([&]() -> sgh_status {
  return transform_single(grid, levels, d, nullptr, 0u, SGH_FLAG_DEHIERARCHIZE, stream);
});
}

sgh_status sgh_transform_ex(double *grid, const int32_t *levels, int32_t d, const int32_t *axis_order,
                            uint32_t axis_mask, uint32_t flags, void *stream) {
  return guarded([&]() -> sgh_status {
  return transform_single(grid, levels, d, axis_order, axis_mask, flags, stream);
});
}

sgh_status sgh_hierarchize_ex(double *grid, const int32_t *levels, int32_t d, const int32_t *axis_order,
                              uint32_t flags, void *workspace, size_t ws_bytes, void *stream) {
  (void)workspace;                                 // every single-grid pass runs in place (sgh.h)
  (void)ws_bytes;
  return guarded([&]() -> sgh_status {
  return transform_single(grid, levels, d, axis_order, 0u, flags, stream);
});
}

size_t sgh_workspace_bytes(const int32_t *levels, int32_t d, int64_t num_grids, uint32_t flags) {
  return sgh_batched_workspace_bytes(levels, d, num_grids, flags);
}

sgh_status sgh_dehierarchize_batched(double *const *grids, const int32_t *levels, int32_t d, int64_t num_grids,
                                     uint32_t flags, void *workspace, size_t ws_bytes, void *stream) {
  return sgh_hierarchize_batched(grids, levels, d, num_grids, flags | SGH_FLAG_DEHIERARCHIZE, workspace, ws_bytes,
                                 stream);
}

size_t sgh_batched_workspace_bytes(const int32_t *levels, int32_t d, int64_t num_grids, uint32_t flags) {
  return guarded_value<size_t>(0, [&]() -> size_t {
  if (validate_batch(nullptr, levels, d, num_grids, false) != SGH_OK || num_grids == 0) return 0;
  BatchedPlan P;
  build_batched_plan(nullptr, levels, d, num_grids, flags, P);
  return P.table_bytes();
});
}

sgh_status sgh_hierarchize_batched(double *const *grids, const int32_t *levels, int32_t d, int64_t num_grids,
                                   uint32_t flags, void *workspace, size_t ws_bytes, void *stream) {
  return guarded([&]() -> sgh_status {
  return run_batched(grids, levels, d, num_grids, flags, workspace, ws_bytes, static_cast<cudaStream_t>(stream));
});
}

sgh_status sgh_fill_uniform(double *grid, int64_t n, uint64_t seed, uint64_t grid_id, int64_t index_offset,
                            void *stream) {
  if (n < 0) return invalid("n < 0");
  if (n == 0) return SGH_OK;
  if (!grid) return invalid("grid is NULL");
  FillItem f{grid, n, host_splitmix_finalise(seed ^ host_splitmix_finalise(grid_id)), index_offset};
  cudaError_t e = launch_fill(nullptr, nullptr, 1, f, util_chunks(n), static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(e, "fill launch");
  count_launch();
  return SGH_OK;
}

static sgh_status make_items(double *const *grids, const int64_t *sizes, const uint64_t *grid_ids, int64_t num_grids,
                             uint64_t seed, std::vector<unsigned char> &host, size_t &prefix_base, int64_t &chunks) {
  std::vector<FillItem> items(num_grids);
  std::vector<int64_t> prefix(num_grids + 1);
  int64_t acc = 0;
  for (int64_t g = 0; g < num_grids; ++g) {
    if (!grids[g] || sizes[g] < 0) return invalid("bad grid pointer or size");
    const uint64_t gid = grid_ids ? grid_ids[g] : 0;
    items[g] = FillItem{grids[g], sizes[g], host_splitmix_finalise(seed ^ host_splitmix_finalise(gid)), 0};
    prefix[g] = acc;
    acc += util_chunks(sizes[g]);
  }
  prefix[num_grids] = acc;
  chunks = acc;
  prefix_base = (num_grids * sizeof(FillItem) + 255) / 256 * 256;
  host.assign(prefix_base + (num_grids + 1) * sizeof(int64_t), 0);
  std::memcpy(host.data(), items.data(), num_grids * sizeof(FillItem));
  std::memcpy(host.data() + prefix_base, prefix.data(), (num_grids + 1) * sizeof(int64_t));
  return SGH_OK;
}

sgh_status sgh_fill_uniform_batched(double *const *grids, const int64_t *sizes, const uint64_t *grid_ids,
                                    int64_t num_grids, uint64_t seed, void *workspace, size_t ws_bytes,
                                    void *stream) {
  return guarded([&]() -> sgh_status {
  if (num_grids < 0) return invalid("num_grids < 0");
  if (num_grids == 0) return SGH_OK;
  if (!grids || !sizes) return invalid("grids/sizes is NULL");
  std::vector<unsigned char> host;
  size_t pb = 0;
  int64_t chunks = 0;
  sgh_status st = make_items(grids, sizes, grid_ids, num_grids, seed, host, pb, chunks);
  if (st != SGH_OK) return st;
  if (!workspace || ws_bytes < host.size()) {
    set_error("workspace too small for batched fill");
    return SGH_ERR_WORKSPACE;
  }
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  st = staged_upload(workspace, host.data(), host.size(), s);
  if (st != SGH_OK) return st;
  FillItem dummy{};
  cudaError_t e = launch_fill(reinterpret_cast<const FillItem *>(workspace),
                              reinterpret_cast<const int64_t *>(static_cast<unsigned char *>(workspace) + pb),
                              (int)num_grids, dummy, chunks, s);
  if (e != cudaSuccess) return cuda_fail(e, "batched fill launch");
  count_launch();
  return SGH_OK;
});
}

sgh_status sgh_digest(const double *grid, int64_t n, int64_t index_offset, uint64_t *out_host, void *stream) {
  if (n < 0 || !out_host) return invalid("bad digest arguments");
  if (n == 0) { *out_host = 0; return SGH_OK; }
  if (!grid) return invalid("grid is NULL");
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return cuda_fail(e, "cudaGetDevice");
  unsigned long long *acc = nullptr;
  {
    std::lock_guard<std::mutex> lk(g_scratch_mu);
    auto it = g_digest_scratch.find(dev);
    if (it == g_digest_scratch.end()) {
      e = cudaMalloc(&acc, sizeof(unsigned long long));
      if (e != cudaSuccess) return cuda_fail(e, "cudaMalloc(digest scratch)");
      g_digest_scratch[dev] = acc;
    } else {
      acc = it->second;
    }
  }
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  e = cudaMemsetAsync(acc, 0, sizeof(unsigned long long), s);
  if (e != cudaSuccess) return cuda_fail(e, "cudaMemsetAsync");
  FillItem f{const_cast<double *>(grid), n, 0, index_offset};
  e = launch_digest(nullptr, nullptr, 1, f, util_chunks(n), acc, s);
  if (e != cudaSuccess) return cuda_fail(e, "digest launch");
  count_launch();
  unsigned long long h = 0;
  e = cudaMemcpyAsync(&h, acc, sizeof h, cudaMemcpyDeviceToHost, s);
  if (e != cudaSuccess) return cuda_fail(e, "cudaMemcpyAsync(digest)");
  e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) return cuda_fail(e, "cudaStreamSynchronize(digest)");
  *out_host = h;
  return SGH_OK;
}

sgh_status sgh_digest_batched(double *const *grids, const int64_t *sizes, int64_t num_grids, uint64_t *out_host,
                              void *workspace, size_t ws_bytes, void *stream) {
  return guarded([&]() -> sgh_status {
  if (num_grids < 0) return invalid("num_grids < 0");
  if (num_grids == 0) return SGH_OK;
  if (!grids || !sizes || !out_host) return invalid("NULL argument");
  std::vector<unsigned char> host;
  size_t pb = 0;
  int64_t chunks = 0;
  sgh_status st = make_items(grids, sizes, nullptr, num_grids, 0, host, pb, chunks);
  if (st != SGH_OK) return st;
  const size_t out_off = (host.size() + 255) / 256 * 256;
  const size_t need = out_off + num_grids * sizeof(unsigned long long);
  if (!workspace || ws_bytes < need) {
    set_error("workspace too small for batched digest");
    return SGH_ERR_WORKSPACE;
  }
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  unsigned char *ws = static_cast<unsigned char *>(workspace);
  unsigned long long *d_out = reinterpret_cast<unsigned long long *>(ws + out_off);
  cudaError_t e = cudaMemsetAsync(d_out, 0, num_grids * sizeof(unsigned long long), s);
  if (e != cudaSuccess) return cuda_fail(e, "cudaMemsetAsync");
  st = staged_upload(ws, host.data(), host.size(), s);
  if (st != SGH_OK) return st;
  FillItem dummy{};
  e = launch_digest(reinterpret_cast<const FillItem *>(ws), reinterpret_cast<const int64_t *>(ws + pb),
                    (int)num_grids, dummy, chunks, d_out, s);
  if (e != cudaSuccess) return cuda_fail(e, "batched digest launch");
  count_launch();
  e = cudaMemcpyAsync(out_host, d_out, num_grids * sizeof(unsigned long long), cudaMemcpyDeviceToHost, s);
  if (e != cudaSuccess) return cuda_fail(e, "cudaMemcpyAsync(digests)");
  e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) return cuda_fail(e, "cudaStreamSynchronize(digests)");
  return SGH_OK;
});
}

int64_t sgh_plan_describe(const int32_t *levels, int32_t d, uint32_t flags, char *buf, size_t cap) {
  return guarded_value<int64_t>(-1, [&]() -> int64_t {
  if (validate_levels(levels, d, nullptr) != SGH_OK || (flags & ~kKnownFlags)) return -1;
  std::vector<std::vector<Task>> passes;
  plan_grid(nullptr, levels, d, flags, passes);
  static const char *names[] = {"FLAT_SLABS", "FLAT_BLOCKS", "STRIDED", "REG", "FUSED"};
  std::string out;
  char line[256];
  for (size_t k = 0; k < passes.size(); ++k) {
    std::snprintf(line, sizeof line, "pass %zu:\n", k);
    out += line;
    for (const Task &t : passes[k]) {
      if (t.kind == KIND_FUSED) {
        std::string lv;
        for (int j = 0; j < t.m; ++j) lv += (j ? "," : "") + std::to_string(int(t.gl[j]));
        std::snprintf(line, sizeof line,
                      "  FUSED W=%d levels=(%s) special=%d bt=%d bt2=%d aligned=%d pad=%d skip=%u P=%d R=%d A=%d "
                      "ej=%d runlen=%lld tiles=%lld points=%.0f\n",
                      t.W, lv.c_str(), t.bj, t.bj >= 0 ? t.bt : -1, t.bj >= 0 ? t.bt2 : -1,
                      t.bj >= 0 ? t.aligned : 1, t.sy > 0, t.skipmask, t.P, t.R, t.bj >= 0 ? t.A : 0, t.bj >= 0 ? t.ej : 0,
                      (long long)(t.W > 1 ? t.W : t.bj < 0 ? int64_t(t.R) * t.P : (t.Gj == t.A ? int64_t(t.A) * t.ej : t.A)),
                      (long long)t.tiles, task_points(t));
      } else {
        std::snprintf(line, sizeof line, "  %s l=%d t=%d W=%d points=%.0f\n", names[t.kind], t.l, t.t, t.W,
                      task_points(t));
      }
      out += line;
    }
  }
  if (buf && cap) {
    const size_t n = std::min(cap - 1, out.size());
    std::memcpy(buf, out.data(), n);
    buf[n] = 0;
  }
  return (int64_t)out.size();
});
}

double sgh_plan_cost(const int32_t *levels, int32_t d, uint32_t flags) {
  return guarded_value<double>(-1.0, [&]() -> double {
  int64_t N = 0;
  if (validate_levels(levels, d, &N) != SGH_OK || (flags & ~kKnownFlags)) return -1.0;
  std::vector<std::vector<Task>> passes;
  plan_grid(nullptr, levels, d, flags & kPlanFlags, passes);
  double c = 0;
  for (const auto &ph : passes) c += pass_cost(ph);
  return c * double(N) * 16e-3;                       // 16 B per point and pass / (TB/s) -> ns
});
}

uint64_t sgh_launch_count(void) { return g_launches.load(); }

const char *sgh_status_string(sgh_status s) {
  switch (s) {
    case SGH_OK: return "SGH_OK";
    case SGH_ERR_INVALID_ARGUMENT: return "SGH_ERR_INVALID_ARGUMENT";
    case SGH_ERR_CAPACITY: return "SGH_ERR_CAPACITY";
    case SGH_ERR_CUDA: return "SGH_ERR_CUDA";
    case SGH_ERR_NCCL: return "SGH_ERR_NCCL";
    case SGH_ERR_WORKSPACE: return "SGH_ERR_WORKSPACE";
    default: return "SGH_ERR_UNKNOWN";
  }
}

const char *sgh_last_error(void) { return g_last_error.c_str(); }

const char *sgh_version(void) { return "sgh 0.1.0 (sm_100a)"; }

}  // extern "C"
