// sgh_common.cuh -- internal types of libsgh (not part of the C ABI).
//
// A hierarchization along one axis of one grid (one iteration of Alg. 1's
// outer loop) is planned as a short list of PHASES.  Each phase is
// a Task: a strided "pole view" of the grid plus the kernel kind that runs it.
//
// Pole view (all offsets in elements):
//   element (o, i, r) with o in [0,O), 1-based pole index i in [1, n], n = 2^l-1,
//   column r in [0,S) lives at   base + o*OS + (i-1)*PS + r.
// The top-level view of axis k is O = prod_{j>k} n_j, S = prod_{j<k} n_j,
// PS = S, OS = n_k*S, base = 0 (row-major, x_1 fastest: P:227).
//
// Long poles are split into aligned blocks of 2^t points (SURVEY 8(a) a3.iii,
// derived from P:127 finest-first and P:140 predecessor rule): a point i with
// tz(i) < t has both predecessors inside [b 2^t, (b+1) 2^t], so a block tile
// with one halo row computes all its fine points.  The remaining "coarse
// lattice" {i : 2^t | i} is itself a level-(l-t) pole view with
//   PS' = 2^t PS,  base' = base + (2^t - 1) PS,
// handled by a later phase (hierarchize) or an earlier one (dehierarchize).
#pragma once
#include <cstdint>

namespace sgh {

constexpr int kThreads = 256;      // every kernel runs 256-thread CTAs
constexpr int kFlatT = 4096;       // FLAT tile: 2^12 elements (32 KB)
constexpr int kFlatMaxS = 64;      // FLAT handles views with S < 64 columns
constexpr int kFlatCap = kFlatT + kFlatMaxS + 2;
constexpr int kStridedWMax = 128;  // STRIDED tile width W in {32, 64, 128} columns
constexpr int kStridedTileDoubles = 8960;  // STRIDED tile budget: (2^t + 1) * (W + 2) doubles (70 KB)
constexpr int kRegMaxL = 4;        // REG kernel: poles of up to 15 points in registers
constexpr int kFusedT = 8192;      // FUSED W > 1 tile budget per pipeline stage (doubles, excl. row padding)
constexpr int kFusedT1 = 8192;     // FUSED W == 1 tile budget (tuning: SGH_FUSED_T1)

enum Kind : int32_t {
  KIND_FLAT_SLABS = 0,   // R whole slabs (o) per tile; needs PS==S, OS==n*S, n*S <= kFlatT
  KIND_FLAT_BLOCKS = 1,  // one 2^t-row block (+halo) of one slab per tile; PS==S, OS==n*S
  KIND_STRIDED = 2,      // (o, block, 32-column group) tiles, any strides
  KIND_REG = 3,          // thread per column, whole pole in registers, l <= kRegMaxL
  KIND_FUSED = 4,        // whole poles of a run of consecutive axes in one tile
  KIND_COUNT = 5
};

// magic-number division for 32-bit numerators < 2^31 (divisor >= 1)
struct FDiv {
  uint32_t d, m, s;
};

inline FDiv make_fdiv(uint32_t d) {
  FDiv f;
  f.d = d;
  uint32_t s = 0;
  while (s < 32 && (1ull << s) < d) ++s;
  f.s = s;
  f.m = (uint32_t)((((1ull << 32) * ((1ull << s) - d)) / d) + 1);
  return f;
}

#ifdef __CUDACC__
__device__ __forceinline__ uint32_t fdiv(uint32_t x, const FDiv &f) {
  return (__umulhi(x, f.m) + x) >> f.s;
}
#endif

struct Task {
  double *grid;
  int64_t O, OS, PS, S, base;
  int64_t tiles;      // CTAs this task needs
  int64_t ncb;        // STRIDED: column groups per (o, block)
  int32_t l;          // pole level (n = 2^l - 1)
  int32_t t;          // block level; t == l means whole poles
  int32_t kind;
  int32_t R;          // FLAT_SLABS: slabs per tile
  int32_t W;          // STRIDED: tile width (columns)
  int32_t rlog;       // FLAT_BLOCKS / STRIDED: the tiles cover 2^rlog consecutive blocks (of level t)
  int64_t blk0;       //   starting at block blk0 (all blocks: rlog = l - t, blk0 = 0; a shard's
                      //   super-block only in the halo-sharded pass)
  FDiv fS;            // division by S   (FLAT kinds, S < 2^31)
  FDiv fNS;           // division by n*S (FLAT_SLABS)
  // FUSED: axes a..a+m-1 of the grid transformed together, whole poles.
  //   W == 1: the group starts at a unit-stride axis; a unit = P contiguous
  //           doubles at base + u*P (O units), a tile = R units.
  //   W  > 1: a unit = (o, column group): P rows of W columns at
  //           base + o*OS + row*S + cb*W + c, ncb column groups.
  // Inside a unit, axis j of the group has row stride gR[j] = prod_{i<j} n_i.
  int32_t m;          // axes in the group
  int32_t P;          // rows per unit = prod of the group's local extents
  int8_t gl[16];      // the group's levels
  int32_t gR[16];     // row strides
  FDiv fR[16];        // division by gR[j]
  // FUSED with a SPECIAL axis bj (bj < 0: none, the group is dense).  The
  // special axis either is BLOCKED (bt < gl[bj]: the tile holds an aligned
  // block of 2^bt points plus its two end points, local y = 0..2^bt at
  // 0-based pole index b 2^bt - 1 + y, and writes only the block's fine points
  // y = 1..2^bt-1) or is a coarse LATTICE (bt >= gl[bj]:
  // whole poles, but with a global stride Gj other than the dense one).  The
  // group axes before bj are dense (row stride S), the ones after it are dense
  // among themselves (the first at stride Gnext).  A tile row r_local =
  // x + A (y + ej z) sits at global offset x S + y Gj + z Gnext.
  int32_t bj;         // special axis (index in the group), -1: none
  int32_t bt;         // its block level (>= gl[bj]: not blocked)
  int32_t nb_log;     // log2(blocks per pole) (0 if not blocked)
  int32_t A;          // tile rows before the special axis (= gR[bj])
  int32_t ej;         // local extent of the special axis (2^bt + 1, or n)
  int32_t aligned;    // 1: global and SMEM 8-byte phases agree row by row (16-byte copies)
  int64_t Gj, Gnext;  // global strides (elements) of the special axis and of the next group axis
  FDiv fA, fE;        // division by A, by ej
  // TWO blocked axes (W == 1 only, SURVEY 8(a) a4 block scheme for C4): the
  // group axis bj + 1 (the last one of the group) is blocked too, with block
  // level bt2 (< 0: not).  The tile holds (2^bt + 1) x (2^bt2 + 1) points and
  // writes the points that are fine along both axes; the rest (the "cross") is
  // done by later phases (planner).
  int32_t bt2;
  int32_t nb2_log;    // log2(blocks of axis bj + 1)
  // Cross phases of a two-blocked group: group axes in skipmask are laid out
  // in the tile but NOT transformed (a pass along the other axis only), and
  // the tile index o may be split into o1 + O1 o2 at o1 OS + o2 OS2 (O1 > 0).
  uint32_t skipmask;
  int32_t O1;
  int64_t OS2;
  // per-axis constants of a FULL tile (R units / one special box), precomputed
  // on the host so a tile needs no integer division: gOk[j] = tile rows /
  // (extent_j gR[j]) (outer pole index count), fNP[j] = division by the
  // number of poles gOk[j] gR[j] W
  int32_t gOk[16];
  FDiv fNP[16];
  // PADDED W == 1 tile layout (sy > 0): SMEM pitches of the special axis' rows
  // and of the rows after it.  A dense tile row r = x + A (y + ej z) sits in
  // SMEM at x + y sy + z sz instead of at r, with sy = parity(Gj) and
  // sz = parity(Gnext) (mod 2): every run of A elements then starts at the
  // 8-byte phase of its global address, so lattice views (Gj even) load and
  // store with 16-byte / bulk copies like dense tiles.  sy == 0: dense.
  int32_t sy, sz;
  // BLOCK RANGE of the second blocked axis (halo-sharded box plans): the
  // tiles cover 2^nb2_log consecutive blocks starting at block blk2_0 of the
  // pole's 2^nb2_tot blocks (nb2_tot == 0: all blocks, blk2_0 = 0)
  int32_t nb2_tot, pad0_;
  int64_t blk2_0;
};

static_assert(sizeof(Task) % 8 == 0, "Task must stay 8-byte aligned");

// harness utilities (fill / digest) work on lists of these
struct FillItem {
  double *ptr;
  int64_t n;
  uint64_t key;          // mix64(seed ^ mix64(grid_id)); unused by the digest
  int64_t index_offset;  // global flat index of ptr[0]
};

}  // namespace sgh
