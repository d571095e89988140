// sgh_sharded.cu -- one grid sharded along its slowest axis x_d over P ranks
// (BASELINE.json north_star: "a single grid too large for one pass is sharded
// along its slowest axis, with the pass along that axis done after an NCCL
// all-to-all re-shard over NVLink").
//
// Poles along axis k are independent (Alg. 1 "for all 1-dim poles"), so
// a row shard of x_d transforms axes 1..d-1 locally.  For the pass along x_d
// the grid is re-sharded into column blocks of the flattened x_1..x_{d-1}
// index: rank q receives from every rank s the block rows(s) x C_q; the blocks
// concatenated in rank order are the row-major slab n_d x |C_q|, whose poles
// along x_d are complete.  After the pass a second all-to-all returns the
// slab rows to their owners.  Every point sees the same per-axis operations in
// the same order as on one GPU, so the result is bitwise identical.
//
// Dyadic row shards (P = 2^p): rank r owns the 1-based x_d indices
// [r 2^{l_d-p}, (r+1) 2^{l_d-p}) intersected with [1, n_d].
#include <cuda_runtime.h>
#include <nccl.h>
#include <nccl_device.h>

#include <algorithm>
#include <cstring>
#include <functional>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/sgh.h"
#include "sgh_common.cuh"
#include "sgh_plan.hpp"

namespace sgh {

struct ShardGeom {
  int P = 1, rank = 0, d = 0;
  int32_t levels[SGH_MAX_D];
  int64_t C = 1;          // columns = prod_{k<d-1} n_k
  int64_t nd = 1;         // n_d
  std::vector<int64_t> row_begin, rows;   // per rank, 0-based rows of x_d
  std::vector<int64_t> col_begin, cols;   // per rank, column blocks
};

static sgh_status shard_rows_impl(const int32_t *levels, int32_t d, int32_t nranks, int32_t rank, int64_t *rb,
                                  int64_t *re) {
  sgh_status st = validate_levels(levels, d, nullptr);
  if (st != SGH_OK) return st;
  if (nranks < 1 || (nranks & (nranks - 1)) || rank < 0 || rank >= nranks)
    return invalid("nranks must be a power of two and 0 <= rank < nranks");
  const int ld = levels[d - 1];
  int p = 0;
  while ((1 << p) < nranks) ++p;
  if (p > ld) return invalid("nranks exceeds 2^{l_d}");
  const int64_t blk = int64_t(1) << (ld - p);
  const int64_t nd = (int64_t(1) << ld) - 1;
  const int64_t lo1 = std::max<int64_t>(int64_t(rank) * blk, 1);          // 1-based
  const int64_t hi1 = std::min<int64_t>((int64_t(rank) + 1) * blk - 1, nd);  // inclusive
  *rb = lo1 - 1;
  *re = hi1;  // exclusive, 0-based
  return SGH_OK;
}

static sgh_status make_geom(const int32_t *levels, int32_t d, int P, int rank, ShardGeom &G) {
  if (d < 2) return invalid("the sharded path needs d >= 2");
  G.P = P;
  G.rank = rank;
  G.d = d;
  for (int k = 0; k < d; ++k) G.levels[k] = levels[k];
  G.C = 1;
  for (int k = 0; k < d - 1; ++k) G.C *= (int64_t(1) << levels[k]) - 1;
  G.nd = (int64_t(1) << levels[d - 1]) - 1;
  G.row_begin.resize(P);
  G.rows.resize(P);
  G.col_begin.resize(P);
  G.cols.resize(P);
  for (int q = 0; q < P; ++q) {
    int64_t b, e;
    sgh_status st = shard_rows_impl(levels, d, P, q, &b, &e);
    if (st != SGH_OK) return st;
    G.row_begin[q] = b;
    G.rows[q] = e - b;
    G.col_begin[q] = (G.C * q) / P;
    G.cols[q] = (G.C * (q + 1)) / P - G.col_begin[q];
  }
  return SGH_OK;
}

static int64_t max_rows(const ShardGeom &G) { return *std::max_element(G.rows.begin(), G.rows.end()); }
static int64_t max_cols(const ShardGeom &G) { return *std::max_element(G.cols.begin(), G.cols.end()); }

// elements of each of the two staging buffers of one rank
static int64_t stage_elems(const ShardGeom &G) {
  return std::max(max_rows(G) * G.C, G.nd * max_cols(G));
}

static sgh_status launch_phases(std::vector<Task> &phases, bool inv, cudaStream_t s) {
  if (inv) std::reverse(phases.begin(), phases.end());
  for (const Task &t : phases) {
    cudaError_t e = launch_single(t, inv, s);
    if (e != cudaSuccess) return cuda_fail(e, "kernel launch (sharded)");
    count_launch();
  }
  return SGH_OK;
}

// axes 0..d-2 of a row shard: `rows` stacked (d-1)-dimensional grids, planned
// like one grid (plan_grid_rows: fused / blocked groups, the plan the
// single-grid call takes for the leading axes) -- each point sees axes
// 1..d-1 in order with the oracle's operations
static sgh_status shard_rows_axes(double *shard, const int32_t *levels, int d, int64_t rows, bool inv,
                                  cudaStream_t s) {
  if (rows <= 0) return SGH_OK;
  std::vector<std::vector<Task>> passes;
  plan_grid_rows(shard, levels, d - 1, rows, inv ? uint32_t(SGH_FLAG_DEHIERARCHIZE) : 0u, passes);
  for (auto &ph : passes) {
    sgh_status st = launch_phases(ph, inv, s);
    if (st != SGH_OK) return st;
  }
  return SGH_OK;
}

// step 1: axes 0..d-2 on the local row shard of `rank`
static sgh_status local_axes(double *shard, const ShardGeom &G, int rank, bool inv, cudaStream_t s) {
  return shard_rows_axes(shard, G.levels, G.d, G.rows[rank], inv, s);
}

// pack: shard [rows][C] -> send, block q = [rows][cols_q] at offset rows*col_begin_q
static sgh_status pack(const double *shard, double *send, const ShardGeom &G, int rank, cudaStream_t s) {
  const int64_t R = G.rows[rank];
  for (int q = 0; q < G.P; ++q) {
    if (R == 0 || G.cols[q] == 0) continue;
    cudaError_t e = cudaMemcpy2DAsync(send + R * G.col_begin[q], G.cols[q] * 8, shard + G.col_begin[q], G.C * 8,
                                      G.cols[q] * 8, R, cudaMemcpyDeviceToDevice, s);
    if (e != cudaSuccess) return cuda_fail(e, "pack");
  }
  return SGH_OK;
}

static sgh_status unpack(const double *recv, double *shard, const ShardGeom &G, int rank, cudaStream_t s) {
  const int64_t R = G.rows[rank];
  for (int q = 0; q < G.P; ++q) {
    if (R == 0 || G.cols[q] == 0) continue;
    cudaError_t e = cudaMemcpy2DAsync(shard + G.col_begin[q], G.C * 8, recv + R * G.col_begin[q], G.cols[q] * 8,
                                      G.cols[q] * 8, R, cudaMemcpyDeviceToDevice, s);
    if (e != cudaSuccess) return cuda_fail(e, "unpack");
  }
  return SGH_OK;
}

// step 4: the axis-(d-1) pass on the slab [n_d][cols_rank] of rank `rank`
static sgh_status slab_axis(double *slab, const ShardGeom &G, int rank, bool inv, cudaStream_t s) {
  const int64_t W = G.cols[rank];
  if (W == 0) return SGH_OK;
  std::vector<Task> phases;
  plan_view(slab, 1, G.nd * W, W, W, 0, G.levels[G.d - 1], phases);
  return launch_phases(phases, inv, s);
}

// ---------------------------------------------------------------- NCCL comm
struct Comm {
  ncclComm_t nccl = nullptr;
  int nranks = 1, rank = 0;
  // device-API (LSA) exchange, after sgh_comm_lsa_enable: a symmetric window
  // (every rank's slab) and a device communicator with one LSA barrier per CTA
  bool lsa = false;
  void *win_buf = nullptr;
  size_t win_bytes = 0;
  ncclWindow_t win = nullptr;
  ncclDevComm dev{};
};

static sgh_status nccl_fail(ncclResult_t r, const char *where) {
  set_error(std::string(where) + ": " + ncclGetErrorString(r));
  return SGH_ERR_NCCL;
}

// send[q] block (rows_rank x cols_q) -> recv of q at rows offset; symmetric
static sgh_status exchange_forward(const double *send, double *recv, const ShardGeom &G, Comm *c, cudaStream_t s) {
  const int r = c->rank;
  ncclResult_t nr = ncclGroupStart();
  if (nr != ncclSuccess) return nccl_fail(nr, "ncclGroupStart");
  for (int q = 0; q < G.P; ++q) {
    const size_t scount = size_t(G.rows[r] * G.cols[q]);
    const size_t rcount = size_t(G.rows[q] * G.cols[r]);
    if (scount) {
      nr = ncclSend(send + G.rows[r] * G.col_begin[q], scount, ncclDouble, q, c->nccl, s);
      if (nr != ncclSuccess) { ncclGroupEnd(); return nccl_fail(nr, "ncclSend"); }
    }
    if (rcount) {
      nr = ncclRecv(recv + G.row_begin[q] * G.cols[r], rcount, ncclDouble, q, c->nccl, s);
      if (nr != ncclSuccess) { ncclGroupEnd(); return nccl_fail(nr, "ncclRecv"); }
    }
  }
  nr = ncclGroupEnd();
  if (nr != ncclSuccess) return nccl_fail(nr, "ncclGroupEnd");
  return SGH_OK;
}

static sgh_status exchange_backward(const double *slab, double *recv, const ShardGeom &G, Comm *c, cudaStream_t s) {
  const int r = c->rank;
  ncclResult_t nr = ncclGroupStart();
  if (nr != ncclSuccess) return nccl_fail(nr, "ncclGroupStart");
  for (int q = 0; q < G.P; ++q) {
    const size_t scount = size_t(G.rows[q] * G.cols[r]);
    const size_t rcount = size_t(G.rows[r] * G.cols[q]);
    if (scount) {
      nr = ncclSend(slab + G.row_begin[q] * G.cols[r], scount, ncclDouble, q, c->nccl, s);
      if (nr != ncclSuccess) { ncclGroupEnd(); return nccl_fail(nr, "ncclSend"); }
    }
    if (rcount) {
      nr = ncclRecv(recv + G.rows[r] * G.col_begin[q], rcount, ncclDouble, q, c->nccl, s);
      if (nr != ncclSuccess) { ncclGroupEnd(); return nccl_fail(nr, "ncclRecv"); }
    }
  }
  nr = ncclGroupEnd();
  if (nr != ncclSuccess) return nccl_fail(nr, "ncclGroupEnd");
  return SGH_OK;
}

static sgh_status sharded_nccl(double *shard, const int32_t *levels, int32_t d, void *comm, void *workspace,
                               size_t ws_bytes, void *stream, bool inv) {
  if (!comm) return invalid("comm is NULL");
  Comm *c = static_cast<Comm *>(comm);
  ShardGeom G;
  sgh_status st = validate_levels(levels, d, nullptr);
  if (st != SGH_OK) return st;
  st = make_geom(levels, d, c->nranks, c->rank, G);
  if (st != SGH_OK) return st;
  if (!shard && G.rows[c->rank] > 0) return invalid("shard is NULL");
  const int64_t E = stage_elems(G);
  if (!workspace || ws_bytes < size_t(2 * E * 8)) {
    set_error("workspace smaller than sgh_sharded_workspace_bytes()");
    return SGH_ERR_WORKSPACE;
  }
  double *bufA = static_cast<double *>(workspace);
  double *bufB = bufA + E;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int r = c->rank;
  if ((st = local_axes(shard, G, r, inv, s)) != SGH_OK) return st;
  if ((st = pack(shard, bufA, G, r, s)) != SGH_OK) return st;
  if ((st = exchange_forward(bufA, bufB, G, c, s)) != SGH_OK) return st;
  if ((st = slab_axis(bufB, G, r, inv, s)) != SGH_OK) return st;
  if ((st = exchange_backward(bufB, bufA, G, c, s)) != SGH_OK) return st;
  return unpack(bufA, shard, G, r, s);
}

// ------------------------------------------------------------ loopback (test)
// P virtual ranks on one device; the exchange is a device-to-device copy.
static sgh_status sharded_loopback(double *const *shards, const int32_t *levels, int32_t d, int32_t P,
                                   void *workspace, size_t ws_bytes, void *stream, bool inv) {
  ShardGeom G;
  sgh_status st = validate_levels(levels, d, nullptr);
  if (st != SGH_OK) return st;
  int64_t b, e;
  if ((st = shard_rows_impl(levels, d, P, 0, &b, &e)) != SGH_OK) return st;
  if ((st = make_geom(levels, d, P, 0, G)) != SGH_OK) return st;
  if (!shards) return invalid("shards is NULL");
  const int64_t E = stage_elems(G);
  if (!workspace || ws_bytes < size_t(2 * E * 8) * size_t(P)) {
    set_error("workspace smaller than nranks * sgh_sharded_workspace_bytes()");
    return SGH_ERR_WORKSPACE;
  }
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  double *ws = static_cast<double *>(workspace);
  auto A = [&](int q) { return ws + 2 * E * q; };
  auto Bf = [&](int q) { return ws + 2 * E * q + E; };
  for (int r = 0; r < P; ++r) {
    if (!shards[r] && G.rows[r] > 0) return invalid("shards[r] is NULL");
    if ((st = local_axes(shards[r], G, r, inv, s)) != SGH_OK) return st;
    if ((st = pack(shards[r], A(r), G, r, s)) != SGH_OK) return st;
  }
  for (int r = 0; r < P; ++r)
    for (int q = 0; q < P; ++q) {
      const int64_t cnt = G.rows[r] * G.cols[q];
      if (!cnt) continue;
      cudaError_t ce = cudaMemcpyAsync(Bf(q) + G.row_begin[r] * G.cols[q], A(r) + G.rows[r] * G.col_begin[q], cnt * 8,
                                       cudaMemcpyDeviceToDevice, s);
      if (ce != cudaSuccess) return cuda_fail(ce, "loopback exchange");
    }
  for (int q = 0; q < P; ++q)
    if ((st = slab_axis(Bf(q), G, q, inv, s)) != SGH_OK) return st;
  for (int q = 0; q < P; ++q)
    for (int r = 0; r < P; ++r) {
      const int64_t cnt = G.rows[r] * G.cols[q];
      if (!cnt) continue;
      cudaError_t ce = cudaMemcpyAsync(A(r) + G.rows[r] * G.col_begin[q], Bf(q) + G.row_begin[r] * G.cols[q], cnt * 8,
                                       cudaMemcpyDeviceToDevice, s);
      if (ce != cudaSuccess) return cuda_fail(ce, "loopback exchange back");
    }
  for (int r = 0; r < P; ++r)
    if ((st = unpack(A(r), shards[r], G, r, s)) != SGH_OK) return st;
  return SGH_OK;
}

// ================================================ halo + coarse-lattice path
// SURVEY 8(f) 1, derived from Alg. 1's finest-first order and the
// predecessor rule exactly like a3.iii: with dyadic shards, rank r's
// rows are the aligned super-block [r 2^T, (r+1) 2^T) of the x_d poles
// (T = l_d - p).  Every point of it except its first row has both predecessors
// in [r 2^T, (r+1) 2^T]: the shard plus ONE halo row, the next shard's first
// row.  The first rows {q 2^T : q = 1..P-1} form the coarse lattice, a level-p
// pole per column.  Hierarchization: gather the first rows of all ranks
// (ncclAllGather of C doubles per rank), take the halo from them, transform the
// super-block's interior (block tiles + the super-block's own lattice, all
// restricted to block range r), then hierarchize the gathered coarse rows
// (every rank, redundantly: P - 1 rows) and write back the own first row.
// Dehierarchization: coarse first (gather, dehierarchize, write back own row,
// take the NODAL halo), then the interior coarse -> fine.  Communication per
// rank: C doubles out, P C in, instead of two all-to-alls of ~N/P each.
//
// The shard buffer holds rows [b, e) of x_d and ONE spare row after them (the
// halo slot; its content on return is unspecified).

// Block-restricted plan of the interior of super-block r (block level T) of a
// pole view (global pole indexing through `base`): aligned sub-blocks of the
// largest level a tile holds, then the super-block's own coarse lattice the
// same way, until the lattice inside the super-block is empty.
static bool plan_view_range(double *grid, int64_t O, int64_t OS, int64_t PS, int64_t S, int64_t base, int l, int T,
                            int64_t r, std::vector<Task> &phases) {
  while (T > 0) {
    int t = T;
    std::vector<Task> one;
    while (t > 0 && !(one.clear(), plan_view_fine(grid, O, OS, PS, S, base, l, t, one))) --t;
    if (t == 0) return false;
    Task &k = one.back();
    k.rlog = T - t;                                   // the 2^{T-t} blocks of super-block r
    k.blk0 = r << (T - t);
    if (k.kind == KIND_FLAT_BLOCKS) k.R = 1;          // one block per tile here
    k.tiles = (O << k.rlog) * (k.kind == KIND_STRIDED ? k.ncb : 1);
    phases.push_back(k);
    base += ((int64_t(1) << t) - 1) * PS;             // the lattice {i : 2^t | i}
    PS <<= t;
    l -= t;
    T -= t;
  }
  return true;
}

struct HaloGeom {
  int P = 1, p = 0, d = 0, T = 0;
  int32_t levels[SGH_MAX_D];
  int64_t C = 1;
  std::vector<int64_t> rows;
};

static sgh_status make_halo_geom(const int32_t *levels, int32_t d, int P, HaloGeom &H) {
  if (d < 1) return invalid("d < 1");
  sgh_status st = validate_levels(levels, d, nullptr);
  if (st != SGH_OK) return st;
  if (P < 2 || (P & (P - 1))) return invalid("the halo-sharded path needs nranks = 2^p >= 2");
  H.P = P;
  H.d = d;
  while ((1 << H.p) < P) ++H.p;
  if (H.p > levels[d - 1] - 1) return invalid("nranks must be <= 2^{l_d - 1}");
  H.T = levels[d - 1] - H.p;
  for (int k = 0; k < d; ++k) H.levels[k] = levels[k];
  H.C = 1;
  for (int k = 0; k < d - 1; ++k) H.C *= (int64_t(1) << levels[k]) - 1;
  H.rows.resize(P);
  for (int q = 0; q < P; ++q) {
    int64_t b, e;
    if ((st = shard_rows_impl(levels, d, P, q, &b, &e)) != SGH_OK) return st;
    H.rows[q] = e - b;
  }
  return SGH_OK;
}

// axes 0..d-2 of rank r's shard (rows of x_d as the outer index)
static sgh_status halo_local_axes(double *shard, const HaloGeom &H, int r, bool inv, cudaStream_t s) {
  return shard_rows_axes(shard, H.levels, H.d, H.rows[r], inv, s);
}

// the interior of rank r's super-block along x_d
static sgh_status halo_interior(double *shard, const HaloGeom &H, int r, bool inv, cudaStream_t s) {
  std::vector<Task> phases;
  const int64_t first = (int64_t(r) << H.T);          // global 1-based index of shard row 0 (r >= 1)
  const int64_t base = (r == 0) ? 0 : -(first - 1) * H.C;
  if (!plan_view_range(shard, 1, 0, H.C, H.C, base, H.levels[H.d - 1], H.T, r, phases))
    return invalid("no tile fits the sharded interior pass");
  return launch_phases(phases, inv, s);
}

// the coarse lattice: gathered first rows G[q] (q = 1..P-1) as level-p poles
static sgh_status halo_coarse(double *G, const HaloGeom &H, bool inv, cudaStream_t s) {
  std::vector<Task> phases;
  plan_view(G, 1, 0, H.C, H.C, H.C, H.p, phases);
  return launch_phases(phases, inv, s);
}

static sgh_status d2d(double *dst, const double *src, int64_t n, cudaStream_t s, const char *what) {
  if (n <= 0) return SGH_OK;
  cudaError_t e = cudaMemcpyAsync(dst, src, size_t(n) * 8, cudaMemcpyDeviceToDevice, s);
  return e == cudaSuccess ? SGH_OK : cuda_fail(e, what);
}

// one rank's steps around the gather; `gather` fills G from every rank's row 0
static sgh_status halo_rank_steps(double *shard, double *G, const HaloGeom &H, int r, bool inv, cudaStream_t s,
                                  const std::function<sgh_status()> &gather, bool do_local, bool do_gather) {
  sgh_status st;
  const int64_t C = H.C, R = H.rows[r];
  if (do_local && (st = halo_local_axes(shard, H, r, inv, s)) != SGH_OK) return st;
  if (do_gather && (st = gather()) != SGH_OK) return st;
  if (!inv) {
    if (r + 1 < H.P && (st = d2d(shard + R * C, G + (r + 1) * C, C, s, "halo row")) != SGH_OK) return st;
    if ((st = halo_interior(shard, H, r, false, s)) != SGH_OK) return st;
    if ((st = halo_coarse(G, H, false, s)) != SGH_OK) return st;   // redundant on every rank
    if (r >= 1 && (st = d2d(shard, G + r * C, C, s, "coarse row back")) != SGH_OK) return st;
  } else {
    if ((st = halo_coarse(G, H, true, s)) != SGH_OK) return st;
    if (r >= 1 && (st = d2d(shard, G + r * C, C, s, "coarse row back")) != SGH_OK) return st;
    if (r + 1 < H.P && (st = d2d(shard + R * C, G + (r + 1) * C, C, s, "halo row")) != SGH_OK) return st;
    if ((st = halo_interior(shard, H, r, true, s)) != SGH_OK) return st;
  }
  return SGH_OK;
}

// FUSED hierarchization of rank r's shard (one box plan, plan_shard_box): G
// holds every rank's ORIGINAL first row (gathered before any transform); the
// halo is G[r + 1]; the box plan writes the super-block's interior; the coarse
// rows G[1..P-1] form a grid of levels (l_1..l_{d-1}, p), hierarchized whole
// (every rank, redundantly); rank r >= 1 takes its first row back.  Every
// point sees the oracle's axis order with the oracle's operations:
// bitwise.  Per rank ~1 HBM round trip instead of the two of halo_rank_steps.
static sgh_status halo_fused_hier(double *shard, double *G, const HaloGeom &H, int r, std::vector<Task> &box,
                                  cudaStream_t s) {
  sgh_status st;
  const int64_t C = H.C, R = H.rows[r];
  if (r + 1 < H.P && (st = d2d(shard + R * C, G + (r + 1) * C, C, s, "halo row")) != SGH_OK) return st;
  if ((st = launch_phases(box, false, s)) != SGH_OK) return st;
  int32_t lv[SGH_MAX_D];
  for (int k = 0; k + 1 < H.d; ++k) lv[k] = H.levels[k];
  lv[H.d - 1] = H.p;                                  // the coarse lattice: P - 1 rows
  std::vector<std::vector<Task>> passes;
  plan_grid(G + C, lv, H.d, 0u, passes);
  for (auto &ph : passes)
    if ((st = launch_phases(ph, false, s)) != SGH_OK) return st;
  if (r >= 1 && (st = d2d(shard, G + r * C, C, s, "coarse row back")) != SGH_OK) return st;
  return SGH_OK;
}

static sgh_status sharded_halo_nccl(double *shard, const int32_t *levels, int32_t d, void *comm, void *workspace,
                                    size_t ws_bytes, void *stream, bool inv, bool fused) {
  if (!comm) return invalid("comm is NULL");
  Comm *c = static_cast<Comm *>(comm);
  HaloGeom H;
  sgh_status st = make_halo_geom(levels, d, c->nranks, H);
  if (st != SGH_OK) return st;
  if (!shard) return invalid("shard is NULL");
  if (!workspace || ws_bytes < size_t(H.P * H.C * 8)) {
    set_error("workspace smaller than sgh_sharded_halo_workspace_bytes()");
    return SGH_ERR_WORKSPACE;
  }
  double *G = static_cast<double *>(workspace);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  auto gather = [&]() -> sgh_status {
    ncclResult_t nr = ncclAllGather(shard, G, size_t(H.C), ncclDouble, c->nccl, s);
    return nr == ncclSuccess ? SGH_OK : nccl_fail(nr, "ncclAllGather (coarse rows)");
  };
  // fused or not must be the same decision on every rank (the gather happens
  // at a different point): decided from rank 0's plan, whose tile shapes are
  // every rank's
  std::vector<Task> probe, box;
  if (!inv && fused && plan_shard_box(nullptr, H.levels, H.d, H.T, 0, probe)) {
    if (!plan_shard_box(shard, H.levels, H.d, H.T, c->rank, box))
      return invalid("internal: the fused halo plan of this rank differs from rank 0's");
    if ((st = gather()) != SGH_OK) return st;         // the ORIGINAL first rows
    return halo_fused_hier(shard, G, H, c->rank, box, s);
  }
  return halo_rank_steps(shard, G, H, c->rank, inv, s, gather, true, true);
}

// P virtual ranks on one device (test): the gather is P device copies.
static sgh_status sharded_halo_loopback(double *const *shards, const int32_t *levels, int32_t d, int32_t P,
                                        void *workspace, size_t ws_bytes, void *stream, bool inv, bool fused) {
  HaloGeom H;
  sgh_status st = make_halo_geom(levels, d, P, H);
  if (st != SGH_OK) return st;
  if (!shards) return invalid("shards is NULL");
  for (int r = 0; r < P; ++r)
    if (!shards[r]) return invalid("shards[r] is NULL");
  if (!workspace || ws_bytes < size_t(H.P * H.C * 8) * size_t(P)) {
    set_error("workspace smaller than nranks * sgh_sharded_halo_workspace_bytes()");
    return SGH_ERR_WORKSPACE;
  }
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  double *ws = static_cast<double *>(workspace);
  const int64_t GC = H.P * H.C;
  if (!inv && fused) {
    std::vector<std::vector<Task>> boxes(P);
    bool all = true;
    for (int r = 0; r < P && all; ++r) all = plan_shard_box(shards[r], H.levels, H.d, H.T, r, boxes[r]);
    if (all) {
      for (int r = 0; r < P; ++r)                      // every rank's G = all ORIGINAL first rows
        for (int q = 0; q < P; ++q)
          if ((st = d2d(ws + r * GC + q * H.C, shards[q], H.C, s, "loopback gather")) != SGH_OK) return st;
      for (int r = 0; r < P; ++r)
        if ((st = halo_fused_hier(shards[r], ws + r * GC, H, r, boxes[r], s)) != SGH_OK) return st;
      return SGH_OK;
    }
  }
  for (int r = 0; r < P; ++r)
    if ((st = halo_local_axes(shards[r], H, r, inv, s)) != SGH_OK) return st;
  for (int r = 0; r < P; ++r)                          // every rank's G = all first rows
    for (int q = 0; q < P; ++q)
      if ((st = d2d(ws + r * GC + q * H.C, shards[q], H.C, s, "loopback gather")) != SGH_OK) return st;
  for (int r = 0; r < P; ++r)
    if ((st = halo_rank_steps(shards[r], ws + r * GC, H, r, inv, s, nullptr, false, false)) != SGH_OK) return st;
  return SGH_OK;
}

// ====================================== device-API (LSA) all-to-all re-shard
// the re-shard of the all-to-all path done inside kernels
// over NVLink peer memory (NCCL 2.28 device API, load/store-accessible team)
// instead of pack -> ncclSend/Recv -> unpack.  Every rank's slab n_d x |C_q|
// (the layout the receiver's x_d pass needs, unchanged) lives in a symmetric
// window.  Forward: each rank PUSHES its rows(r) x C_q blocks straight from
// its shard into rank q's window at row offset row_begin(r) -- the pack and
// the exchange are one kernel.  Backward: each rank PULLS rows(r) x C_q from
// every rank q's window into its shard's column block -- the exchange and the
// unpack are one kernel.  Ordering: CTA b of every rank meets CTA b of every
// other rank at an LSA barrier (one per CTA index): push = barrier (no rank
// still reads the windows from a previous call) -> stores -> barrier
// (release: the owner's x_d pass sees them); pull = barrier (acquire: every
// rank's x_d pass is done) -> loads.  The arithmetic (local axes, x_d pass) is
// the same launches as the NCCL path: bitwise.  The loopback variant runs the
// same kernels for P virtual ranks on one device with a table of window
// pointers and no barriers (stream order).
constexpr int kLsaThreads = 512;
constexpr int kLsaMaxCtas = 296;       // LSA barriers requested per communicator
constexpr int kLsaMaxP = 64;

struct ReshardArgs {
  double *shard;                 // [R][C]: read by the push, written by the pull
  int64_t R, C, row_begin;       // this rank's rows of x_d and their global offset
  int P;
  int64_t nch;                   // chunks per (row, column block): ceil(max |C_q| / (kReshardU * kLsaThreads))
  double *peer[kLsaMaxP];        // loopback: every rank's window (LSA: unused)
};

// work items (i, q, k): chunk k (kReshardU * blockDim elements) of segment
// (i, q) = row i of the shard, column block C_q -- contiguous on both sides
// (shard row i, window row row_begin + i of width |C_q|); all of a thread's
// loads are issued before its stores
constexpr int kReshardU = 4;

template <bool PULL>
__device__ __forceinline__ void reshard_items(const ReshardArgs &a, double *const *base) {
  const int64_t ch = int64_t(kReshardU) * blockDim.x;
  const int64_t per_row = int64_t(a.P) * a.nch;
  const int64_t nitems = a.R * per_row;
  for (int64_t g = blockIdx.x; g < nitems; g += gridDim.x) {
    const int64_t i = g / per_row;
    const int64_t rem = g - i * per_row;
    const int q = int(rem / a.nch);
    const int64_t k = rem - int64_t(q) * a.nch;
    const int64_t c0 = a.C * q / a.P, w = a.C * (q + 1) / a.P - c0;
    const int64_t j0 = k * ch;
    if (j0 >= w) continue;
    double *wr = base[q] + (a.row_begin + i) * w + j0;
    double *sh = a.shard + i * a.C + c0 + j0;
    const double *src = PULL ? wr : sh;
    double *dst = PULL ? sh : wr;
    const int64_t n = w - j0 < ch ? w - j0 : ch;
    double v[kReshardU];
#pragma unroll
    for (int u = 0; u < kReshardU; ++u) {
      const int64_t j = threadIdx.x + int64_t(u) * blockDim.x;
      if (j < n) v[u] = src[j];
    }
#pragma unroll
    for (int u = 0; u < kReshardU; ++u) {
      const int64_t j = threadIdx.x + int64_t(u) * blockDim.x;
      if (j < n) dst[j] = v[u];
    }
  }
}

template <bool LSA, bool PULL>
__global__ void __launch_bounds__(kLsaThreads) k_reshard(const __grid_constant__ ReshardArgs a,
                                                         const __grid_constant__ ncclDevComm dc, ncclWindow_t win) {
  __shared__ double *base[kLsaMaxP];
  for (int q = threadIdx.x; q < a.P; q += blockDim.x)
    base[q] = LSA ? static_cast<double *>(ncclGetLsaPointer(win, 0, ncclTeamRankToLsa(dc, ncclTeamWorld(dc), q)))
                  : a.peer[q];
  if constexpr (LSA) {
    ncclLsaBarrierSession<ncclCoopCta> bar(ncclCoopCta(), dc, ncclTeamLsa(dc), dc.lsaBarrier, blockIdx.x);
    bar.sync(ncclCoopCta(), cuda::memory_order_acq_rel);
    __syncthreads();
    // segment (i, q): row i of the shard, column block C_q -- contiguous on
    // both sides (shard row i, window row row_begin + i of width |C_q|)
    reshard_items<PULL>(a, base);
    if (!PULL) bar.sync(ncclCoopCta(), cuda::memory_order_acq_rel);
  } else {
    __syncthreads();
    reshard_items<PULL>(a, base);
  }
}

// the same number of CTAs on every rank (one LSA barrier each), all co-resident
static int lsa_ctas() {
  static int ctas = 0;
  static std::mutex mu;
  std::lock_guard<std::mutex> lk(mu);
  if (!ctas) {
    int dev = 0, sms = 0, occ = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_reshard<true, false>, kLsaThreads, 0);
    ctas = std::max(1, std::min(kLsaMaxCtas, sms * std::max(occ, 1)));
  }
  return ctas;
}

static int64_t lsa_window_elems(const ShardGeom &G) { return G.nd * max_cols(G); }

static sgh_status reshard_launch(bool lsa, bool pull, ReshardArgs a, Comm *c, cudaStream_t s) {
  const int64_t ch = int64_t(kReshardU) * kLsaThreads;
  a.nch = ((a.C + a.P - 1) / a.P + ch - 1) / ch;
  const int grid = lsa ? lsa_ctas() : int(std::min<int64_t>(std::max<int64_t>(a.R * a.P * a.nch, 1), 2 * 148));
  ncclDevComm dc{};
  if (lsa) dc = c->dev;
  ncclWindow_t w = lsa ? c->win : nullptr;
  if (lsa && pull) k_reshard<true, true><<<grid, kLsaThreads, 0, s>>>(a, dc, w);
  else if (lsa) k_reshard<true, false><<<grid, kLsaThreads, 0, s>>>(a, dc, w);
  else if (pull) k_reshard<false, true><<<grid, kLsaThreads, 0, s>>>(a, dc, w);
  else k_reshard<false, false><<<grid, kLsaThreads, 0, s>>>(a, dc, w);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(e, "kernel launch (k_reshard)");
  count_launch();
  return SGH_OK;
}

static sgh_status lsa_enable(Comm *c, size_t bytes) {
  if (c->lsa) return invalid("the device-API exchange is already enabled on this communicator");
  if (c->nranks > kLsaMaxP) return invalid("the device-API exchange supports at most 64 ranks");
  bytes = std::max<size_t>((bytes + 4095) / 4096 * 4096, 4096);
  ncclResult_t r = ncclMemAlloc(&c->win_buf, bytes);
  if (r != ncclSuccess) return nccl_fail(r, "ncclMemAlloc (LSA window)");
  r = ncclCommWindowRegister(c->nccl, c->win_buf, bytes, &c->win, NCCL_WIN_COLL_SYMMETRIC);
  if (r != ncclSuccess) {
    ncclMemFree(c->win_buf);
    c->win_buf = nullptr;
    return nccl_fail(r, "ncclCommWindowRegister");
  }
  ncclDevCommRequirements req;
  std::memset(&req, 0, sizeof req);
  req.lsaBarrierCount = kLsaMaxCtas;
  r = ncclDevCommCreate(c->nccl, &req, &c->dev);
  if (r != ncclSuccess) {
    ncclCommWindowDeregister(c->nccl, c->win);
    ncclMemFree(c->win_buf);
    c->win_buf = nullptr;
    c->win = nullptr;
    return nccl_fail(r, "ncclDevCommCreate");
  }
  if (c->dev.lsaSize != c->nranks) {
    ncclDevCommDestroy(c->nccl, &c->dev);
    ncclCommWindowDeregister(c->nccl, c->win);
    ncclMemFree(c->win_buf);
    c->win_buf = nullptr;
    c->win = nullptr;
    set_error("the load/store-accessible (NVLink) team does not span every rank of the communicator");
    return SGH_ERR_NCCL;
  }
  c->win_bytes = bytes;
  c->lsa = true;
  return SGH_OK;
}

static void lsa_release(Comm *c) {
  if (!c->lsa) return;
  ncclDevCommDestroy(c->nccl, &c->dev);
  ncclCommWindowDeregister(c->nccl, c->win);
  ncclMemFree(c->win_buf);
  c->lsa = false;
  c->win_buf = nullptr;
  c->win = nullptr;
}

static sgh_status sharded_lsa(double *shard, const int32_t *levels, int32_t d, void *comm, void *stream, bool inv) {
  if (!comm) return invalid("comm is NULL");
  Comm *c = static_cast<Comm *>(comm);
  if (!c->lsa) return invalid("sgh_comm_lsa_enable() was not called on this communicator");
  ShardGeom G;
  sgh_status st = validate_levels(levels, d, nullptr);
  if (st != SGH_OK) return st;
  if ((st = make_geom(levels, d, c->nranks, c->rank, G)) != SGH_OK) return st;
  if (!shard && G.rows[c->rank] > 0) return invalid("shard is NULL");
  if (size_t(lsa_window_elems(G)) * 8 > c->win_bytes) {
    set_error("LSA window smaller than sgh_sharded_lsa_window_bytes()");
    return SGH_ERR_WORKSPACE;
  }
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int r = c->rank;
  ReshardArgs a{};
  a.shard = shard;
  a.R = G.rows[r];
  a.C = G.C;
  a.row_begin = G.row_begin[r];
  a.P = G.P;
  if ((st = local_axes(shard, G, r, inv, s)) != SGH_OK) return st;
  if ((st = reshard_launch(true, false, a, c, s)) != SGH_OK) return st;
  if ((st = slab_axis(static_cast<double *>(c->win_buf), G, r, inv, s)) != SGH_OK) return st;
  return reshard_launch(true, true, a, c, s);
}

static sgh_status sharded_lsa_loopback(double *const *shards, const int32_t *levels, int32_t d, int32_t P,
                                       void *workspace, size_t ws_bytes, void *stream, bool inv) {
  ShardGeom G;
  sgh_status st = validate_levels(levels, d, nullptr);
  if (st != SGH_OK) return st;
  int64_t b, e;
  if ((st = shard_rows_impl(levels, d, P, 0, &b, &e)) != SGH_OK) return st;
  if (P > kLsaMaxP) return invalid("the device-API exchange supports at most 64 ranks");
  if ((st = make_geom(levels, d, P, 0, G)) != SGH_OK) return st;
  if (!shards) return invalid("shards is NULL");
  const int64_t E = lsa_window_elems(G);
  if (!workspace || ws_bytes < size_t(E * 8) * size_t(P)) {
    set_error("workspace smaller than nranks * sgh_sharded_lsa_window_bytes()");
    return SGH_ERR_WORKSPACE;
  }
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  double *ws = static_cast<double *>(workspace);
  ReshardArgs a{};
  a.C = G.C;
  a.P = P;
  for (int q = 0; q < P; ++q) a.peer[q] = ws + E * q;
  for (int r = 0; r < P; ++r)
    if (!shards[r] && G.rows[r] > 0) return invalid("shards[r] is NULL");
  for (int r = 0; r < P; ++r) {
    if ((st = local_axes(shards[r], G, r, inv, s)) != SGH_OK) return st;
    a.shard = shards[r];
    a.R = G.rows[r];
    a.row_begin = G.row_begin[r];
    if ((st = reshard_launch(false, false, a, nullptr, s)) != SGH_OK) return st;
  }
  for (int q = 0; q < P; ++q)
    if ((st = slab_axis(a.peer[q], G, q, inv, s)) != SGH_OK) return st;
  for (int r = 0; r < P; ++r) {
    a.shard = shards[r];
    a.R = G.rows[r];
    a.row_begin = G.row_begin[r];
    if ((st = reshard_launch(false, true, a, nullptr, s)) != SGH_OK) return st;
  }
  return SGH_OK;
}

}  // namespace sgh

using namespace sgh;

extern "C" {

sgh_status sgh_shard_rows(const int32_t *levels, int32_t d, int32_t nranks, int32_t rank, int64_t *row_begin,
                          int64_t *row_end) {
  return guarded([&]() -> sgh_status {
  if (!row_begin || !row_end) return invalid("NULL output pointer");
  return shard_rows_impl(levels, d, nranks, rank, row_begin, row_end);
});
}

sgh_status sgh_shard_layout(const int32_t *levels, int32_t d, int32_t nranks, int64_t *row_begin, int64_t *rows,
                            int64_t *col_begin, int64_t *cols) {
  return guarded([&]() -> sgh_status {
  if (!row_begin || !rows || !col_begin || !cols) return invalid("NULL output pointer");
  ShardGeom G;
  sgh_status st = validate_levels(levels, d, nullptr);
  if (st != SGH_OK) return st;
  int64_t b, e;
  if ((st = shard_rows_impl(levels, d, nranks, 0, &b, &e)) != SGH_OK) return st;
  if ((st = make_geom(levels, d, nranks, 0, G)) != SGH_OK) return st;
  for (int q = 0; q < nranks; ++q) {
    row_begin[q] = G.row_begin[q];
    rows[q] = G.rows[q];
    col_begin[q] = G.col_begin[q];
    cols[q] = G.cols[q];
  }
  return SGH_OK;
});
}

double sgh_sharded_plan_bytes(const int32_t *levels, int32_t d, int32_t nranks, int32_t rank, uint32_t flags,
                              int32_t path) {
  return guarded_value<double>(-1.0, [&]() -> double {
  if (flags & ~uint32_t(SGH_FLAG_DEHIERARCHIZE | SGH_FLAG_PER_AXIS)) return -1.0;
  if (rank < 0 || rank >= nranks || (path != 0 && path != 1)) return -1.0;
  const bool inv = (flags & SGH_FLAG_DEHIERARCHIZE) != 0;
  auto points = [](const std::vector<Task> &ph) {
    double p = 0;
    for (const Task &t : ph) p += task_points(t);
    return p;
  };
  double pts = 0;
  std::vector<std::vector<Task>> passes;
  if (path == 0) {
    ShardGeom G;
    int64_t b, e;
    if (validate_levels(levels, d, nullptr) != SGH_OK || shard_rows_impl(levels, d, nranks, 0, &b, &e) != SGH_OK ||
        make_geom(levels, d, nranks, rank, G) != SGH_OK)
      return -1.0;
    plan_grid_rows(nullptr, G.levels, d - 1, G.rows[rank], inv ? uint32_t(SGH_FLAG_DEHIERARCHIZE) : 0u, passes);
    for (const auto &ph : passes) pts += points(ph);
    pts += 2.0 * double(G.rows[rank]) * double(G.C);          // pack + unpack copies
    std::vector<Task> slab;
    if (G.cols[rank] > 0) plan_view(nullptr, 1, G.nd * G.cols[rank], G.cols[rank], G.cols[rank], 0, G.levels[d - 1], slab);
    pts += points(slab);
  } else {
    HaloGeom H;
    if (make_halo_geom(levels, d, nranks, H) != SGH_OK) return -1.0;
    std::vector<Task> box;
    if (!inv && !(flags & SGH_FLAG_PER_AXIS) && plan_shard_box(nullptr, H.levels, d, H.T, rank, box)) {
      pts += points(box);                                     // fused: one box plan over the shard
      int32_t lv[SGH_MAX_D];
      for (int k = 0; k + 1 < d; ++k) lv[k] = H.levels[k];
      lv[d - 1] = H.p;
      plan_grid(nullptr, lv, d, 0u, passes);                  // the coarse rows (redundantly)
      for (const auto &ph : passes) pts += points(ph);
      pts += double(H.C) * ((rank >= 1) + (rank + 1 < H.P));  // halo row in, own coarse row back
      return 16.0 * pts;
    }
    plan_grid_rows(nullptr, H.levels, d - 1, H.rows[rank], inv ? uint32_t(SGH_FLAG_DEHIERARCHIZE) : 0u, passes);
    for (const auto &ph : passes) pts += points(ph);
    std::vector<Task> in;
    if (!plan_view_range(nullptr, 1, 0, H.C, H.C, 0, H.levels[d - 1], H.T, rank, in)) return -1.0;
    for (const Task &t : in)                                  // 2^rlog blocks of 2^t - 1 fine points each
      pts += double(t.O) * double(t.S) * double(int64_t(1) << t.rlog) * double((int64_t(1) << t.t) - 1);
    std::vector<Task> co;
    plan_view(nullptr, 1, 0, H.C, H.C, H.C, H.p, co);
    pts += points(co);
    pts += double(H.C) * ((rank >= 1) + (rank + 1 < H.P));  // halo row in, own coarse row back
  }
  return 16.0 * pts;
});
}

sgh_status sgh_comm_unique_id(void *out) {
  if (!out) return invalid("out is NULL");
  ncclUniqueId id;
  ncclResult_t r = ncclGetUniqueId(&id);
  if (r != ncclSuccess) return nccl_fail(r, "ncclGetUniqueId");
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId is 128 bytes");
  std::memcpy(out, &id, sizeof id);
  return SGH_OK;
}

sgh_status sgh_comm_create(void **comm, const void *nccl_unique_id, int32_t nranks, int32_t rank) {
  return guarded([&]() -> sgh_status {
  if (!comm || !nccl_unique_id) return invalid("NULL argument");
  if (nranks < 1 || rank < 0 || rank >= nranks) return invalid("bad nranks/rank");
  ncclUniqueId id;
  std::memcpy(&id, nccl_unique_id, sizeof id);
  Comm *c = new Comm();
  c->nranks = nranks;
  c->rank = rank;
  ncclResult_t r = ncclCommInitRank(&c->nccl, nranks, id, rank);
  if (r != ncclSuccess) {
    delete c;
    return nccl_fail(r, "ncclCommInitRank");
  }
  *comm = c;
  return SGH_OK;
});
}

void sgh_comm_destroy(void *comm) {
  if (!comm) return;
  Comm *c = static_cast<Comm *>(comm);
  if (c->nccl) lsa_release(c);
  if (c->nccl) ncclCommDestroy(c->nccl);
  delete c;
}

size_t sgh_sharded_workspace_bytes(const int32_t *levels, int32_t d, int32_t nranks) {
  return guarded_value<size_t>(0, [&]() -> size_t {
  ShardGeom G;
  if (validate_levels(levels, d, nullptr) != SGH_OK) return 0;
  int64_t b, e;
  if (shard_rows_impl(levels, d, nranks, 0, &b, &e) != SGH_OK) return 0;
  if (make_geom(levels, d, nranks, 0, G) != SGH_OK) return 0;
  return size_t(2 * stage_elems(G) * 8);
});
}

sgh_status sgh_hierarchize_sharded(double *shard, const int32_t *levels, int32_t d, void *comm, void *workspace,
                                   size_t ws_bytes, void *stream) {
  return guarded([&]() -> sgh_status {
  return sharded_nccl(shard, levels, d, comm, workspace, ws_bytes, stream, false);
});
}

sgh_status sgh_dehierarchize_sharded(double *shard, const int32_t *levels, int32_t d, void *comm, void *workspace,
                                     size_t ws_bytes, void *stream) {
  return guarded([&]() -> sgh_status {
  return sharded_nccl(shard, levels, d, comm, workspace, ws_bytes, stream, true);
});
}

size_t sgh_sharded_halo_workspace_bytes(const int32_t *levels, int32_t d, int32_t nranks) {
  return guarded_value<size_t>(0, [&]() -> size_t {
  HaloGeom H;
  if (make_halo_geom(levels, d, nranks, H) != SGH_OK) return 0;
  return size_t(H.P * H.C * 8);
});
}

sgh_status sgh_transform_sharded_halo(double *shard, const int32_t *levels, int32_t d, void *comm, uint32_t flags,
                                      void *workspace, size_t ws_bytes, void *stream) {
  return guarded([&]() -> sgh_status {
  if (flags & ~uint32_t(SGH_FLAG_DEHIERARCHIZE | SGH_FLAG_PER_AXIS)) return invalid("unknown flags");
  return sharded_halo_nccl(shard, levels, d, comm, workspace, ws_bytes, stream, (flags & SGH_FLAG_DEHIERARCHIZE) != 0,
                           (flags & SGH_FLAG_PER_AXIS) == 0);
});
}

sgh_status sgh_transform_sharded_halo_loopback(double *const *shards, const int32_t *levels, int32_t d,
                                               int32_t nranks, uint32_t flags, void *workspace, size_t ws_bytes,
                                               void *stream) {
  return guarded([&]() -> sgh_status {
  if (flags & ~uint32_t(SGH_FLAG_DEHIERARCHIZE | SGH_FLAG_PER_AXIS)) return invalid("unknown flags");
  return sharded_halo_loopback(shards, levels, d, nranks, workspace, ws_bytes, stream,
                               (flags & SGH_FLAG_DEHIERARCHIZE) != 0, (flags & SGH_FLAG_PER_AXIS) == 0);
});
}

sgh_status sgh_transform_sharded_loopback(double *const *shards, const int32_t *levels, int32_t d, int32_t nranks,
                                          uint32_t flags, void *workspace, size_t ws_bytes, void *stream) {
  return guarded([&]() -> sgh_status {
  if (flags & ~uint32_t(SGH_FLAG_DEHIERARCHIZE)) return invalid("unknown flags");
  return sharded_loopback(shards, levels, d, nranks, workspace, ws_bytes, stream,
                          (flags & SGH_FLAG_DEHIERARCHIZE) != 0);
});
}

sgh_status sgh_comm_lsa_enable(void *comm, size_t window_bytes) {
  return guarded([&]() -> sgh_status {
  if (!comm) return invalid("comm is NULL");
  return lsa_enable(static_cast<Comm *>(comm), window_bytes);
});
}

size_t sgh_sharded_lsa_window_bytes(const int32_t *levels, int32_t d, int32_t nranks) {
  return guarded_value<size_t>(0, [&]() -> size_t {
  ShardGeom G;
  if (validate_levels(levels, d, nullptr) != SGH_OK) return 0;
  int64_t b, e;
  if (shard_rows_impl(levels, d, nranks, 0, &b, &e) != SGH_OK) return 0;
  if (make_geom(levels, d, nranks, 0, G) != SGH_OK) return 0;
  return size_t(lsa_window_elems(G) * 8);
});
}

sgh_status sgh_transform_sharded_lsa(double *shard, const int32_t *levels, int32_t d, void *comm, uint32_t flags,
                                     void *stream) {
  return guarded([&]() -> sgh_status {
  return sharded_lsa(shard, levels, d, comm, stream, (flags & SGH_FLAG_DEHIERARCHIZE) != 0);
});
}

sgh_status sgh_transform_sharded_lsa_loopback(double *const *shards, const int32_t *levels, int32_t d,
                                              int32_t nranks, uint32_t flags, void *workspace, size_t ws_bytes,
                                              void *stream) {
  return guarded([&]() -> sgh_status {
  return sharded_lsa_loopback(shards, levels, d, nranks, workspace, ws_bytes, stream,
                              (flags & SGH_FLAG_DEHIERARCHIZE) != 0);
});
}

}  // extern "C"
