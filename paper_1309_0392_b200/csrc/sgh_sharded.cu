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

#include <algorithm>
#include <cstring>
#include <functional>
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

// step 1: axes 0..d-2 on the local row shard of `rank`
static sgh_status local_axes(double *shard, const ShardGeom &G, int rank, bool inv, cudaStream_t s) {
  std::vector<Task> phases;
  for (int k = 0; k < G.d - 1; ++k) {
    phases.clear();
    plan_axis(shard, G.levels, G.d, k, phases, G.rows[rank]);
    sgh_status st = launch_phases(phases, inv, s);
    if (st != SGH_OK) return st;
  }
  return SGH_OK;
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

}  // namespace sgh

using namespace sgh;

extern "C" {

sgh_status sgh_shard_rows(const int32_t *levels, int32_t d, int32_t nranks, int32_t rank, int64_t *row_begin,
                          int64_t *row_end) {
  if (!row_begin || !row_end) return invalid("NULL output pointer");
  return shard_rows_impl(levels, d, nranks, rank, row_begin, row_end);
}

sgh_status sgh_shard_layout(const int32_t *levels, int32_t d, int32_t nranks, int64_t *row_begin, int64_t *rows,
                            int64_t *col_begin, int64_t *cols) {
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
}

void sgh_comm_destroy(void *comm) {
  if (!comm) return;
  Comm *c = static_cast<Comm *>(comm);
  if (c->nccl) ncclCommDestroy(c->nccl);
  delete c;
}

size_t sgh_sharded_workspace_bytes(const int32_t *levels, int32_t d, int32_t nranks) {
  ShardGeom G;
  if (validate_levels(levels, d, nullptr) != SGH_OK) return 0;
  int64_t b, e;
  if (shard_rows_impl(levels, d, nranks, 0, &b, &e) != SGH_OK) return 0;
  if (make_geom(levels, d, nranks, 0, G) != SGH_OK) return 0;
  return size_t(2 * stage_elems(G) * 8);
}

sgh_status sgh_hierarchize_sharded(double *shard, const int32_t *levels, int32_t d, void *comm, void *workspace,
                                   size_t ws_bytes, void *stream) {
  return sharded_nccl(shard, levels, d, comm, workspace, ws_bytes, stream, false);
}

sgh_status sgh_dehierarchize_sharded(double *shard, const int32_t *levels, int32_t d, void *comm, void *workspace,
                                     size_t ws_bytes, void *stream) {
  return sharded_nccl(shard, levels, d, comm, workspace, ws_bytes, stream, true);
}

sgh_status sgh_transform_sharded_loopback(double *const *shards, const int32_t *levels, int32_t d, int32_t nranks,
                                          uint32_t flags, void *workspace, size_t ws_bytes, void *stream) {
  if (flags & ~uint32_t(SGH_FLAG_DEHIERARCHIZE)) return invalid("unknown flags");
  return sharded_loopback(shards, levels, d, nranks, workspace, ws_bytes, stream,
                          (flags & SGH_FLAG_DEHIERARCHIZE) != 0);
}

}  // extern "C"
