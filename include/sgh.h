/*
 * sgh.h -- C ABI of libsgh: B200-native (sm_100a) hierarchization of the
 * anisotropic full grids of the sparse grid combination technique
 * (arXiv 1309.0392, "hierarchization ... preprocessing step facilitating the
 * communication").
 *
 * Citation format: P:n = PAPER.md line n, S:n = SPEC.md line n (SPEC is a CPU
 * program spec written from the paper; used for interface conventions only).
 *
 * ---------------------------------------------------------------- layout
 * A grid with level vector l = (l_1..l_d) has n_k = 2^{l_k} - 1 interior
 * points along axis k ("refinement level 1 consist of one single grid
 * point"; zero boundary, not stored).  It is stored as N = prod_k n_k IEEE
 * binary64 values, row-major with x_1 the FASTEST-varying index (P:227
 * "standard row major order", P:236 / P:292).  The point with 1-based
 * per-axis indices (i_1..i_d) lives at flat offset sum_k (i_k - 1) S_k with
 * S_k = prod_{j<k} n_j.  No padding, no alignment requirement beyond 8 bytes.
 *
 * ---------------------------------------------------------------- method
 * Hierarchization (Alg. 1): for k = 1..d in order, every 1-D pole
 * along axis k is transformed, levels l_k down to 2, point i on level lam
 * (i = s(2j+1), s = 2^{l_k - lam}):
 *      x[i] = x[i] - 0.5 * x[i - s];   x[i] = x[i] - 0.5 * x[i + s]
 * where a predecessor on the boundary (i - s = 0 or i + s = 2^{l_k}) is
 * absent and that update is skipped.  Dehierarchization is the inverse
 * base change: levels 2 up to l_k, "+0.5*left then +0.5*right".
 * Results are bitwise identical to the literal Alg. 1 executed on the CPU
 * ("Parity"); the same holds for dehierarchization.
 *
 * ---------------------------------------------------------------- rules
 *  - All grid / workspace / shard pointers are DEVICE pointers owned by the
 *    caller, unless a parameter says "host".  The library never allocates
 *    device memory inside the hot calls.
 *  - `stream` is a cudaStream_t passed as void* (NULL = legacy default stream).
 *    Every call is stream-ordered and asynchronous unless stated otherwise.
 *  - Buffers are modified in place; the caller guarantees exclusive access
 *    until the stream reaches the call.  Grids in one batch must not overlap.
 *  - Arguments are validated before anything is enqueued (all or nothing).
 *    Status codes only; no exception crosses the ABI.  Launch failures return
 *    SGH_ERR_CUDA with the detail in sgh_last_error(); asynchronous device
 *    faults surface at the caller's next synchronisation.
 *  - There is exactly one backend (CUDA, sm_100a).  No CPU fallback: if no
 *    suitable device is present the calls return SGH_ERR_CUDA.
 */
#ifndef SGH_H
#define SGH_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    SGH_OK = 0,
    SGH_ERR_INVALID_ARGUMENT = 1, /* d<1 or d>SGH_MAX_D, l_k<1, NULL pointer, bad permutation, num_grids<0 */
    SGH_ERR_CAPACITY = 2,         /* l_k > SGH_MAX_LEVEL or N*8 overflows int64         */
    SGH_ERR_CUDA = 3,             /* CUDA launch / runtime error; see sgh_last_error()                 */
    SGH_ERR_NCCL = 4,             /* NCCL error in the sharded path                                     */
    SGH_ERR_WORKSPACE = 5         /* workspace NULL or smaller than sgh_*_workspace_bytes()             */
} sgh_status;

#define SGH_MAX_D 16     /* the paper goes up to d = 10 (Fig. fig:10D) */
#define SGH_MAX_LEVEL 30 /* n_k = 2^30 - 1 points on one axis               */

/* flags for the _ex / batched calls */
#define SGH_FLAG_NONE 0u
#define SGH_FLAG_DEHIERARCHIZE 1u /* run the inverse transform instead  */
#define SGH_FLAG_PER_AXIS 2u      /* one HBM round trip per axis: disable the multi-axis
                                     FUSED kernel (a4); results are bitwise identical */
#define SGH_FLAG_WHOLE_POLES 4u   /* fused groups hold whole poles only: no BLOCKED
                                     groups (an axis split into aligned 2^t blocks +
                                     end points, its coarse lattice a later phase;
                                     SURVEY 8(a) a3.iii/a4); results are bitwise identical */
#define SGH_FLAG_TABLE_RESIDENT 64u /* batched calls: the caller asserts that `workspace` still
                                     holds, unmodified, the task table the library wrote there
                                     in its previous batched call with the same grids, levels,
                                     flags and stream; the library then skips the table upload
                                     if that call's plan last uploaded to this workspace */
#define SGH_FLAG_TWO_BLOCKED 32u  /* take the two-blocked plan (two adjacent axes in aligned
                                     blocks + cross phases) wherever one
                                     exists, instead of the cost model's choice: selects a
                                     plan family (tests); results are bitwise identical */

/* ------------------------------------------------------------ geometry */

/* N = prod_k (2^{l_k} - 1).  levels: host array of d int32.
 * Returns -1 if the level vector is invalid or N*8 overflows int64. */
int64_t sgh_num_points(const int32_t *levels, int32_t d);

/* ------------------------------------------------------- single grid */

/* Hierarchize one grid in place (Alg. 1), axes 1..d in order.
 * grid: device pointer to N doubles (layout above).  levels: host int32[d].
 * Needs no workspace: every pass the planner picks (fused multi-axis tiles,
 * blocked and two-blocked groups, per-axis kernels) runs in place. */
sgh_status sgh_hierarchize(double *grid, const int32_t *levels, int32_t d, void *stream);

/* Dehierarchize one grid in place (inverse base change; reading R9). */
sgh_status sgh_dehierarchize(double *grid, const int32_t *levels, int32_t d, void *stream);

/* General single-grid entry.
 *  axis_order: host int32[d], a permutation of 0..d-1 (0-based axes), or NULL
 *              for the paper's order 0..d-1 ("for d <- 1..dim").
 *  axis_mask:  bit k set = transform along axis k; 0 means "all axes".
 *              (Used by the sharded path: local axes only.)
 *  flags:      SGH_FLAG_DEHIERARCHIZE for the inverse.
 * Other orders agree with the paper's only up to rounding (reading R7). */
sgh_status sgh_transform_ex(double *grid, const int32_t *levels, int32_t d,
                            const int32_t *axis_order, uint32_t axis_mask,
                            uint32_t flags, void *stream);

/* The SURVEY 8(b) spelling of the general entry: sgh_transform_ex with all
 * axes (axis_mask 0).  workspace / ws_bytes are accepted and unused (may be
 * NULL / 0): every single-grid plan runs in place. */
sgh_status sgh_hierarchize_ex(double *grid, const int32_t *levels, int32_t d, const int32_t *axis_order,
                              uint32_t flags, void *workspace, size_t ws_bytes, void *stream);

/* ------------------------------------------ batched combination set */

/* Bytes of device workspace the batched calls need for num_grids grids of
 * dimension d (descriptor tables).  levels: host int32[num_grids][d]. */
size_t sgh_batched_workspace_bytes(const int32_t *levels, int32_t d, int64_t num_grids, uint32_t flags);

/* Hierarchize (or, with SGH_FLAG_DEHIERARCHIZE, dehierarchize) num_grids
 * independent grids (the combination grids, "hierarchized in parallel").
 *  grids:     host array of num_grids DEVICE pointers (each N_g doubles).
 *  levels:    host int32[num_grids][d], row-major (grid g's level vector at g*d).
 *  workspace: device buffer of >= sgh_batched_workspace_bytes() bytes, 16-byte
 *             aligned; it holds the per-launch task tables and must not be
 *             reused by the caller until the stream has passed this call.
 * One grouped launch per (axis round, phase, kernel kind) over all grids.
 * Grids of differing d must be padded with trailing level-1 axes. */
sgh_status sgh_hierarchize_batched(double *const *grids, const int32_t *levels, int32_t d,
                                   int64_t num_grids, uint32_t flags,
                                   void *workspace, size_t ws_bytes, void *stream);

/* SURVEY 8(b) spellings: sgh_hierarchize_batched with SGH_FLAG_DEHIERARCHIZE
 * set, and sgh_batched_workspace_bytes. */
sgh_status sgh_dehierarchize_batched(double *const *grids, const int32_t *levels, int32_t d,
                                     int64_t num_grids, uint32_t flags,
                                     void *workspace, size_t ws_bytes, void *stream);
size_t sgh_workspace_bytes(const int32_t *levels, int32_t d, int64_t num_grids, uint32_t flags);

/* Device bytes sgh_transform_batched_host() needs: every grid (256-byte
 * aligned) plus one task table per transfer chunk. */
size_t sgh_batched_host_buffer_bytes(const int32_t *levels, int32_t d, int64_t num_grids, uint32_t flags);

/* End-to-end variant with HOST buffers (the e2e path): host_grids[g] are host
 * pointers (pinned for full PCIe speed), transformed in place.
 * device_buffer: >= sgh_batched_host_buffer_bytes() bytes, 256-byte aligned.
 * Grids are copied in, transformed and copied back in chunks of ~64 MB; the
 * copies run on two library-owned streams overlapped with the transform, and
 * `stream` waits for the last copy-out, so after synchronising `stream` every
 * host grid holds its result.  Mostly asynchronous w.r.t. the host: each
 * chunk's task table goes through a 4-slot pinned staging ring, so with more
 * than 4 chunks the call waits on the host until an earlier chunk's table
 * upload has completed (the call returns while the last chunks are still in
 * flight).  Grids whose host memory is contiguous move with one copy per run
 * in each direction. */
sgh_status sgh_transform_batched_host(double *const *host_grids, const int32_t *levels, int32_t d,
                                      int64_t num_grids, uint32_t flags,
                                      void *device_buffer, size_t device_buffer_bytes,
                                      void *stream);

/* ----------------------------------------------- sharded single grid */

/* Rows [row_begin, row_end) (0-based indices of x_d, the slowest axis) owned
 * by `rank` of `nranks` when one grid is sharded along x_d.  nranks must be a
 * power of two <= n_d + 1; shards are the dyadic blocks
 * [r 2^{l_d - p}, (r+1) 2^{l_d - p}) of 1-based indices intersected with
 * [1, n_d] (so rank 0 holds one row fewer).  Host-only; no device work. */
sgh_status sgh_shard_rows(const int32_t *levels, int32_t d, int32_t nranks, int32_t rank,
                          int64_t *row_begin, int64_t *row_end);

/* The whole exchange plan of the sharded path (host-only): for every rank q,
 * its x_d rows [row_begin[q], row_begin[q]+rows[q]) and its column block
 * [col_begin[q], col_begin[q]+cols[q]) of the flattened x_1..x_{d-1} index
 * (col_begin[q] = floor(q C / P), C = prod_{k<d} n_k).  Forward re-shard: rank
 * s sends rows(s) x cols(q) (row-major, packed) to rank q, which places it at
 * row row_begin[s] of its n_d x cols(q) slab.  Output arrays hold nranks entries.
 * Requires d >= 2. */
sgh_status sgh_shard_layout(const int32_t *levels, int32_t d, int32_t nranks, int64_t *row_begin, int64_t *rows,
                            int64_t *col_begin, int64_t *cols);

/* Library-owned NCCL communicator created from a 128-byte ncclUniqueId that
 * the caller broadcasts (e.g. with torch.distributed).  *comm receives an
 * opaque handle.  Blocking (NCCL init is collective over all ranks). */
sgh_status sgh_comm_create(void **comm, const void *nccl_unique_id, int32_t nranks, int32_t rank);
void sgh_comm_destroy(void *comm);
/* Writes the 128-byte ncclUniqueId into out (host buffer of >= 128 bytes). */
sgh_status sgh_comm_unique_id(void *out);

/* Workspace bytes of the sharded calls (two all-to-all staging buffers). */
size_t sgh_sharded_workspace_bytes(const int32_t *levels, int32_t d, int32_t nranks);

/* Hierarchize a grid sharded along x_d over the ranks of `comm`.  shard: this
 * rank's rows (sgh_shard_rows), row-major, (row_end-row_begin) * prod_{k<d} n_k
 * doubles.  Axes 1..d-1 are transformed locally; the axis-d pass runs after an
 * NCCL all-to-all re-shard into column blocks and the result is returned to
 * row sharding by a second all-to-all.  Collective: every rank must call it.
 * Bitwise equal to the single-GPU result. */
sgh_status sgh_hierarchize_sharded(double *shard, const int32_t *levels, int32_t d, void *comm,
                                   void *workspace, size_t ws_bytes, void *stream);
sgh_status sgh_dehierarchize_sharded(double *shard, const int32_t *levels, int32_t d, void *comm,
                                     void *workspace, size_t ws_bytes, void *stream);

/* Test utility: the sharded algorithm above for `nranks` VIRTUAL ranks on the
 * current device (the all-to-all becomes device-to-device copies).  shards:
 * host array of nranks device pointers (rank r's rows, sgh_shard_rows).
 * workspace: nranks * sgh_sharded_workspace_bytes() bytes.  Exercises the same
 * planning, packing and slab passes as the NCCL path on a single GPU. */
sgh_status sgh_transform_sharded_loopback(double *const *shards, const int32_t *levels, int32_t d, int32_t nranks,
                                          uint32_t flags, void *workspace, size_t ws_bytes, void *stream);

/* ---- halo + coarse-lattice sharded pass ----
 * The same row sharding of x_d over nranks = 2^p ranks (sgh_shard_rows), but
 * the axis-d pass needs no re-shard: rank r's rows are the aligned
 * super-block [r 2^T, (r+1) 2^T) of every x_d pole (T = l_d - p), whose
 * interior depends only on the shard plus ONE halo row (the next shard's first
 * row), by Alg. 1's finest-first order and predecessor rule;
 * the shards' first rows form the coarse lattice, a level-p pole per column.
 * One ncclAllGather of prod_{k<d} n_k doubles per rank gathers the first rows
 * (halo and coarse lattice at once); every rank transforms the P - 1 coarse
 * rows redundantly and keeps its own.  Bitwise equal to the single-GPU result.
 *  shard:     this rank's rows (row_end - row_begin) * C doubles followed by ONE
 *             spare row of C doubles (the halo slot; unspecified on return),
 *             C = prod_{k<d} n_k.
 *  workspace: >= sgh_sharded_halo_workspace_bytes() bytes (nranks * C doubles).
 *  flags:     SGH_FLAG_DEHIERARCHIZE for the inverse (coarse lattice first);
 *             SGH_FLAG_PER_AXIS: the unfused hierarchization below.
 * Hierarchization is FUSED by default: the ORIGINAL first rows are gathered
 * before any transform, and one box plan over the shard (axes 1..d-1 whole /
 * in aligned blocks together with blocks of x_d inside the super-block and the
 * super-block's own coarse lattice as later classes; the a4 block scheme)
 * writes the interior in ~1 HBM round trip; the gathered coarse rows are then
 * hierarchized as a grid of levels (l_1..l_{d-1}, p).  Unfused (and the
 * inverse): axes 1..d-1 on the shard, then the gather, then the x_d interior.
 * Errors: INVALID_ARGUMENT if nranks is not a power of two >= 2 or
 * nranks > 2^{l_d - 1}.  Collective: every rank calls it. */
size_t sgh_sharded_halo_workspace_bytes(const int32_t *levels, int32_t d, int32_t nranks);
sgh_status sgh_transform_sharded_halo(double *shard, const int32_t *levels, int32_t d, void *comm, uint32_t flags,
                                      void *workspace, size_t ws_bytes, void *stream);
/* Test utility: the halo path for `nranks` VIRTUAL ranks on the current device
 * (the all-gather becomes device copies).  shards[r]: rank r's rows + spare
 * row; workspace: nranks * sgh_sharded_halo_workspace_bytes() bytes. */
sgh_status sgh_transform_sharded_halo_loopback(double *const *shards, const int32_t *levels, int32_t d,
                                               int32_t nranks, uint32_t flags, void *workspace, size_t ws_bytes,
                                               void *stream);

/* ---- device-API (LSA) exchange for the all-to-all path (SURVEY 8(f) 4 iii) ----
 * The re-shard of sgh_hierarchize_sharded done inside kernels over NVLink peer
 * memory (NCCL 2.28 device API) instead of pack -> ncclSend/Recv -> unpack:
 * rank r's kernel stores its rows(r) x C_q blocks straight into rank q's slab
 * (a symmetric window, layout n_d x |C_q| row-major) and, after the x_d pass
 * (Alg. 1's outer loop reaching d), loads its blocks back from
 * every rank's slab into its shard.  Same arithmetic and order as the NCCL
 * path: bitwise identical to the single-grid transform.
 *
 * sgh_comm_lsa_enable: COLLECTIVE over the communicator's ranks, once (not in
 *   the hot call): allocates (ncclMemAlloc) and registers a symmetric window of
 *   window_bytes (>= sgh_sharded_lsa_window_bytes of the largest grid to be
 *   transformed; library-owned, freed by sgh_comm_destroy) and a device
 *   communicator with one LSA barrier per exchange CTA.  SGH_ERR_NCCL when the
 *   load/store-accessible team does not span every rank (e.g. ranks on several
 *   nodes) or the device API is unavailable; SGH_ERR_INVALID_ARGUMENT when
 *   already enabled or nranks > 64.
 * sgh_transform_sharded_lsa: COLLECTIVE; shard = this rank's rows (no spare
 *   row), in place; flags: SGH_FLAG_DEHIERARCHIZE for the inverse.  Needs no
 *   workspace (the window is the slab).  SGH_ERR_WORKSPACE if the window is
 *   too small.  Stream-ordered; the exchange kernels synchronize with the
 *   peers' exchange kernels through the LSA barriers only.
 * sgh_transform_sharded_lsa_loopback (test): the same kernels for nranks
 *   VIRTUAL ranks on the current device (window pointers from a table, no
 *   barriers); workspace: nranks * sgh_sharded_lsa_window_bytes() bytes. */
sgh_status sgh_comm_lsa_enable(void *comm, size_t window_bytes);
size_t sgh_sharded_lsa_window_bytes(const int32_t *levels, int32_t d, int32_t nranks);
sgh_status sgh_transform_sharded_lsa(double *shard, const int32_t *levels, int32_t d, void *comm, uint32_t flags,
                                     void *stream);
sgh_status sgh_transform_sharded_lsa_loopback(double *const *shards, const int32_t *levels, int32_t d,
                                              int32_t nranks, uint32_t flags, void *workspace, size_t ws_bytes,
                                              void *stream);

/* ----------------------------------------- harness utilities (not the method) */

/* Seeded counter-based fill: value of global flat
 * index i = index_offset + k is 2*((mix64(key+i)>>11)*2^-53) - 1 with
 * key = mix64(seed ^ mix64(grid_id)), mix64 = splitmix64. */
sgh_status sgh_fill_uniform(double *grid, int64_t n, uint64_t seed, uint64_t grid_id,
                            int64_t index_offset, void *stream);

/* Batched fill: grid g gets grid_id = grid_ids[g] (host int64 array), offset 0. */
sgh_status sgh_fill_uniform_batched(double *const *grids, const int64_t *sizes, const uint64_t *grid_ids,
                                    int64_t num_grids, uint64_t seed, void *workspace, size_t ws_bytes,
                                    void *stream);

/* Order-independent digest sum_i mix64(bits(v_i) ^ (i * 0x9E3779B97F4A7C15))
 * mod 2^64 over i = index_offset + k.  Writes *out_host; SYNCHRONISES stream. */
sgh_status sgh_digest(const double *grid, int64_t n, int64_t index_offset, uint64_t *out_host, void *stream);

/* Per-grid digests of a batch into out_host[num_grids]; synchronises. */
sgh_status sgh_digest_batched(double *const *grids, const int64_t *sizes, int64_t num_grids,
                              uint64_t *out_host, void *workspace, size_t ws_bytes, void *stream);

/* ------------------------------------------------ ablation (report only)
 * the paper's BFS data layout of a 1-D pole (Fig.
 * fig:hierDehier: points in breadth-first order of the binary hierarchy --
 * root first, level by level, left to right; natural 1-based point
 * i = (2 j + 1) 2^{l - lam} at BFS position 2^{lam-1} - 1 + j).  Not the
 * product layout; timed against the row-major kernels by
 * scripts/ablation_bfs.py.  Device pointers to 2^l - 1 doubles, stream-ordered.
 *  permute: to_bfs != 0: dst[BFS(p)] = src[natural]; else the inverse.
 *  hierarchize: out of place (one-pass stencil of the entering values; in and
 *               out must not alias); dehierarchize: in place, one launch per
 *               level, coarse -> fine.  Bitwise equal to Alg. 1 on the
 *               permuted data.  Errors: INVALID_ARGUMENT (NULL / aliased / l
 *               outside 1..SGH_MAX_LEVEL), CUDA. */
sgh_status sgh_ablation_bfs_permute_1d(const double *src, double *dst, int32_t l, int32_t to_bfs, void *stream);
sgh_status sgh_ablation_bfs_hierarchize_1d(const double *in, double *out, int32_t l, void *stream);
sgh_status sgh_ablation_bfs_dehierarchize_1d(double *grid, int32_t l, void *stream);

/* The planner's estimate of a grid's transform time in ns (its cost model:
 * 16 B per point and pass over each kernel kind's measured B200 rate), host
 * only; -1 on invalid arguments.  Used to balance grids over ranks by time
 * rather than points (bench.py, C5 with N > 1). */
double sgh_plan_cost(const int32_t *levels, int32_t d, uint32_t flags);

/* Optional per-launch timing of the transform kernels (process-wide).
 * sgh_profile_enable(1) clears the record list and starts recording: every
 * transform kernel launch is bracketed by two CUDA events on its own stream.
 * sgh_profile_enable(0) stops (and clears).  sgh_profile_read fills up to
 * `capacity` records (waiting for their events) and returns the number of
 * records; out may be NULL to query the count.  kind: 0 FLAT_SLABS,
 * 1 FLAT_BLOCKS, 2 STRIDED, 3 REG, 4 FUSED (k_fused), 5 gather, 6 scatter,
 * 7 FUSED contiguous-run tiles on the pipelined bulk-copy kernel (k_fpipe).
 * bytes = 16 x points transformed (gather / scatter: their own byte model). */
typedef struct {
    int32_t kind;
    int32_t level;    /* REG: pole level; STRIDED / FUSED / kind 7: tile width W; else the task's l */
    int32_t inverse;  /* 1 for dehierarchization */
    int32_t variant;  /* FUSED: 0 dense, 1 BLOCKED tiles, 2 coarse-lattice views, 3 both */
    double bytes;     /* algorithmic bytes (one read + one write per point) */
    double ms;        /* event-timed duration, -1 if unavailable */
} sgh_launch_record;
sgh_status sgh_profile_enable(int32_t on);
int64_t sgh_profile_read(sgh_launch_record *out, int64_t capacity);

/* ------------------------------- combination technique gather / scatter
 * The communication phase the hierarchization exists for ("the
 * hierarchical surpluses ... communicated").
 * SPARSE GRID of level sum n: the hierarchical subspaces W_lam, lam_k >= 1,
 * |lam|_1 <= n, stored in ONE device array in the SG LAYOUT: subspaces by level
 * sum ascending, then lexicographically ascending in (lam_1..lam_d); inside
 * W_lam its prod_k 2^{lam_k - 1} points row-major with j_1 fastest (point
 * x_k = (2 j_k + 1) 2^{-lam_k}).  Grid l holds W_lam for lam <= l: its point
 * (i_1..i_d) is (lam_k = l_k - tz(i_k), j_k = i_k >> (tz(i_k) + 1)).
 * Limits: d <= SGH_MAX_D, n <= 62, every grid |l|_1 <= n and N < 2^31. */
#define SGH_FLAG_SCATTER 8u   /* sgh_combi_workspace_bytes: size for sgh_scatter (default: sgh_gather) */

/* Points of the sparse grid (sum over level sums s = d..n of C(s-1, d-1) 2^{s-d});
 * -1 if (d, n) is unsupported. */
int64_t sgh_sparse_num_points(int32_t d, int32_t n);

/* Device workspace (task tables) of sgh_gather (flags 0) or sgh_scatter
 * (SGH_FLAG_SCATTER) for these grids; 0 on invalid arguments. */
size_t sgh_combi_workspace_bytes(const int32_t *levels, int32_t d, int64_t num_grids, int32_t n, uint32_t flags);

/* GATHER: sparse[(lam, j)] = sum over the grids g holding W_lam, in the order
 * given, of coeffs[g] * grids[g][point(lam, j)] (accumulated from +0.0, one
 * rounded multiply and one rounded add per term: bitwise the oracle's
 * grid-by-grid accumulation).  Subspaces held by no grid get 0.
 *  grids:  host array of num_grids DEVICE pointers (hierarchical surpluses);
 *  levels: host int32[num_grids][d];  coeffs: host double[num_grids] (the
 *          combination coefficients (-1)^q C(d-1, q), or any weights);
 *  sparse: device array of sgh_sparse_num_points(d, n) doubles (written).
 *  Errors: SGH_ERR_INVALID_ARGUMENT (NULL arguments, invalid levels, a grid
 *  whose level sum exceeds n or with N >= 2^31 points, unsupported (d, n) or
 *  n - d > 30), SGH_ERR_WORKSPACE (workspace missing, misaligned or smaller
 *  than sgh_combi_workspace_bytes), SGH_ERR_CUDA (launch failure). */
sgh_status sgh_gather(const double *const *grids, const int32_t *levels, const double *coeffs, int32_t d,
                      int64_t num_grids, int32_t n, double *sparse, void *workspace, size_t ws_bytes, void *stream);

/* GATHER over a RANGE of subspaces, optionally continuing a running sum.
 *  sub_begin, sub_end: subspace indices in SG order (level sum ascending,
 *          then lexicographic, 0 <= sub_begin <= sub_end <=
 *          sgh_sparse_num_subspaces(d, n)); only the sparse points of these
 *          subspaces -- the contiguous range [sgh_sparse_subspace_offset(d, n,
 *          sub_begin), ..offset(sub_end)) -- are read or written.
 *  flags:  0 or SGH_FLAG_ACCUMULATE: each sum starts from the value already in
 *          sparse (the running sum of the grids that come earlier in the global
 *          grid order) instead of +0.0.  A partition of the grid list into
 *          CONTIGUOUS blocks, gathered block after block with ACCUMULATE,
 *          performs exactly the additions of one gather over the whole list,
 *          in the same order: bitwise equal.  That is the multi-GPU
 *          gather: rank r owns grid block r and continues the
 *          partial sums received from rank r-1, pipelined over subspace
 *          ranges (paper_1309_0392_b200.gather_chain).
 *  The workspace of sgh_combi_workspace_bytes (full range) is sufficient.
 *  Errors: SGH_ERR_INVALID_ARGUMENT for a range out of bounds, unknown flags
 *  or n - d > 30 (a subspace larger than any grid can hold); otherwise as
 *  sgh_gather.  An empty range does nothing. */
#define SGH_FLAG_ACCUMULATE 16u
/* SGH_FLAG_X1_BFS (sgh_gather_ex): every grid's x_1 rows are stored in BFS
 * order (sgh_permute_x1_bfs) -- the gather then reads contiguous runs of each
 * level's points instead of one double per 2^{l_1 - lam_1 + 1}; same values,
 * same additions in the same order: bitwise equal to the row-major gather. */
#define SGH_FLAG_X1_BFS 128u
sgh_status sgh_gather_ex(const double *const *grids, const int32_t *levels, const double *coeffs, int32_t d,
                         int64_t num_grids, int32_t n, double *sparse, int64_t sub_begin, int64_t sub_end,
                         uint32_t flags, void *workspace, size_t ws_bytes, void *stream);
/* Number of subspaces W_lam of the sparse grid (C(n, d)), and the sparse
 * offset of subspace index i in SG order (i = count: the total points); -1 on
 * invalid arguments. */
int64_t sgh_sparse_num_subspaces(int32_t d, int32_t n);
int64_t sgh_sparse_subspace_offset(int32_t d, int32_t n, int64_t index);

/* Out-of-place permutation of every x_1 row (n_1 = 2^{l_1} - 1 contiguous
 * doubles) of each grid into BFS order (Fig. fig:hierDehier: the
 * level-1 point, then level 2, .., each level by j_1): natural 1-based index i,
 * level lam = l_1 - tz(i), j = i >> (tz(i) + 1), goes to position
 * 2^{lam-1} - 1 + j.  The layout SGH_FLAG_X1_BFS gathers from.
 *  src, dst: host arrays of num_grids DEVICE pointers (N doubles each; dst[g]
 *            must not alias src[g]); levels: host int32[num_grids][d].
 *  Stream-ordered; one launch per 96 grids.  Errors: INVALID_ARGUMENT (NULL /
 *  aliased pointers, invalid levels), CUDA. */
sgh_status sgh_permute_x1_bfs(const double *const *src, double *const *dst, const int32_t *levels, int32_t d,
                              int64_t num_grids, void *stream);

/* SCATTER: every point of every grid receives its sparse-grid value
 * (restriction of the combined surpluses; dehierarchize the grids afterwards
 * for nodal values). */
sgh_status sgh_scatter(double *const *grids, const int32_t *levels, int32_t d, int64_t num_grids, int32_t n,
                       const double *sparse, void *workspace, size_t ws_bytes, void *stream);

/* Host-only: the HBM bytes (16 B per point written by a kernel or copied on
 * the device) one sharded call plans for rank `rank` of `nranks` -- the local
 * axes 1..d-1 of its row shard (planned like a whole grid: fused / blocked
 * groups over the stacked (d-1)-dimensional rows), then path 0 (all-to-all,
 * sgh_hierarchize_sharded): pack + unpack copies and the slab pass along x_d;
 * path 1 (halo, sgh_transform_sharded_halo): the super-block interior, the
 * gathered coarse rows and the halo / coarse row copies.  Network bytes are
 * not included.  flags: 0, SGH_FLAG_DEHIERARCHIZE, SGH_FLAG_PER_AXIS (the
 * unfused halo hierarchization).  -1 on invalid
 * arguments.  SURVEY 8(a) a7 / 8(f) 1. */
double sgh_sharded_plan_bytes(const int32_t *levels, int32_t d, int32_t nranks, int32_t rank, uint32_t flags,
                              int32_t path);

/* Host-only description of the plan the library would run for one grid with
 * these flags (no CUDA call): one line per pass ("pass k:"), then one line per
 * phase with its kernel kind, tile width, special axis / block level and the
 * points it writes.  Writes at most cap bytes (NUL-terminated) into buf (may be
 * NULL) and returns the full length, or -1 on invalid levels / flags. */
int64_t sgh_plan_describe(const int32_t *levels, int32_t d, uint32_t flags, char *buf, size_t cap);

/* Number of kernels this library has launched in this process (all calls).
 * Used by bench.py to report gpu_launches. */
uint64_t sgh_launch_count(void);

const char *sgh_status_string(sgh_status s);
/* Detail of the last error on the calling thread ("" if none). */
const char *sgh_last_error(void);
/* Library version string. */
const char *sgh_version(void);

#ifdef __cplusplus
}
#endif
#endif /* SGH_H */
