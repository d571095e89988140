/*
 * oracle.h -- plain, slow, obviously-correct CPU oracle for the hierarchization
 * of combination-technique grids (arXiv 1309.0392).
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing in the product path (the CUDA library
 * libsgh.so and its Python binding) may include, link, import or execute
 * anything under oracle/.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may.  The oracle shares no code, header,
 * table or constant generator with the CUDA path.
 *
 * Citation format: P:n = PAPER.md line n; S:n = SPEC.md line n (the CPU
 * program spec written from the paper; used here for readings only).
 *
 * Conventions:
 *   - level vector l = (l_1..l_d), n_k = 2^{l_k} - 1 interior points per axis,
 *     zero boundary ("level 1 consist of one single grid point").
 *   - row-major with x_1 the fastest-varying index.
 *   - inside a pole, 1-based index i in 1..n, coordinate x = i * 2^{-l};
 *     hierarchical predecessors of i are i -/+ 2^{tz(i)} (Fig. 3).
 *   - all floating point is IEEE binary64; compiled with -ffp-contract=off.
 *
 * Parity status per function is stated in DESIGN.md ("Oracle pins").
 */
#ifndef SGH_ORACLE_H
#define SGH_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* N = prod_k (2^{l_k} - 1).  -1 on invalid levels or overflow. */
int64_t sgo_num_points(const int32_t *levels, int32_t d);

/* Alg. 1, literal: for dimension k = axis (0-based) only, every
 * pole in direction k, levels l_k down to 2, every point on the level in
 * increasing i:  x[i] = x[i] - 0.5*left;  x[i] = x[i] - 0.5*right   (absent
 * predecessor -> that update is skipped).  Returns 0, or -1 on bad args. */
int sgo_hierarchize_axis(double *grid, const int32_t *levels, int32_t d, int32_t axis);

/* Alg. 1 outer loop "for d <- 1..dim".  axis_order may be NULL
 * (= 0,1,..,d-1) or a permutation of 0..d-1. */
int sgo_hierarchize(double *grid, const int32_t *levels, int32_t d, const int32_t *axis_order);

/* Dehierarchization (P:77 prose "transforming the function values from the
 * hierarchical back to the regular grid basis"; reading S:167-171): exact
 * inverse order, levels 2 up to l_k, x[i] = x[i] + 0.5*left; x[i] = x[i] + 0.5*right. */
int sgo_dehierarchize_axis(double *grid, const int32_t *levels, int32_t d, int32_t axis);
int sgo_dehierarchize(double *grid, const int32_t *levels, int32_t d, const int32_t *axis_order);

/* Timing only (bench.py cpu_baseline): sgo_hierarchize (inverse = 0) or
 * sgo_dehierarchize (inverse = 1) with axis order 1..d and the poles of every
 * axis pass split over `threads` pthreads (poles are independent);
 * bitwise the same result.  Returns 0, or -1 on bad args. */
int sgo_transform_threads(double *grid, const int32_t *levels, int32_t d, int32_t inverse, int32_t threads);

/* Alg. 1 instrumented ("verified by instructing the code"): performs the
 * same updates and counts every floating point add/sub and multiply. */
int sgo_counted_hierarchize(double *grid, const int32_t *levels, int32_t d,
                            int64_t *adds, int64_t *mults);

/* Eq. 1 with the corrected per-pole term (reading R1):
 * F = 2 * sum_i (2^{l_i+1} - 2 l_i - 2) * prod_{j!=i} (2^{l_j} - 1).  -1 on overflow. */
int64_t sgo_flop_count(const int32_t *levels, int32_t d);

/* Second, independent oracle: the defining base change.
 * Builds the dense matrix B[p][q] = prod_k phi_{q_k}(x_{p,k}) of hat functions
 * phi_{lam,j}(x) = max(0, 1 - 2^lam |x - (2j+1) 2^-lam|) and solves
 * B alpha = u by Gaussian elimination with partial pivoting.
 * N must be <= 2048.  Returns 0, -1 on bad args, -2 if N too large. */
int sgo_basis_solve(const double *nodal, double *alpha, const int32_t *levels, int32_t d);

/* Hierarchical interpolant sum_q alpha_q prod_k phi_{q_k}(x_k) at x in (0,1)^d
 * (S:258-263).  Evaluated by brute force over all N surpluses. */
double sgo_evaluate(const double *alpha, const int32_t *levels, int32_t d, const double *x);

/* Oracle-side twin of the seeded input generator (SURVEY 8(d) "Fill"):
 * mix64 = splitmix64 finaliser; key = mix64(seed ^ mix64(grid_id));
 * value(i) = 2 * ((mix64(key + i) >> 11) * 2^-53) - 1,  i = index_offset + k. */
void sgo_fill_uniform(double *grid, int64_t n, uint64_t seed, uint64_t grid_id, int64_t index_offset);

/* Order-independent digest: sum_i mix64(bits(v_i) ^ (i * 0x9E3779B97F4A7C15)) mod 2^64. */
uint64_t sgo_digest(const double *grid, int64_t n, int64_t index_offset);

/* ---- combination technique communication phase ----
 * The sparse grid of level sum n is the set of hierarchical subspaces W_lam,
 * lam_k >= 1, |lam|_1 <= n; a combination grid l holds exactly the
 * subspaces lam <= l, its point (i_1..i_d) belonging to lam_k = l_k - tz(i_k),
 * j_k = i_k >> (tz(i_k) + 1) (the predecessor structure of P:140).
 * SG LAYOUT: subspaces by level sum ascending, then lexicographically ascending
 * in (lam_1..lam_d); inside a subspace the 2^{lam_k - 1} odd points per axis,
 * row-major with j_1 fastest (x_k = (2 j_k + 1) 2^{-lam_k}).
 * The oracle enumerates the subspaces one by one (no counting formula); it
 * supports n^d <= 2^26 (a dense lam -> offset table). */
int64_t sgo_sparse_num_points(int32_t d, int32_t n);

/* gather (the combination formula on hierarchical surpluses):
 *   sparse = 0;  for g = 0..num_grids-1 in order:  for every point of grid g:
 *     sparse[SG(lam, j)] = sparse[SG(lam, j)] + coeffs[g] * grid_g[point]
 * (plain multiply then add; no FMA).  grids[g]: grid g's surpluses, levels
 * row-major [num_grids][d].  Every grid must have |l_g|_1 <= n.  0 / -1. */
int sgo_gather(const double *const *grids, const int32_t *levels, const double *coeffs, int64_t num_grids,
               int32_t d, int32_t n, double *sparse);

/* scatter: every point of every grid receives its sparse-grid value,
 *   grid_g[point] = sparse[SG(lam, j)].  0 / -1. */
int sgo_scatter(double *const *grids, const int32_t *levels, int64_t num_grids, int32_t d, int32_t n,
                const double *sparse);

#ifdef __cplusplus
}
#endif
#endif
