/*
 * oracle.c -- plain CPU oracle for hierarchization of combination grids
 * (arXiv 1309.0392).  TEST INFRASTRUCTURE ONLY: see oracle.h.
 *
 * Every routine is a direct transcription of the passage it cites; there is no
 * blocking, fusion or reordering beyond what Alg. 1 states.  Poles are gathered
 * into a scratch vector, transformed, and scattered back (a plain copy; it does
 * not change any arithmetic).
 *
 * Build: gcc -O2 -std=c11 -ffp-contract=off -fPIC -shared oracle.c -o liboracle.so -lm -lpthread
 */
#include "oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------ helpers */

static int valid_levels(const int32_t *levels, int32_t d) {
    if (!levels || d < 1 || d > 64) return 0;
    for (int32_t k = 0; k < d; ++k)
        if (levels[k] < 1 || levels[k] > 40) return 0;
    return 1;
}

int64_t sgo_num_points(const int32_t *levels, int32_t d) {
    if (!valid_levels(levels, d)) return -1;
    int64_t n = 1;
    for (int32_t k = 0; k < d; ++k) {
        int64_t nk = ((int64_t)1 << levels[k]) - 1; /* level l -> 2^l - 1 points */
        if (n > INT64_MAX / nk) return -1;
        n *= nk;
    }
    return n;
}

/* The three extents of the pole decomposition along axis k (0-based):
 * S = prod_{j<k} n_j (stride between pole points), n = n_k, O = prod_{j>k} n_j. */
static void pole_extents(const int32_t *levels, int32_t d, int32_t k,
                         int64_t *S, int64_t *n, int64_t *O) {
    int64_t s = 1, o = 1;
    for (int32_t j = 0; j < k; ++j) s *= ((int64_t)1 << levels[j]) - 1;
    for (int32_t j = k + 1; j < d; ++j) o *= ((int64_t)1 << levels[j]) - 1;
    *S = s;
    *n = ((int64_t)1 << levels[k]) - 1;
    *O = o;
}

/* ------------------------------------------------- Alg. 1, one 1-D pole */

/* P:127-131.  x is the pole, x[i-1] holds the point with 1-based index i.
 * Level lam holds the points i = s*(2j+1) with s = 2^{l-lam}; their left and
 * right hierarchical predecessors are i - s and i + s, absent when they
 * fall on the boundary (index 0 or 2^l). */
static void hierarchize_pole(double *x, int32_t l, int64_t *adds, int64_t *mults) {
    const int64_t n = ((int64_t)1 << l) - 1;
    for (int32_t lam = l; lam >= 2; --lam) {          /* "for l <- l_d, ..., 2" */
        const int64_t s = (int64_t)1 << (l - lam);
        for (int64_t i = s; i <= n; i += 2 * s) {      /* "for all x_i on level l" */
            if (i - s >= 1) {                          /* x[i] = x[i] - 0.5*leftPredecessor */
                x[i - 1] = x[i - 1] - 0.5 * x[i - s - 1];
                if (adds) { ++*adds; ++*mults; }
            }
            if (i + s <= n) {                          /* x[i] = x[i] - 0.5*rightPredecessor */
                x[i - 1] = x[i - 1] - 0.5 * x[i + s - 1];
                if (adds) { ++*adds; ++*mults; }
            }
        }
    }
}

/* Inverse (reading R9): levels 2 .. l (coarse to fine), +0.5*left then
 * +0.5*right; the predecessors are already nodal when a level is processed. */
static void dehierarchize_pole(double *x, int32_t l) {
    const int64_t n = ((int64_t)1 << l) - 1;
    for (int32_t lam = 2; lam <= l; ++lam) {
        const int64_t s = (int64_t)1 << (l - lam);
        for (int64_t i = s; i <= n; i += 2 * s) {
            if (i - s >= 1) x[i - 1] = x[i - 1] + 0.5 * x[i - s - 1];
            if (i + s <= n) x[i - 1] = x[i - 1] + 0.5 * x[i + s - 1];
        }
    }
}

/* "for all 1-dim poles in direction d": gather, transform, scatter. */
static int sweep_axis(double *grid, const int32_t *levels, int32_t d, int32_t axis,
                      int inverse, int64_t *adds, int64_t *mults) {
    if (!grid || !valid_levels(levels, d) || axis < 0 || axis >= d) return -1;
    if (levels[axis] == 1) return 0;                   /* single-point poles: no updates */
    int64_t S, n, O;
    pole_extents(levels, d, axis, &S, &n, &O);
    double *pole = (double *)malloc((size_t)n * sizeof(double));
    if (!pole) return -1;
    for (int64_t o = 0; o < O; ++o) {
        for (int64_t r = 0; r < S; ++r) {
            double *base = grid + o * n * S + r;
            for (int64_t i = 0; i < n; ++i) pole[i] = base[i * S];
            if (inverse) dehierarchize_pole(pole, levels[axis]);
            else hierarchize_pole(pole, levels[axis], adds, mults);
            for (int64_t i = 0; i < n; ++i) base[i * S] = pole[i];
        }
    }
    free(pole);
    return 0;
}

int sgo_hierarchize_axis(double *grid, const int32_t *levels, int32_t d, int32_t axis) {
    return sweep_axis(grid, levels, d, axis, 0, NULL, NULL);
}

int sgo_dehierarchize_axis(double *grid, const int32_t *levels, int32_t d, int32_t axis) {
    return sweep_axis(grid, levels, d, axis, 1, NULL, NULL);
}

static int check_order(const int32_t *order, int32_t d) {
    if (!order) return 1;
    int seen[64] = {0};
    for (int32_t k = 0; k < d; ++k) {
        if (order[k] < 0 || order[k] >= d || seen[order[k]]) return 0;
        seen[order[k]] = 1;
    }
    return 1;
}

/* Alg. 1 outer loop: dimensions in order. */
int sgo_hierarchize(double *grid, const int32_t *levels, int32_t d, const int32_t *axis_order) {
    if (!grid || !valid_levels(levels, d) || !check_order(axis_order, d)) return -1;
    for (int32_t k = 0; k < d; ++k) {
        int rc = sgo_hierarchize_axis(grid, levels, d, axis_order ? axis_order[k] : k);
        if (rc) return rc;
    }
    return 0;
}

int sgo_dehierarchize(double *grid, const int32_t *levels, int32_t d, const int32_t *axis_order) {
    if (!grid || !valid_levels(levels, d) || !check_order(axis_order, d)) return -1;
    for (int32_t k = 0; k < d; ++k) {
        int rc = sgo_dehierarchize_axis(grid, levels, d, axis_order ? axis_order[k] : k);
        if (rc) return rc;
    }
    return 0;
}

/* Timing only (bench.py cpu_baseline, SURVEY 8(c) "--threads T splits poles"):
 * the same Alg. 1 with the poles of each axis pass split into T contiguous
 * ranges, one pthread per range, each with its own pole scratch.  Poles are
 * independent, so the result is bitwise that of sgo_hierarchize. */
struct pole_range {
    double *grid;
    const int32_t *levels;
    int32_t d, axis, inverse;
    int64_t p0, p1;      /* pole indices p = o*S + r in [p0, p1) */
    int rc;
};

static void *pole_range_run(void *arg) {
    struct pole_range *R = (struct pole_range *)arg;
    int64_t S, n, O;
    pole_extents(R->levels, R->d, R->axis, &S, &n, &O);
    double *pole = (double *)malloc((size_t)n * sizeof(double));
    if (!pole) { R->rc = -1; return NULL; }
    for (int64_t p = R->p0; p < R->p1; ++p) {
        const int64_t o = p / S, r = p % S;
        double *base = R->grid + o * n * S + r;
        for (int64_t i = 0; i < n; ++i) pole[i] = base[i * S];
        if (R->inverse) dehierarchize_pole(pole, R->levels[R->axis]);
        else hierarchize_pole(pole, R->levels[R->axis], NULL, NULL);
        for (int64_t i = 0; i < n; ++i) base[i * S] = pole[i];
    }
    free(pole);
    R->rc = 0;
    return NULL;
}

int sgo_transform_threads(double *grid, const int32_t *levels, int32_t d, int32_t inverse, int32_t threads) {
    if (!grid || !valid_levels(levels, d) || threads < 1 || threads > 1024) return -1;
    struct pole_range *R = (struct pole_range *)calloc((size_t)threads, sizeof(*R));
    pthread_t *tid = (pthread_t *)calloc((size_t)threads, sizeof(pthread_t));
    if (!R || !tid) { free(R); free(tid); return -1; }
    int rc = 0;
    for (int32_t k = 0; k < d && !rc; ++k) {           /* P:125, dimensions in order */
        if (levels[k] == 1) continue;
        int64_t S, n, O;
        pole_extents(levels, d, k, &S, &n, &O);
        const int64_t poles = O * S;
        for (int32_t t = 0; t < threads; ++t) {
            R[t] = (struct pole_range){grid, levels, d, k, inverse,
                                       poles * t / threads, poles * (t + 1) / threads, 0};
            if (pthread_create(&tid[t], NULL, pole_range_run, &R[t])) { rc = -1; threads = t; break; }
        }
        for (int32_t t = 0; t < threads; ++t) {
            pthread_join(tid[t], NULL);
            if (R[t].rc) rc = -1;
        }
    }
    free(R);
    free(tid);
    return rc;
}

int sgo_counted_hierarchize(double *grid, const int32_t *levels, int32_t d,
                            int64_t *adds, int64_t *mults) {
    if (!adds || !mults) return -1;
    *adds = 0;
    *mults = 0;
    if (!grid || !valid_levels(levels, d)) return -1;
    for (int32_t k = 0; k < d; ++k) {
        int rc = sweep_axis(grid, levels, d, k, 0, adds, mults);
        if (rc) return rc;
    }
    return 0;
}

/* Eq. 1, per-pole term corrected to 2^{l+1} - 2l - 2 (reading R1). */
int64_t sgo_flop_count(const int32_t *levels, int32_t d) {
    if (!valid_levels(levels, d) || sgo_num_points(levels, d) < 0) return -1;
    int64_t F = 0;
    for (int32_t i = 0; i < d; ++i) {
        int64_t term = ((int64_t)1 << (levels[i] + 1)) - 2 * (int64_t)levels[i] - 2;
        for (int32_t j = 0; j < d; ++j)
            if (j != i) term *= ((int64_t)1 << levels[j]) - 1;
        F += term;
    }
    return 2 * F;
}

/* ------------------------------------------- basis-change brute force */

/* hat function of the 1-D point with 1-based index i on a level-l axis, at x:
 * hierarchical level lam = l - tz(i), centre i 2^-l, support half-width 2^-lam. */
static double hat(int32_t l, int64_t i, double x) {
    int32_t tz = 0;
    while (((i >> tz) & 1) == 0) ++tz;
    const int32_t lam = l - tz;
    const double centre = ldexp((double)i, -l);
    const double v = 1.0 - ldexp(fabs(x - centre), lam);
    return v > 0.0 ? v : 0.0;
}

/* multi-index of flat row-major point p (x_1 fastest), 1-based per axis */
static void unflatten(int64_t p, const int32_t *levels, int32_t d, int64_t *idx) {
    for (int32_t k = 0; k < d; ++k) {
        const int64_t nk = ((int64_t)1 << levels[k]) - 1;
        idx[k] = p % nk + 1;
        p /= nk;
    }
}

int sgo_basis_solve(const double *nodal, double *alpha, const int32_t *levels, int32_t d) {
    if (!nodal || !alpha || !valid_levels(levels, d)) return -1;
    const int64_t N = sgo_num_points(levels, d);
    if (N < 1) return -1;
    if (N > 2048) return -2;
    double *B = (double *)malloc((size_t)(N * N) * sizeof(double));
    double *b = (double *)malloc((size_t)N * sizeof(double));
    int64_t *ip = (int64_t *)malloc((size_t)d * sizeof(int64_t));
    int64_t *iq = (int64_t *)malloc((size_t)d * sizeof(int64_t));
    if (!B || !b || !ip || !iq) { free(B); free(b); free(ip); free(iq); return -1; }
    /* B[p][q] = prod_k phi_{q_k}(x_{p,k}) */
    for (int64_t p = 0; p < N; ++p) {
        unflatten(p, levels, d, ip);
        for (int64_t q = 0; q < N; ++q) {
            unflatten(q, levels, d, iq);
            double v = 1.0;
            for (int32_t k = 0; k < d; ++k)
                v *= hat(levels[k], iq[k], ldexp((double)ip[k], -levels[k]));
            B[p * N + q] = v;
        }
        b[p] = nodal[p];
    }
    /* Gaussian elimination with partial pivoting, then back substitution */
    for (int64_t c = 0; c < N; ++c) {
        int64_t piv = c;
        for (int64_t r = c + 1; r < N; ++r)
            if (fabs(B[r * N + c]) > fabs(B[piv * N + c])) piv = r;
        if (B[piv * N + c] == 0.0) { free(B); free(b); free(ip); free(iq); return -1; }
        if (piv != c) {
            for (int64_t k = 0; k < N; ++k) {
                double t = B[c * N + k]; B[c * N + k] = B[piv * N + k]; B[piv * N + k] = t;
            }
            double t = b[c]; b[c] = b[piv]; b[piv] = t;
        }
        for (int64_t r = c + 1; r < N; ++r) {
            const double f = B[r * N + c] / B[c * N + c];
            if (f == 0.0) continue;
            for (int64_t k = c; k < N; ++k) B[r * N + k] -= f * B[c * N + k];
            b[r] -= f * b[c];
        }
    }
    for (int64_t r = N - 1; r >= 0; --r) {
        double s = b[r];
        for (int64_t k = r + 1; k < N; ++k) s -= B[r * N + k] * alpha[k];
        alpha[r] = s / B[r * N + r];
    }
    free(B); free(b); free(ip); free(iq);
    return 0;
}

double sgo_evaluate(const double *alpha, const int32_t *levels, int32_t d, const double *x) {
    if (!alpha || !x || !valid_levels(levels, d)) return NAN;
    const int64_t N = sgo_num_points(levels, d);
    int64_t iq[64];
    double sum = 0.0;
    for (int64_t q = 0; q < N; ++q) {
        unflatten(q, levels, d, iq);
        double v = alpha[q];
        for (int32_t k = 0; k < d && v != 0.0; ++k) v *= hat(levels[k], iq[k], x[k]);
        sum += v;
    }
    return sum;
}

/* ------------------------------------------ seeded fill + digest (twin) */

static uint64_t mix64(uint64_t z) {
    z += 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

void sgo_fill_uniform(double *grid, int64_t n, uint64_t seed, uint64_t grid_id, int64_t index_offset) {
    const uint64_t key = mix64(seed ^ mix64(grid_id));
    for (int64_t k = 0; k < n; ++k) {
        const uint64_t i = (uint64_t)(index_offset + k);
        const double u = ldexp((double)(mix64(key + i) >> 11), -53);
        grid[k] = 2.0 * u - 1.0;
    }
}

uint64_t sgo_digest(const double *grid, int64_t n, int64_t index_offset) {
    uint64_t h = 0;
    for (int64_t k = 0; k < n; ++k) {
        uint64_t bits;
        memcpy(&bits, &grid[k], sizeof bits);
        const uint64_t i = (uint64_t)(index_offset + k);
        h += mix64(bits ^ (i * 0x9E3779B97F4A7C15ull));
    }
    return h;
}

/* ---------------------------------------------------------------------------
 * Combination technique gather / scatter (oracle.h).
 * ------------------------------------------------------------------------- */
struct sg_enum {
  int32_t d, n;
  int64_t *table; /* dense: index sum_k (lam_k - 1) n^k -> offset of W_lam */
  int64_t next;   /* running offset */
  int32_t lam[32];
};

static void sg_rec(struct sg_enum *E, int32_t k, int32_t remaining) {
  if (k == E->d - 1) {
    E->lam[k] = remaining;
    int64_t idx = 0, mul = 1, size = 1;
    for (int32_t q = 0; q < E->d; ++q) {
      idx += (int64_t)(E->lam[q] - 1) * mul;
      mul *= E->n;
      size <<= (E->lam[q] - 1);
    }
    E->table[idx] = E->next;
    E->next += size;
    return;
  }
  for (int32_t v = 1; v <= remaining - (E->d - 1 - k); ++v) { /* lexicographic: lam_k ascending */
    E->lam[k] = v;
    sg_rec(E, k + 1, remaining - v);
  }
}

/* builds the table; returns the number of sparse points, -1 if unsupported */
static int64_t sg_table(int32_t d, int32_t n, int64_t **table_out) {
  if (d < 1 || d > 32 || n < d) return -1;
  double cells = 1;
  for (int32_t k = 0; k < d; ++k) cells *= n;
  if (cells > (double)(1 << 26)) return -1;
  struct sg_enum E;
  E.d = d;
  E.n = n;
  E.next = 0;
  E.table = (int64_t *)malloc(sizeof(int64_t) * (size_t)cells);
  if (!E.table) return -1;
  for (int64_t c = 0; c < (int64_t)cells; ++c) E.table[c] = -1;
  for (int32_t s = d; s <= n; ++s) sg_rec(&E, 0, s); /* level sum ascending */
  if (table_out) *table_out = E.table;
  else free(E.table);
  return E.next;
}

int64_t sgo_sparse_num_points(int32_t d, int32_t n) { return sg_table(d, n, NULL); }

static int tz64(int64_t i) {
  int t = 0;
  while (!(i & 1)) {
    i >>= 1;
    ++t;
  }
  return t;
}

/* sparse index of grid point (i_1..i_d) of a grid with levels l */
static int64_t sg_index(const int64_t *table, int32_t d, int32_t n, const int32_t *l, const int64_t *i) {
  int64_t idx = 0, mul = 1, in = 0, imul = 1;
  for (int32_t k = 0; k < d; ++k) {
    const int t = tz64(i[k]);
    const int32_t lam = l[k] - t;
    const int64_t j = i[k] >> (t + 1);
    idx += (int64_t)(lam - 1) * mul;
    mul *= n;
    in += j * imul;
    imul <<= (lam - 1);
  }
  return table[idx] + in;
}

static int sg_walk(double *const *grids, const double *const *cgrids, const int32_t *levels, const double *coeffs,
                   int64_t num_grids, int32_t d, int32_t n, double *sparse, const double *csparse, int gather) {
  int64_t *table = NULL;
  const int64_t M = sg_table(d, n, &table);
  if (M < 0) return -1;
  if (gather)
    for (int64_t m = 0; m < M; ++m) sparse[m] = 0.0;
  for (int64_t g = 0; g < num_grids; ++g) {
    const int32_t *l = levels + g * d;
    int32_t sum = 0;
    for (int32_t k = 0; k < d; ++k) sum += l[k];
    if (sum > n || sgo_num_points(l, d) < 0) {
      free(table);
      return -1;
    }
    const int64_t N = sgo_num_points(l, d);
    int64_t i[32];
    for (int32_t k = 0; k < d; ++k) i[k] = 1;
    for (int64_t p = 0; p < N; ++p) { /* row-major, x_1 fastest */
      const int64_t s = sg_index(table, d, n, l, i);
      if (gather) sparse[s] = sparse[s] + coeffs[g] * cgrids[g][p];
      else grids[g][p] = csparse[s];
      for (int32_t k = 0; k < d; ++k) {
        if (++i[k] < ((int64_t)1 << l[k])) break;
        i[k] = 1;
      }
    }
  }
  free(table);
  return 0;
}

int sgo_gather(const double *const *grids, const int32_t *levels, const double *coeffs, int64_t num_grids,
               int32_t d, int32_t n, double *sparse) {
  if (!grids || !levels || !coeffs || !sparse) return -1;
  return sg_walk(NULL, grids, levels, coeffs, num_grids, d, n, sparse, NULL, 1);
}

int sgo_scatter(double *const *grids, const int32_t *levels, int64_t num_grids, int32_t d, int32_t n,
                const double *sparse) {
  if (!grids || !levels || !sparse) return -1;
  return sg_walk(grids, NULL, levels, NULL, num_grids, d, n, NULL, sparse, 0);
}
