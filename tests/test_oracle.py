"""Pins for the CPU oracle (oracle/), checked against what the paper and the
mathematics fix -- never against the oracle's own formula retyped.

Each test names the passage (P:n = PAPER.md line, S:n = SPEC.md line) or
DESIGN.md reading it pins.  A plausible mistake in the oracle (dropped term,
wrong sign, wrong predecessor index, transposed axis, wrong level order) fails
at least one of these; see test_negative_controls for explicit mutants.
"""
import itertools
import json
import os

import numpy as np
import pytest

import oracle
import sgh_inputs as si

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _load(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


WE = _load("worked_examples.json")
SD = _load("survey_digests.json")


def normwise(a, b):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    den = np.max(np.abs(b)) if b.size else 0.0
    return float(np.max(np.abs(a - b)) / den) if den > 0 else float(np.max(np.abs(a - b), initial=0.0))


# ------------------------------------------------------------- worked examples
@pytest.mark.parametrize("ex", WE["poles"], ids=lambda e: e["cite"][:6])
def test_pole_worked_examples(ex):
    x = np.array(ex["nodal"], dtype=np.float64)
    oracle.hierarchize(x, [ex["level"]])
    assert x.tolist() == ex["hierarchical"]
    oracle.dehierarchize(x, [ex["level"]])                         # S:173-174 inverse examples
    assert x.tolist() == [float(v) for v in ex["nodal"]]


@pytest.mark.parametrize("ex", WE["grids"], ids=lambda e: e["cite"][:6])
def test_grid_worked_examples(ex):
    x = np.array(ex["nodal"], dtype=np.float64)
    for a in ex["axes"]:
        oracle.hierarchize_axis(x, ex["levels"], a)
    assert x.tolist() == ex["result"]


def _level_bruteforce(l, i):
    """Hierarchical level of 1-based i in a level-l pole: the first grid level
    lam whose points j*2^(l-lam) contain i (Fig. 3 tree)."""
    for lam in range(1, l + 1):
        if i % (1 << (l - lam)) == 0:
            return lam
    raise AssertionError


def _preds_bruteforce(l, i):
    """closest strictly-coarser point on the left / right, None if only the boundary."""
    n = (1 << l) - 1
    lam = _level_bruteforce(l, i)
    left = next((j for j in range(i - 1, 0, -1) if _level_bruteforce(l, j) < lam), None)
    right = next((j for j in range(i + 1, n + 1) if _level_bruteforce(l, j) < lam), None)
    return left, right


@pytest.mark.parametrize("ex", WE["predecessors"], ids=lambda e: e["cite"][:6])
def test_predecessor_examples(ex):
    assert _preds_bruteforce(ex["level"], ex["i"]) == (ex["left"], ex["right"])


@pytest.mark.parametrize("l", range(1, 8))
def test_stencil_matrix_equals_predecessor_definition(l):
    """Hierarchizing unit vectors exposes the oracle's transform matrix H; with
    the one-pass property it must be I - 0.5 (Left + Right) where
    Left/Right are the brute-force predecessors of P:140."""
    n = (1 << l) - 1
    H = np.zeros((n, n))
    for j in range(n):
        e = np.zeros(n)
        e[j] = 1.0
        oracle.hierarchize(e, [l])
        H[:, j] = e
    expect = np.eye(n)
    for i in range(1, n + 1):
        lp, rp = _preds_bruteforce(l, i)
        if lp:
            expect[i - 1, lp - 1] -= 0.5
        if rp:
            expect[i - 1, rp - 1] -= 0.5
    assert np.array_equal(H, expect)


# ------------------------------------------------ brute-force basis change
_SMALL = [(1,), (2,), (5,), (7,), (3, 2), (2, 4), (4, 4), (2, 2, 2), (3, 1, 2), (1, 3, 3),
          (2, 2, 2, 2), (1, 1, 1), (3, 3, 2), (2, 1, 3, 1, 2)]


def test_hat_function_textbook_values():
    """phi of the root of a level-3 pole: 1 at the centre, 1/2 half-way, 0 at the
    boundary (P:51 piecewise-linear basis)."""
    for ex in WE["interpolant"]:
        a = np.zeros(si.num_points(ex["levels"]))
        a[a.size // 2] = ex["alpha_root"]
        assert oracle.evaluate(a, ex["levels"], ex["x"]) == ex["value"]
    a = np.zeros(7)
    a[3] = 1.0
    assert oracle.evaluate(a, [3], [0.999999]) < 1e-5


@pytest.mark.parametrize("levels", _SMALL, ids=str)
def test_alg1_equals_basis_change(levels):
    """Alg. 1 reproduces the defining base change alpha = B^-1 u
     on tiny grids; normwise <= 1e-14."""
    u = si.fill_uniform(si.num_points(levels), grid_id=hash(levels) % 1000)
    alpha_bf = oracle.basis_solve(u, levels)
    alpha = oracle.hierarchize(u.copy(), levels)
    assert normwise(alpha, alpha_bf) <= 1e-14


@pytest.mark.parametrize("levels", [(3, 2), (2, 2, 3), (4,), (1, 2, 3)], ids=str)
def test_interpolant_reproduces_nodal_values(levels):
    """Evaluating the hierarchical interpolant at every grid point gives u back
    (the defining property of surpluses)."""
    N = si.num_points(levels)
    u = si.fill_uniform(N, grid_id=7)
    alpha = oracle.hierarchize(u.copy(), levels)
    for p in range(N):
        x, q = [], p
        for l in levels:
            n = (1 << l) - 1
            x.append(((q % n) + 1) * 2.0 ** -l)
            q //= n
        assert abs(oracle.evaluate(alpha, levels, x) - u[p]) <= 4e-16 * max(1.0, abs(u[p]))


# ------------------------------------------------------------- closed forms
def _hier_levels(levels):
    """lambda_k = l_k - tz(i_k) for every grid point, row-major x_1 fastest."""
    lam = np.zeros(1, dtype=np.int64)
    for l in levels:
        i = np.arange(1, 1 << l)
        tz = np.zeros_like(i)
        for b in range(l):
            tz += ((i >> b) & 1 == 0) & ((i & ((1 << b) - 1)) == 0)
        lam_k = l - tz
        lam = np.add.outer(lam_k, lam)
    return lam.ravel()


@pytest.mark.parametrize("levels", [(5, 5), (3,), (6, 2, 4), (1, 7), (8, 8, 8)], ids=str)
def test_smooth_closed_form_bitwise(levels):
    """f = prod x_k(1-x_k) -> alpha = prod 4^-lambda_k  (BASELINE.json north_star
    closed form, reading R11: f(x) - (f(x-h)+f(x+h))/2 = h^2).  Bitwise."""
    f = si.fill_smooth(levels)
    oracle.hierarchize(f, levels)
    expect = np.ldexp(1.0, -2 * _hier_levels(levels))
    assert np.array_equal(f, expect)


@pytest.mark.parametrize("levels", [(5, 5), (3, 4, 2), (1, 1), (7,), (2, 3, 2, 3)], ids=str)
def test_tent_only_root_surplus(levels):
    """Level-1 piecewise multilinear input (reading R12): only the root surplus
    is non-zero and equals c; everything else exactly 0 (c dyadic so the
    nodal samples are exact)."""
    c = 0.625
    f = si.fill_tent(levels, c)
    oracle.hierarchize(f, levels)
    root = 0
    stride = 1
    for l in levels:
        root += ((1 << (l - 1)) - 1) * stride
        stride *= (1 << l) - 1
    assert f[root] == c
    f[root] = 0.0
    assert not np.any(f)


def test_update_rounds_product_and_difference_separately():
    """Alg. 1's update x <- x - 0.5*x_pred (reading R5/R8) is two
    IEEE operations: RN(0.5*e) then RN(x - that).  With t = 2^-1074 (the
    smallest subnormal), level-2 pole [3t, t, 0]: point 1's right predecessor
    is the root t; RN(0.5 t) is a tie that rounds to even, i.e. +0, so
    alpha_1 = 3t exactly (a single-rounding fma would give RN(2.5 t) = 2t).
    The inverse: 3t + RN(0.5 t) = 3t as well."""
    t = np.ldexp(1.0, -1074)
    u = np.array([3 * t, t, 0.0])
    a = oracle.hierarchize(u.copy(), (2,))
    assert a[0] == 3 * t and a[1] == t and a[2] == 0.0
    assert a[0] != 2 * t
    v = oracle.dehierarchize(np.array([3 * t, t, 0.0]), (2,))
    assert v[0] == 3 * t


# ------------------------------------------------------------- invariants
@pytest.mark.parametrize("levels", [(12, 3), (4, 5, 6), (2, 2, 2, 2, 2), (9,)], ids=str)
def test_round_trip(levels):
    """dehierarchize o hierarchize = identity, normwise <= 1e-13."""
    u = si.fill_uniform(si.num_points(levels), grid_id=3)
    v = oracle.dehierarchize(oracle.hierarchize(u.copy(), levels), levels)
    assert normwise(v, u) <= 1e-13


@pytest.mark.parametrize("levels", [(5, 5), (7, 3, 4), (1, 6, 2), (3, 3, 3, 3), (11,)], ids=str)
@pytest.mark.parametrize("threads", [1, 3, 8])
def test_threaded_timing_oracle_is_alg1(levels, threads):
    """The pole-threaded timing variant (bench cpu_baseline) is bitwise the
    single-thread Alg. 1 in both directions: poles are independent."""
    u = si.fill_uniform(si.num_points(levels), grid_id=5)
    a = oracle.hierarchize(u.copy(), levels)
    b = oracle.transform_threads(u.copy(), levels, threads)
    assert np.array_equal(a.view(np.uint64), b.view(np.uint64))
    c = oracle.dehierarchize(a.copy(), levels)
    e = oracle.transform_threads(a.copy(), levels, threads, inverse=True)
    assert np.array_equal(c.view(np.uint64), e.view(np.uint64))


def test_axis_order_and_linearity():
    """Tensor-product structure: axis permutations agree, and the
    transform is linear, normwise <= 1e-14."""
    levels = (4, 3, 5)
    N = si.num_points(levels)
    u = si.fill_uniform(N, grid_id=11)
    v = si.fill_uniform(N, grid_id=12)
    ref = oracle.hierarchize(u.copy(), levels)
    for perm in ([2, 1, 0], [1, 0, 2], [0, 2, 1]):
        assert normwise(oracle.hierarchize(u.copy(), levels, perm), ref) <= 1e-14
    lin = oracle.hierarchize((2.0 * u - 3.0 * v), levels)
    assert normwise(lin, 2.0 * ref - 3.0 * oracle.hierarchize(v.copy(), levels)) <= 1e-14


def _lattice_take(u, levels, coarse):
    g = u.reshape([(1 << l) - 1 for l in reversed(levels)])
    sl = tuple(slice((1 << (l - m)) - 1, None, 1 << (l - m)) for l, m in zip(reversed(levels), reversed(coarse)))
    return g[sl].ravel()


@pytest.mark.parametrize("levels,coarse", [((6, 5), (3, 2)), ((5, 5, 4), (2, 3, 1)), ((8, 8, 8), (4, 4, 4)),
                                           ((10, 4, 4, 4, 4), (5, 2, 3, 1, 4))], ids=str)
def test_restriction_bitwise(levels, coarse):
    """A point's surplus depends only on itself and its ancestors, all on
    the coarse lattice: hierarchize(u)|lattice == hierarchize_m(u|lattice), bitwise."""
    N = si.num_points(levels)
    u = oracle.fill_uniform(N, si.SEED, 5)
    fine = oracle.hierarchize(u.copy(), levels)
    sub = _lattice_take(u, levels, coarse).copy()
    oracle.hierarchize(sub, coarse)
    assert np.array_equal(_lattice_take(fine, levels, coarse), sub)


def test_embedding():
    """Combination-technique premise: nodal samples of a level-m
    interpolant on a finer grid hierarchize to the coarse surpluses on the
    lattice and 0 elsewhere (up to rounding)."""
    coarse, fine = (2, 3), (4, 5)
    a = si.fill_uniform(si.num_points(coarse), grid_id=21)
    nodal_c = oracle.dehierarchize(a.copy(), coarse)   # = interpolant at coarse points
    # sample the interpolant at every fine point
    u = np.empty(si.num_points(fine))
    for p in range(u.size):
        x, q = [], p
        for l in fine:
            n = (1 << l) - 1
            x.append(((q % n) + 1) * 2.0 ** -l)
            q //= n
        u[p] = oracle.evaluate(a, coarse, x)
    assert normwise(_lattice_take(u, fine, coarse), nodal_c) <= 1e-15
    al = oracle.hierarchize(u, fine)
    lat = _lattice_take(al, fine, coarse)
    assert normwise(lat, a) <= 1e-15
    mask = np.ones(al.size, bool)
    idx = _lattice_take(np.arange(al.size, dtype=np.float64), fine, coarse).astype(np.int64)
    mask[idx] = False
    assert np.max(np.abs(al[mask])) <= 3e-16 * np.max(np.abs(a)) * 4


# ------------------------------------------------------------ work counts
@pytest.mark.parametrize("levels,F", [((3,), 16), ((2, 2), 24), ((1,), 0), ((1, 1, 1), 0), ((5, 5), 6448)], ids=str)
def test_counted_updates_small(levels, F):
    """P:202 instrumented count; SPEC S:319-321 values; F = adds + mults, adds = mults."""
    g = si.fill_uniform(si.num_points(levels))
    a, m = oracle.counted_hierarchize(g, levels)
    assert a == m and a + m == F == oracle.flop_count(levels)


def test_counted_equals_corrected_eq1_random():
    """Corrected Eq. 1 (reading R1) == instrumented count for random level vectors."""
    rng = np.random.default_rng(0)
    for _ in range(40):
        d = int(rng.integers(1, 6))
        levels = [int(x) for x in rng.integers(1, 6, size=d)]
        if si.num_points(levels) > 200_000:
            continue
        g = np.zeros(si.num_points(levels))
        a, m = oracle.counted_hierarchize(g, levels)
        assert a + m == oracle.flop_count(levels)


def test_flop_count_config_values():
    fc = SD["flop_counts"]
    for c in ("C1", "C2", "C3", "C4"):
        assert oracle.flop_count(si.CONFIGS[c].levels) == fc[c]
    total = sum(oracle.flop_count(l) for l in si.combination_set(4, 22))
    assert total == fc["C5_total"]


def test_printed_eq1_is_inconsistent():
    """Reading R1: the printed term 2^l - 2l - 2 is negative for l=1,2,
    while the paper's own M and A = F/2 agree with the count."""
    printed = [(1 << l) - 2 * l - 2 for l in range(1, 5)]
    assert printed == [-2, -2, 0, 6]
    counted = []
    for l in range(1, 5):
        a, _m = oracle.counted_hierarchize(np.zeros((1 << l) - 1), [l])
        counted.append(a)
    assert counted == [(1 << (l + 1)) - 2 * l - 2 for l in range(1, 5)] == [0, 2, 8, 22]


# ----------------------------------------------------------- golden digests
def test_fill_first_values():
    v = SD["fill_first_values"]["values"]
    assert oracle.fill_uniform(4, SD["seed"], 0).tolist() == v
    assert si.fill_uniform(4, SD["seed"], 0).tolist() == v


@pytest.mark.parametrize("name", ["C1", "C2", "C3", "C4"])
def test_config_golden_digests(name):
    c = SD["configs"][name]
    N = si.num_points(c["levels"])
    g = oracle.fill_uniform(N, SD["seed"], c["grid_id"])
    assert oracle.digest(g) == int(c["input"], 16)
    if "dehierarchized_fill" in c:
        h = oracle.dehierarchize(g.copy(), c["levels"])
        assert oracle.digest(h) == int(c["dehierarchized_fill"], 16)
        del h
    oracle.hierarchize(g, c["levels"])
    assert oracle.digest(g) == int(c["hierarchized"], 16)
    assert float(np.max(np.abs(g))) == c["max_abs_alpha"]
    if name == "C1":
        assert g[0] == c["alpha_flat0"] and g[480] == c["alpha_root_flat480"]


@pytest.mark.parametrize("gid", ["0", "1", "834", "4254"])
def test_c5_member_golden_digests(gid):
    m = SD["C5"]["members"][gid]
    members = si.combination_set(4, 22)
    assert list(members[int(gid)]) == m["levels"]
    g = oracle.fill_uniform(si.num_points(m["levels"]), SD["seed"], int(gid))
    assert oracle.digest(g) == int(m["input"], 16)
    oracle.hierarchize(g, m["levels"])
    assert oracle.digest(g) == int(m["hierarchized"], 16)


def test_c5_member_set():
    members = si.combination_set(4, 22)
    assert len(members) == SD["C5"]["num_grids"]
    assert sum(si.num_points(l) for l in members) == SD["C5"]["num_points"]
    assert len(set(members)) == len(members)
    # coefficient sum 1
    assert sum(si.combination_coefficient(4, 22, l) for l in members) == 1


# ---------------------------------------------------------- negative controls
def _mutant_pole(x, l, mode):
    n = (1 << l) - 1
    lams = range(2, l + 1) if mode == "coarse_first" else range(l, 1, -1)
    for lam in lams:
        s = 1 << (l - lam)
        for i in range(s, n + 1, 2 * s):
            if mode == "plus":
                if i - s >= 1: x[i - 1] += 0.5 * x[i - s - 1]
                if i + s <= n: x[i - 1] += 0.5 * x[i + s - 1]
            elif mode == "right_only":
                if i + s <= n: x[i - 1] -= 0.5 * x[i + s - 1]
            else:
                if i - s >= 1: x[i - 1] -= 0.5 * x[i - s - 1]
                if i + s <= n: x[i - 1] -= 0.5 * x[i + s - 1]


@pytest.mark.parametrize("mode", ["coarse_first", "plus", "right_only"])
def test_negative_controls(mode):
    """Deliberately wrong transforms must fail the basis-change pin (S:455 spirit)."""
    l = 5
    u = si.fill_uniform((1 << l) - 1, grid_id=99)
    x = u.copy()
    _mutant_pole(x, l, mode)
    assert normwise(x, oracle.basis_solve(u, [l])) > 1e-3


def test_bad_arguments():
    L = oracle.lib()
    assert oracle.num_points([0]) == -1
    assert oracle.num_points([31, 31, 31]) == -1
    with pytest.raises(ValueError):
        oracle.hierarchize(np.zeros(3), [2], axis_order=[1])


# ------------------------------------------- combination technique gather / scatter
# (the communication phase the hierarchization serves)
def _sg_subspaces(d, n):
    """The SG layout by direct enumeration: subspaces lam >= 1, |lam|_1 <= n, level sum
    ascending, then lexicographically ascending; returns [(lam, offset, size)]."""
    out, off = [], 0
    for s in range(d, n + 1):
        for lam in sorted(c for c in itertools.product(range(1, s - d + 2), repeat=d) if sum(c) == s):
            size = 1 << (s - d)
            out.append((lam, off, size))
            off += size
    return out


def _sg_point_coords(lam):
    """Coordinates of the points of subspace lam in layout order (j_1 fastest)."""
    axes = [(2 * np.arange(1 << (l - 1)) + 1) * 2.0 ** -l for l in lam]
    mesh = np.meshgrid(*axes[::-1], indexing="ij")          # last axis slowest
    return np.stack([m.ravel() for m in mesh[::-1]], axis=1)  # (points, d), x_1 fastest


def _grid_coords(levels):
    axes = [np.arange(1, 1 << l) * 2.0 ** -l for l in levels]
    mesh = np.meshgrid(*axes[::-1], indexing="ij")
    return np.stack([m.ravel() for m in mesh[::-1]], axis=1)


@pytest.mark.parametrize("d,n", [(1, 6), (2, 2), (2, 7), (3, 6), (4, 9), (5, 8)])
def test_sparse_layout_size(d, n):
    assert oracle.sparse_num_points(d, n) == sum(sz for _, _, sz in _sg_subspaces(d, n))


def _combi(d, n):
    cs = si.combination_set(d, n)
    return cs, [si.combination_coefficient(d, n, lv) for lv in cs]


@pytest.mark.parametrize("d,n", [(2, 8), (3, 7), (4, 8)])
def test_gather_closed_form_exact(d, n):
    """f = prod x_k (1 - x_k) on every combination grid, hierarchized, gathered:
    every sparse point gets prod 4^-lam_k EXACTLY -- the grids' surpluses are the
    closed form (reading R11) and the coefficients of the grids holding W_lam sum
    to 1 (the combination technique)."""
    cs, co = _combi(d, n)
    grids = [oracle.hierarchize(si.fill_smooth(lv), lv) for lv in cs]
    sp = oracle.gather(grids, cs, co, n)
    for lam, off, sz in _sg_subspaces(d, n):
        assert np.all(sp[off:off + sz] == 4.0 ** -sum(lam)), lam


def _hat(lam, x):
    """phi_{lam,j}(x) for the unique j whose support holds x (0 elsewhere)."""
    h = 2.0 ** -lam
    j = np.floor(x / (2 * h)).astype(np.int64)
    return j, np.maximum(0.0, 1.0 - np.abs(x - (2 * j + 1) * h) / h)


@pytest.mark.parametrize("d,n", [(2, 7), (3, 6)])
def test_gather_reproduces_sparse_interpolant(d, n):
    """Random sparse-grid surpluses s; sample the sparse interpolant
    f = sum s phi on every combination grid (direct hat evaluation, here),
    hierarchize each grid (oracle), gather: the result is s again (the
    combination formula is exact on the sparse grid space), up to rounding."""
    rng = np.random.default_rng(5)
    subs = _sg_subspaces(d, n)
    s = rng.uniform(-1, 1, sum(sz for _, _, sz in subs))
    cs, co = _combi(d, n)
    grids = []
    for lv in cs:
        X = _grid_coords(lv)
        f = np.zeros(len(X))
        for lam, off, sz in subs:                     # one hat per subspace and point
            w = np.ones(len(X))
            idx = np.zeros(len(X), dtype=np.int64)
            mul = 1
            for k in range(d):
                j, v = _hat(lam[k], X[:, k])
                w *= v
                idx += j * mul
                mul <<= lam[k] - 1
            f += w * s[off + idx]
        grids.append(oracle.hierarchize(f, lv))
    got = oracle.gather(grids, cs, co, n)
    assert np.max(np.abs(got - s)) / np.max(np.abs(s)) <= 1e-13


@pytest.mark.parametrize("d,n", [(2, 7), (3, 7), (4, 8)])
def test_scatter_is_restriction(d, n):
    """scatter: grid point x of grid l gets the sparse value of the subspace point
    at x (found here by coordinates); then gather of the scattered surpluses
    returns s (coefficients of the grids holding W_lam sum to 1)."""
    rng = np.random.default_rng(6)
    subs = _sg_subspaces(d, n)
    s = rng.uniform(-1, 1, sum(sz for _, _, sz in subs))
    where = {}
    for lam, off, sz in subs:
        for k, x in enumerate(_sg_point_coords(lam)):
            where[tuple(x)] = off + k
    cs, co = _combi(d, n)
    out = oracle.scatter(s, cs, n)
    for lv, g in zip(cs, out):
        want = s[[where[tuple(x)] for x in _grid_coords(lv)]]
        assert np.array_equal(g, want)
    back = oracle.gather(out, cs, co, n)
    assert np.max(np.abs(back - s)) / np.max(np.abs(s)) <= 1e-13   # rounding of the +-C(d-1,q) sums
