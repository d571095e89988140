"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle.

Bar: the per-axis kernels keep the oracle's per-point
operation order, so every comparison here is BITWISE (0 differing 64-bit
words).  Where the oracle cannot be run at full size (C5: 41 GB) the check is
against golden digests written from the oracle / survey, plus sampled members
compared with the oracle one by one.
"""
import json
import os

import numpy as np
import pytest
import torch

import oracle
import sgh_inputs as si

pytestmark = pytest.mark.gpu

GOLD = os.path.join(os.path.dirname(__file__), "golden")
SD = json.load(open(os.path.join(GOLD, "survey_digests.json")))


@pytest.fixture(scope="module")
def sgh(gpu):
    import paper_1309_0392_b200 as m
    return m


def _bits(a):
    return np.ascontiguousarray(a, dtype=np.float64).view(np.uint64)


def assert_bitwise(got, want):
    got = np.asarray(got, dtype=np.float64)
    want = np.asarray(want, dtype=np.float64)
    assert got.shape == want.shape
    diff = np.nonzero(_bits(got) != _bits(want))[0]
    assert diff.size == 0, f"{diff.size} differing words, first at {diff[:5]}: {got[diff[:3]]} vs {want[diff[:3]]}"


def gpu_transform(sgh, u, levels, inverse=False, guard=4096, misalign=True, **kw):
    """Run the CUDA path on a copy of u placed inside a NaN guard region, at an
    8-mod-16 byte offset; check the guards are untouched; return the result."""
    off = guard + (1 if misalign else 0)
    buf = torch.full((u.size + 2 * off,), float("nan"), dtype=torch.float64, device="cuda")
    g = buf[off:off + u.size]
    g.copy_(torch.from_numpy(u))
    sgh.transform(g, levels, inverse=inverse, **kw)
    torch.cuda.synchronize()
    host = buf.cpu().numpy()
    assert np.all(np.isnan(host[:off])) and np.all(np.isnan(host[off + u.size:])), "guard region written"
    return host[off:off + u.size].copy()


# shapes that hit every kernel kind and edge: l=1 axes, N=1, S just below / at /
# above the FLAT limit (S=31, 63, 127), long contiguous poles (FLAT_BLOCKS +
# lattice recursion), long strided poles (STRIDED blocks + lattice), REG poles.
SHAPES = [
    (1,), (2,), (3,), (5,), (12,), (13,), (16,), (20,),
    (1, 1), (1, 7), (7, 1), (2, 2), (5, 5), (3, 4), (2, 13), (13, 2), (6, 6), (6, 9), (7, 7), (7, 12), (5, 14),
    (1, 1, 1), (3, 1, 4), (2, 5, 3), (4, 4, 4), (8, 2, 6), (1, 9, 2), (5, 5, 5), (2, 2, 10),
    (2, 2, 2, 2), (1, 3, 1, 3), (3, 4, 3, 5), (4, 1, 5, 2), (6, 6, 2, 2),
    (2, 3, 2, 3, 2), (1, 1, 1, 1, 9), (3, 2, 1, 2, 3, 2), (2, 2, 2, 2, 2, 2, 2), (2,) * 10,
    # multi-axis FUSED groups: contiguous (W=1) and column (W=8/16/32) tiles
    (1, 1, 5, 5), (5, 3, 3), (3, 4, 4, 2), (6, 6, 5, 5), (2, 3, 6, 6), (4, 2, 3, 7), (10, 4, 4, 4), (1, 3, 1, 4, 4),
    (7, 6, 6), (3, 5, 6), (2, 2, 6, 5, 1),
    # wide FUSED column tiles (W = 64 / 128) with ragged column groups
    (7, 2, 3), (6, 3, 3), (8, 2, 2, 2), (9, 3, 2), (5, 1, 2, 2),
]

# BLOCKED fused groups (one axis split into aligned 2^t blocks + end points, its
# coarse lattice a later phase): chosen by scripts/blocked_cover.py so that the
# planner's choices cover, for hierarchization and dehierarchization, contiguous
# (W=1) and column (W>1) tiles, the blocked axis first / in the middle / last in
# its group, block levels t = 0, 1, 2 (mod 3) (every top-lattice variant), the
# coarse-lattice views with 16- and 8-byte copies, and multi-step lattice chains.
BLOCKED_SHAPES = [
    (1, 2, 14, 1), (1, 3, 12), (1, 6, 2, 10), (1, 7, 13, 1), (1, 10, 8, 3), (1, 11, 2, 6), (2, 1, 11, 7),
    (2, 2, 4, 6), (2, 7, 11, 2), (2, 9, 4, 7), (3, 1, 6, 12), (3, 7, 7, 4), (4, 4, 1, 12), (4, 6, 2, 2),
    (5, 1, 2, 14), (5, 3, 3, 3), (7, 3, 5, 1), (7, 3, 5, 5), (8, 11, 1, 2), (9, 1, 2, 9), (9, 1, 9, 3),
    (9, 2, 8, 2), (9, 2, 10, 1), (9, 10, 1, 1), (10, 2, 5, 4), (11, 4, 2, 5), (11, 6, 2), (12, 4, 5),
    (14, 1, 3, 4), (8, 8, 8),
]
FUSE_MODES = [True, "whole", False]
FUSE_IDS = ["fused", "whole", "per_axis"]


@pytest.mark.parametrize("levels", SHAPES + BLOCKED_SHAPES, ids=str)
@pytest.mark.parametrize("inverse", [False, True], ids=["hier", "dehier"])
@pytest.mark.parametrize("fuse", FUSE_MODES, ids=FUSE_IDS)
def test_shape_sweep_bitwise(sgh, levels, inverse, fuse):
    N = si.num_points(levels)
    u = si.fill_uniform(N, grid_id=(N * 7 + len(levels)) % 9973)
    want = u.copy()
    (oracle.dehierarchize if inverse else oracle.hierarchize)(want, levels)
    got = gpu_transform(sgh, u, levels, inverse=inverse, fuse=fuse)
    assert_bitwise(got, want)


SUBNORMAL_SHAPES = [(5,), (13,), (6, 6), (14, 3), (8, 8, 8), (6, 6, 5, 5), (10, 4, 4, 4), (2, 7, 11, 2), (9, 2, 8, 2),
                    (3, 7, 7, 4), (12, 4, 5)]


@pytest.mark.parametrize("levels", SUBNORMAL_SHAPES, ids=str)
@pytest.mark.parametrize("inverse", [False, True], ids=["hier", "dehier"])
@pytest.mark.parametrize("fuse", FUSE_MODES, ids=FUSE_IDS)
def test_subnormal_bitwise(sgh, levels, inverse, fuse):
    """Subnormal and near-underflow inputs: 0.5*x is inexact for subnormal x
    with an odd last bit, so a contracted FMA would round once where the
    oracle (built with -ffp-contract=off) rounds the product and the sum
    separately.  Every kernel kind must keep the two roundings (bitwise)."""
    N = si.num_points(levels)
    u = si.fill_uniform(N, grid_id=(N * 5 + 3) % 9973)
    k = np.floor(u * 2.0 ** 52)                                # integers |k| < 2^52, many odd
    sub = np.ldexp(k, -1074)                                   # subnormal multiples of 2^-1074
    near = np.ldexp(u, -1020)                                  # normal, halving reaches subnormal
    x = np.where(np.arange(N) % 3 == 0, near, sub)
    want = x.copy()
    (oracle.dehierarchize if inverse else oracle.hierarchize)(want, levels)
    got = gpu_transform(sgh, x, levels, inverse=inverse, fuse=fuse)
    assert_bitwise(got, want)


@pytest.mark.parametrize("levels", [(5, 5), (3, 4, 2), (7, 6, 3), (2, 3, 2, 3)], ids=str)
def test_axis_orders_and_masks(sgh, levels):
    """Other axis orders: bitwise vs the oracle run in the same order."""
    N = si.num_points(levels)
    u = si.fill_uniform(N, grid_id=17)
    rng = np.random.default_rng(3)
    for _ in range(3):
        perm = [int(x) for x in rng.permutation(len(levels))]
        want = oracle.hierarchize(u.copy(), levels, perm)
        assert_bitwise(gpu_transform(sgh, u, levels, axis_order=perm), want)
    # axis mask: only axis 0 and the last
    mask = 1 | (1 << (len(levels) - 1))
    want = u.copy()
    oracle.hierarchize_axis(want, levels, 0)
    if len(levels) > 1:
        oracle.hierarchize_axis(want, levels, len(levels) - 1)
    assert_bitwise(gpu_transform(sgh, u, levels, axis_mask=mask), want)


@pytest.mark.parametrize("levels", [(5, 5), (8, 8, 8), (10, 4, 4, 4, 4), (14, 13)], ids=["C1", "C2", "C3", "C4"])
def test_closed_form_bitwise(sgh, levels):
    """f = prod x(1-x) -> alpha = prod 4^-lambda (BASELINE.json closed form), bitwise, at C1..C4."""
    f = torch.from_numpy(si.fill_smooth(levels)).cuda()
    sgh.hierarchize(f, levels)
    lam = None
    for l in levels:
        i = torch.arange(1, 1 << l, device="cuda", dtype=torch.int64)
        tz = torch.zeros_like(i)
        for b in range(l):
            tz += ((i & ((1 << (b + 1)) - 1)) == 0).to(torch.int64)
        lk = l - tz
        lam = lk if lam is None else (lk[:, None] + lam[None, :]).reshape(-1)
    want = torch.ldexp(torch.ones_like(f), -2 * lam)
    assert torch.equal(f, want)


@pytest.mark.parametrize("levels", [(5, 5), (3, 4, 2), (9, 7)], ids=str)
def test_tent_exact(sgh, levels):
    f = torch.from_numpy(si.fill_tent(levels, 0.625)).cuda()
    sgh.hierarchize(f, levels)
    nz = torch.nonzero(f).flatten().tolist()
    assert len(nz) == 1 and f[nz[0]].item() == 0.625


def test_fill_matches_input_module_and_oracle(sgh):
    for n, gid, off in [(1, 0, 0), (961, 0, 0), (100_003, 5, 17), (4097, 4254, 1 << 33)]:
        g = torch.empty(n, dtype=torch.float64, device="cuda")
        sgh.fill_uniform(g, si.SEED, gid, off)
        host = g.cpu().numpy()
        assert_bitwise(host, si.fill_uniform(n, si.SEED, gid, off))
        assert sgh.digest(g, off) == oracle.digest(host, off)


@pytest.mark.parametrize("name", ["C1", "C2", "C3", "C4"])
def test_config_golden_and_oracle(sgh, name):
    """Full-size configs: GPU digest == survey golden digest == oracle digest,
    plus an element-wise bitwise check against the oracle's output."""
    c = SD["configs"][name]
    levels = c["levels"]
    N = si.num_points(levels)
    g = torch.empty(N, dtype=torch.float64, device="cuda")
    sgh.fill_uniform(g, SD["seed"], c["grid_id"])
    assert sgh.digest(g) == int(c["input"], 16)
    sgh.hierarchize(g, levels)
    assert sgh.digest(g) == int(c["hierarchized"], 16)
    want = oracle.fill_uniform(N, SD["seed"], c["grid_id"])
    oracle.hierarchize(want, levels)
    assert_bitwise(g.cpu().numpy(), want)
    assert float(g.abs().max()) == c["max_abs_alpha"]
    if "dehierarchized_fill" in c:
        sgh.fill_uniform(g, SD["seed"], c["grid_id"])
        sgh.dehierarchize(g, levels)
        assert sgh.digest(g) == int(c["dehierarchized_fill"], 16)


@pytest.mark.parametrize("name", ["S1", "S10"])
@pytest.mark.parametrize("inverse", [False, True], ids=["hier", "dehier"])
def test_paper_sweep_tops_bitwise(sgh, name, inverse):
    """The paper's sweep shapes at their largest sizes: the 1-D
    l = 27 grid (134 M points, 1.07 GB; long-pole blocks + 2-level lattice) and
    the 10-D (9,2,...,2) grid, element-wise bitwise vs the oracle."""
    levels = si.SWEEPS[name].levels
    N = si.num_points(levels)
    g = torch.empty(N, dtype=torch.float64, device="cuda")
    sgh.fill_uniform(g, si.SEED, 7)
    (sgh.dehierarchize if inverse else sgh.hierarchize)(g, levels)
    want = oracle.fill_uniform(N, si.SEED, 7)
    (oracle.dehierarchize if inverse else oracle.hierarchize)(want, levels)
    assert_bitwise(g.cpu().numpy(), want)


@pytest.mark.parametrize("name,top", [("S1", 26), ("S10", 9)])
def test_paper_sweeps_small_levels(sgh, name, top):
    """Every level of the sweeps (1-D l = 1..26 step 5 + the tops' neighbours;
    10-D l_1 = 1..9), bitwise, hierarchize then dehierarchize."""
    lvs = si.sweep_levels(name, top)
    if name == "S1":
        lvs = [lv for lv in lvs if lv[0] % 5 == 1 or lv[0] >= 24]
    for lv in lvs:
        N = si.num_points(lv)
        u = si.fill_uniform(N, grid_id=lv[0])
        want = oracle.hierarchize(u.copy(), lv)
        got = gpu_transform(sgh, u, lv, guard=64)
        assert_bitwise(got, want)
        assert_bitwise(gpu_transform(sgh, want, lv, inverse=True, guard=64), oracle.dehierarchize(want.copy(), lv))


TWO_BLOCKED_SHAPES = [(10, 10), (11, 8), (13, 6), (12, 7), (1, 1, 11, 9), (12, 12), (7, 7), (5, 9), (9, 5), (3, 3)]


@pytest.mark.parametrize("levels", TWO_BLOCKED_SHAPES, ids=str)
def test_two_blocked_bitwise(sgh, levels):
    """The two-blocked plan (SURVEY 8(a) a4 block scheme: tiles fine along both
    axes, then the cross phases) forced on 2-D grids: bitwise vs the oracle."""
    N = si.num_points(levels)
    u = si.fill_uniform(N, grid_id=N % 977)
    want = oracle.hierarchize(u.copy(), levels)
    assert_bitwise(gpu_transform(sgh, u, levels, fuse="two_blocked"), want)


@pytest.mark.parametrize("levels", TWO_BLOCKED_SHAPES, ids=str)
def test_two_blocked_dehier_bitwise(sgh, levels):
    """Dehierarchization with the two-blocked plan (a-lattice of every row,
    fine-a of the coarse-b rows, b-lattice, the tiles with their b-end rows
    untouched, fine-b of the coarse-a columns) forced on 2-D grids: bitwise vs
    the oracle, also for the round trip (the oracle's own round trip, which
    is not the identity bit for bit)."""
    N = si.num_points(levels)
    a = si.fill_uniform(N, grid_id=N % 983)
    want = oracle.dehierarchize(a.copy(), levels)
    assert_bitwise(gpu_transform(sgh, a, levels, inverse=True, fuse="two_blocked"), want)
    h = oracle.hierarchize(a.copy(), levels)
    assert_bitwise(gpu_transform(sgh, h, levels, inverse=True, fuse="two_blocked"),
                   oracle.dehierarchize(h.copy(), levels))


PREFIX_TWO_BLOCKED_SHAPES = [(5, 7, 9), (2, 2, 9, 9), (1, 5, 7, 9), (5, 1, 7, 9), (4, 6, 8), (3, 3, 8, 7),
                             (2, 10, 10), (5, 5, 5), (3, 4, 3), (2, 2, 2, 5, 5), (3, 9, 4), (4, 4, 11)]


@pytest.mark.parametrize("levels", PREFIX_TWO_BLOCKED_SHAPES, ids=str)
def test_prefix_two_blocked_bitwise(sgh, levels):
    """Prefix two-blocked hierarchization (grids with >= 3 non-trivial axes:
    prefix axes whole, the last two in aligned blocks, then the classes of
    points coarse along {a}, {b}, {a, b}, recursively) forced with
    fuse="two_blocked": bitwise vs the oracle."""
    N = si.num_points(levels)
    u = si.fill_uniform(N, grid_id=N % 991)
    assert "bt2=" in sgh.plan_describe(levels, fuse="two_blocked")
    want = oracle.hierarchize(u.copy(), levels)
    assert_bitwise(gpu_transform(sgh, u, levels, fuse="two_blocked"), want)


PREFIX_TWO_BLOCKED_INV_SHAPES = [(2, 2, 9, 9), (4, 6, 8), (2, 10, 10), (5, 5, 5), (3, 4, 3), (2, 2, 2, 5, 5),
                                 (3, 9, 4), (4, 4, 11), (3, 7, 9), (2, 8, 8), (1, 3, 1, 7, 9)]


@pytest.mark.parametrize("levels", PREFIX_TWO_BLOCKED_INV_SHAPES, ids=str)
def test_prefix_two_blocked_dehier_bitwise(sgh, levels):
    """Prefix two-blocked DEhierarchization (one level: the points coarse along
    both blocked axes through a and then b, the class coarse along b, the box
    tiles with their end rows untouched, the class coarse along a in two
    halves) forced with fuse="two_blocked": bitwise vs the oracle, also on the
    oracle's own hierarchization output."""
    N = si.num_points(levels)
    a = si.fill_uniform(N, grid_id=N % 997)
    d = sgh.plan_describe(levels, inverse=True, fuse="two_blocked")
    assert any(int(x.split("bt2=")[1].split()[0]) >= 2 for x in d.splitlines() if "bt2=" in x)
    assert_bitwise(gpu_transform(sgh, a, levels, inverse=True, fuse="two_blocked"),
                   oracle.dehierarchize(a.copy(), levels))
    h = oracle.hierarchize(a.copy(), levels)
    assert_bitwise(gpu_transform(sgh, h, levels, inverse=True, fuse="two_blocked"),
                   oracle.dehierarchize(h.copy(), levels))


def test_two_blocked_c4_golden(sgh):
    c = SD["configs"]["C4"]
    g = torch.empty(si.num_points(c["levels"]), dtype=torch.float64, device="cuda")
    sgh.fill_uniform(g, SD["seed"], c["grid_id"])
    sgh.transform(g, c["levels"], fuse="two_blocked")
    assert sgh.digest(g) == int(c["hierarchized"], 16)


@pytest.mark.parametrize("levels", [(8, 8, 8), (14, 13), (10, 4, 4, 4, 4)], ids=["C2", "C4", "C3"])
def test_round_trip_device(sgh, levels):
    N = si.num_points(levels)
    g = torch.empty(N, dtype=torch.float64, device="cuda")
    sgh.fill_uniform(g, 1, 2)
    u = g.clone()
    sgh.hierarchize(g, levels)
    sgh.dehierarchize(g, levels)
    err = (g - u).abs().max() / u.abs().max()
    assert float(err) <= 1e-13


# --------------------------------------------------------------- batched
def _batch_check(sgh, members, ids, inverse=False, fuse=True):
    b = sgh.GridBatch(members, grid_ids=ids)
    b.fill_uniform(SD["seed"])
    b.transform(inverse, fuse=fuse)
    torch.cuda.synchronize()
    for lv, gid, v in zip(members, ids, b.views):
        want = oracle.fill_uniform(si.num_points(lv), SD["seed"], gid)
        (oracle.dehierarchize if inverse else oracle.hierarchize)(want, lv)
        assert_bitwise(v.cpu().numpy(), want)


def test_batched_table_resident_sequences(sgh):
    """Repeated batched calls skip the task-table upload when the batch's own
    workspace still holds the same plan's table (SGH_FLAG_TABLE_RESIDENT):
    hier, hier (resident), dehier, dehier (resident), a digest (reuses the
    workspace), hier, whole-pole hier -- every step bitwise vs the oracle
    applying the same sequence."""
    members = [(3, 4, 2), (6, 5, 1), (2, 2, 2), (7, 3, 3), (1, 9, 2), (5, 5, 5)]
    ids = list(range(len(members)))
    b = sgh.GridBatch(members, grid_ids=ids)
    b.fill_uniform(SD["seed"])
    want = [oracle.fill_uniform(si.num_points(lv), SD["seed"], g) for lv, g in zip(members, ids)]
    for op, fuse in [("h", True), ("h", True), ("d", True), ("d", True), ("digest", None), ("h", True),
                     ("h", "whole"), ("d", "whole")]:
        if op == "digest":
            b.digests()
            continue
        b.transform(op == "d", fuse=fuse)
        torch.cuda.synchronize()
        for w, lv in zip(want, members):
            (oracle.dehierarchize if op == "d" else oracle.hierarchize)(w, lv)
        for v, w in zip(b.views, want):
            assert_bitwise(v.cpu().numpy(), w)


@pytest.mark.parametrize("inverse", [False, True], ids=["hier", "dehier"])
@pytest.mark.parametrize("fuse", FUSE_MODES, ids=FUSE_IDS)
def test_batched_mixed_bitwise(sgh, inverse, fuse):
    rng = np.random.default_rng(11)
    members = [tuple(int(x) for x in rng.integers(1, 8, size=3)) for _ in range(60)]
    members += [(1, 1, 1), (13, 1, 2), (1, 12, 1), (2, 2, 11), (7, 7, 3)]
    members += [tuple(lv[:3]) + (1,) * (3 - len(lv)) for lv in BLOCKED_SHAPES if len(lv) <= 3 or lv[3:] == (1,)]
    _batch_check(sgh, members, list(range(len(members))), inverse, fuse)


@pytest.mark.parametrize("fuse", FUSE_MODES, ids=FUSE_IDS)
@pytest.mark.parametrize("inverse", [False, True], ids=["hier", "dehier"])
def test_batched_c5_sample_vs_oracle(sgh, fuse, inverse):
    """A sample of the C5 set (every 97th member plus the extremes), each compared
    with the oracle element by element."""
    cs = si.combination_set(4, 22)
    ids = sorted(set(list(range(0, len(cs), 97)) + [0, 1, 834, 1329, 1330, 4254]))
    _batch_check(sgh, [cs[i] for i in ids], ids, inverse, fuse)


def test_batched_c5_full_golden(sgh):
    """The whole C5 set (4,255 grids, 41 GB) in one batched call: per-grid
    digests summed == survey golden sums; four members == golden digests;
    then dehierarchization (of the hierarchized set, and of the fill) over the
    whole set against the oracle's digest sums."""
    cs = si.combination_set(4, 22)
    free, _ = torch.cuda.mem_get_info()
    if free < 46e9:
        pytest.skip("needs ~42 GB of free device memory")
    b = sgh.GridBatch(cs)
    b.fill_uniform(SD["seed"])
    din = b.digests()
    assert sum(din) % (1 << 64) == int(SD["C5"]["sum_input"], 16)
    b.hierarchize()
    dh = b.digests()
    assert sum(dh) % (1 << 64) == int(SD["C5"]["sum_hierarchized"], 16)
    for gid, m in SD["C5"]["members"].items():
        assert dh[int(gid)] == int(m["hierarchized"], 16)
        assert din[int(gid)] == int(m["input"], 16)
    b.dehierarchize()
    for gid in (0, 1, 834, 2000, 4254):                # round trip, normwise (reading R10)
        u = torch.from_numpy(oracle.fill_uniform(si.num_points(cs[gid]), SD["seed"], gid)).cuda()
        assert float((b.views[gid] - u).abs().max() / u.abs().max()) <= 1e-13
    # the round trip over the WHOLE set, bitwise: the sum of the per-grid digests
    # equals the oracle's (tests/golden/c5_oracle_digests.json, written by
    # scripts/golden/c5_oracle_digests.py from oracle/ only)
    od = json.load(open(os.path.join(GOLD, "c5_oracle_digests.json")))
    assert sum(b.digests()) % (1 << 64) == int(od["sum_round_trip"], 16)
    # dehierarchization of the fill over the whole set, bitwise
    b.fill_uniform(SD["seed"])
    b.dehierarchize()
    assert sum(b.digests()) % (1 << 64) == int(od["sum_dehierarchized_fill"], 16)


def test_batched_host_e2e(sgh):
    cs = si.combination_set(4, 14)
    hosts = [torch.from_numpy(si.fill_uniform(si.num_points(lv), SD["seed"], g)).pin_memory()
             for g, lv in enumerate(cs)]
    buf = torch.empty(sgh.batched_host_buffer_bytes(cs) // 8 + 64, dtype=torch.float64, device="cuda")
    sgh.transform_batched_host(hosts, cs, buf)
    torch.cuda.synchronize()
    for g, (lv, h) in enumerate(zip(cs, hosts)):
        want = oracle.hierarchize(si.fill_uniform(si.num_points(lv), SD["seed"], g), lv)
        assert_bitwise(h.numpy(), want)


def test_batched_host_e2e_multichunk_contiguous(sgh):
    """The e2e host path with many ~64 MB transfer chunks (more than the
    4-slot staging ring) and grids that are views of ONE pinned buffer (the
    contiguous-run placement: one copy per run of host-contiguous grids, the
    next chunk's grids copied in while the previous chunk is transformed);
    run twice (the second call hits the plan cache), bitwise vs the oracle."""
    cs = si.combination_set(4, 17)                       # ~520 MB: ~8 chunks of 64 MB
    sizes = [si.num_points(lv) for lv in cs]
    host = torch.empty(sum(sizes), dtype=torch.float64).pin_memory()
    views, off = [], 0
    for n in sizes:
        views.append(host[off:off + n])
        off += n
    fills = [si.fill_uniform(n, SD["seed"], g) for g, n in enumerate(sizes)]
    buf = torch.empty(sgh.batched_host_buffer_bytes(cs) // 8 + 64, dtype=torch.float64, device="cuda")
    pick = sorted(set(range(0, len(cs), 37)) | {0, len(cs) - 1})
    for rep in range(2):
        for v, f in zip(views, fills):
            v.copy_(torch.from_numpy(f))
        sgh.transform_batched_host(views, cs, buf)
        torch.cuda.synchronize()
        for g in pick:
            assert_bitwise(views[g].numpy(), oracle.hierarchize(fills[g].copy(), cs[g]))


# --------------------------------------------------------------- sharded
@pytest.mark.parametrize("levels,P", [((6, 5), 2), ((6, 5), 4), ((5, 4, 6), 8), ((3, 7), 8), ((8, 2, 3, 4), 4),
                                      ((14, 13), 8)], ids=str)
@pytest.mark.parametrize("inverse", [False, True], ids=["hier", "dehier"])
def test_sharded_loopback_bitwise(sgh, levels, P, inverse):
    """The sharded algorithm (row shards of x_d, re-shard to column blocks,
    axis-d pass, re-shard back) on P virtual ranks equals the single-grid
    oracle bitwise."""
    N = si.num_points(levels)
    u = si.fill_uniform(N, grid_id=77)
    want = u.copy()
    (oracle.dehierarchize if inverse else oracle.hierarchize)(want, levels)
    C = N // ((1 << levels[-1]) - 1)
    shards = []
    for r in range(P):
        b, e = sgh.shard_rows(levels, P, r)
        shards.append(torch.from_numpy(u[b * C:e * C].copy()).cuda())
    ws = torch.empty(P * sgh.sharded_workspace_bytes(levels, P) // 8, dtype=torch.float64, device="cuda")
    sgh.transform_sharded_loopback(shards, levels, ws, inverse=inverse)
    got = torch.cat(shards).cpu().numpy()
    assert_bitwise(got, want)


@pytest.mark.parametrize("levels,P", [((6, 5), 2), ((6, 5), 4), ((5, 4, 6), 8), ((3, 7), 8), ((8, 2, 3, 4), 4),
                                      ((4, 2), 2), ((2, 3, 9), 16), ((14, 13), 8), ((14, 13), 2), ((27,), 8),
                                      ((7, 7, 8), 4), ((5, 9), 2), ((9, 6), 16)], ids=str)
@pytest.mark.parametrize("inverse,fused", [(False, True), (False, False), (True, True)],
                         ids=["hier", "hier_unfused", "dehier"])
def test_sharded_halo_loopback_bitwise(sgh, levels, P, inverse, fused):
    """Halo + coarse-lattice sharded pass on P virtual ranks:
    shard interiors from shard + one halo row, coarse lattice from the gathered
    first rows; equals the single-grid oracle bitwise.  Hierarchization is fused
    by default (one box plan per shard over ORIGINAL end rows, then the coarse
    rows as a grid) and also run unfused.  Spare rows are NaN-filled (never read
    as data)."""
    N = si.num_points(levels)
    u = si.fill_uniform(N, grid_id=78)
    want = u.copy()
    (oracle.dehierarchize if inverse else oracle.hierarchize)(want, levels)
    C = N // ((1 << levels[-1]) - 1)
    shards = []
    for r in range(P):
        b, e = sgh.shard_rows(levels, P, r)
        buf = torch.full(((e - b + 1) * C,), float("nan"), dtype=torch.float64, device="cuda")
        buf[:(e - b) * C].copy_(torch.from_numpy(u[b * C:e * C]))
        shards.append(buf)
    ws = torch.empty(P * sgh.sharded_halo_workspace_bytes(levels, P) // 8, dtype=torch.float64, device="cuda")
    sgh.transform_sharded_halo_loopback(shards, levels, ws, inverse=inverse, fused=fused)
    got = torch.cat([s[:-C] for s in shards]).cpu().numpy()
    assert_bitwise(got, want)


@pytest.mark.parametrize("levels", [(8, 8, 8), (14, 13), (5, 4, 6)], ids=str)
@pytest.mark.parametrize("inverse", [False, True], ids=["hier", "dehier"])
def test_sharded_nccl_one_rank_bitwise(sgh, levels, inverse):
    """The NCCL transport itself on the one GPU the pool provides: a one-rank
    communicator (library-owned, from a unique id broadcast over a one-rank
    gloo group) through sgh_hierarchize_sharded -- the grouped
    ncclSend / ncclRecv all-to-all runs (to itself), the pack / slab / unpack
    copies with it; bitwise vs the oracle."""
    import socket

    import torch.distributed as dist
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1)
    try:
        comm = sgh.ShardComm()
        N = si.num_points(levels)
        u = si.fill_uniform(N, grid_id=91)
        want = (oracle.dehierarchize if inverse else oracle.hierarchize)(u.copy(), levels)
        g = torch.from_numpy(u.copy()).cuda()
        ws = torch.empty(sgh.sharded_workspace_bytes(levels, 1) // 8 + 1, dtype=torch.float64, device="cuda")
        comm.transform(g, levels, ws, inverse=inverse)
        torch.cuda.synchronize()
        assert_bitwise(g.cpu().numpy(), want)
        comm.close()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("levels,P", [((6, 5), 2), ((5, 4, 6), 8), ((3, 7), 8), ((8, 2, 3, 4), 4), ((4, 2), 2),
                                      ((2, 3, 9), 16), ((14, 13), 8), ((14, 13), 2), ((7, 7, 8), 4), ((9, 6), 1)],
                         ids=str)
@pytest.mark.parametrize("inverse", [False, True], ids=["hier", "dehier"])
def test_sharded_lsa_loopback_bitwise(sgh, levels, P, inverse):
    """The device-API exchange kernels (SURVEY 8(f) 4 iii; push of rows(r) x C_q
    into rank q's slab, pull back into the shard) for P virtual ranks on one
    GPU: every rank's blocks land where the x_d pass needs them; bitwise vs the
    single-grid oracle."""
    N = si.num_points(levels)
    u = si.fill_uniform(N, grid_id=83)
    want = (oracle.dehierarchize if inverse else oracle.hierarchize)(u.copy(), levels)
    C = N // ((1 << levels[-1]) - 1)
    shards = []
    for r in range(P):
        b, e = sgh.shard_rows(levels, P, r)
        shards.append(torch.from_numpy(u[b * C:e * C].copy()).cuda())
    ws = torch.full((P * sgh.sharded_lsa_window_bytes(levels, P) // 8,), float("nan"), dtype=torch.float64,
                    device="cuda")
    sgh.transform_sharded_lsa_loopback(shards, levels, ws, inverse=inverse)
    got = torch.cat(shards).cpu().numpy()
    assert_bitwise(got, want)


@pytest.mark.parametrize("levels", [(8, 8, 8), (14, 13), (5, 4, 6)], ids=str)
@pytest.mark.parametrize("inverse", [False, True], ids=["hier", "dehier"])
def test_sharded_lsa_one_rank_bitwise(sgh, levels, inverse):
    """The NCCL device-API exchange itself on the one GPU the pool provides: a
    one-rank communicator with a symmetric window and LSA barriers
    (sgh_comm_lsa_enable); k_reshard pushes into / pulls from the window
    through ncclGetLsaPointer; bitwise vs the oracle."""
    import socket

    import torch.distributed as dist
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1)
    try:
        comm = sgh.ShardComm()
        comm.enable_lsa(sgh.sharded_lsa_window_bytes(levels, 1))
        N = si.num_points(levels)
        u = si.fill_uniform(N, grid_id=92)
        want = (oracle.dehierarchize if inverse else oracle.hierarchize)(u.copy(), levels)
        g = torch.from_numpy(u.copy()).cuda()
        comm.transform_lsa(g, levels, inverse=inverse)
        torch.cuda.synchronize()
        assert_bitwise(g.cpu().numpy(), want)
        g2 = torch.from_numpy(u.copy()).cuda()       # a second call reuses the window and barriers
        comm.transform_lsa(g2, levels, inverse=inverse)
        torch.cuda.synchronize()
        assert_bitwise(g2.cpu().numpy(), want)
        comm.close()
    finally:
        dist.destroy_process_group()


def test_survey_abi_spellings_bitwise(sgh):
    """The SURVEY 8(b) spellings: sgh_hierarchize_ex (workspace accepted,
    unused) and sgh_dehierarchize_batched / sgh_workspace_bytes, called through
    the C ABI directly: bitwise vs the oracle."""
    import ctypes
    lv = (5, 4, 6)
    N = si.num_points(lv)
    u = si.fill_uniform(N, grid_id=5)
    g = torch.from_numpy(u.copy()).cuda()
    a = (ctypes.c_int32 * 3)(*lv)
    assert sgh.lib.sgh_hierarchize_ex(ctypes.c_void_p(g.data_ptr()), a, 3, None, 0, None, 0, None) == 0
    torch.cuda.synchronize()
    h = oracle.hierarchize(u.copy(), lv)
    assert_bitwise(g.cpu().numpy(), h)
    members = [(5, 4, 6), (3, 3, 3), (7, 2, 1)]
    flat = (ctypes.c_int32 * 9)(*[x for m in members for x in m])
    hosts = [oracle.hierarchize(si.fill_uniform(si.num_points(m), grid_id=i), m) for i, m in enumerate(members)]
    gs = [torch.from_numpy(x.copy()).cuda() for x in hosts]
    ptrs = (ctypes.c_void_p * 3)(*[x.data_ptr() for x in gs])
    wsb = sgh.lib.sgh_workspace_bytes(flat, 3, 3, 1)
    assert wsb == sgh.lib.sgh_batched_workspace_bytes(flat, 3, 3, 1) > 0
    ws = torch.empty(wsb // 8 + 2, dtype=torch.float64, device="cuda")
    assert sgh.lib.sgh_dehierarchize_batched(ptrs, flat, 3, 3, 0, ctypes.c_void_p(ws.data_ptr()), ws.numel() * 8,
                                             None) == 0
    torch.cuda.synchronize()
    for x, hst, m in zip(gs, hosts, members):
        assert_bitwise(x.cpu().numpy(), oracle.dehierarchize(hst.copy(), m))


def test_launch_count_increases(sgh):
    before = sgh.launch_count()
    g = torch.zeros(961, dtype=torch.float64, device="cuda")
    sgh.hierarchize(g, [5, 5])
    torch.cuda.synchronize()
    assert sgh.launch_count() > before


# --------------------------------------------- combination technique gather / scatter
@pytest.mark.parametrize("d,n", [(1, 9), (2, 10), (3, 9), (4, 12), (5, 9), (4, 16)], ids=str)
def test_gather_scatter_bitwise(sgh, d, n):
    """gather (coefficient-weighted sum of the grids' surpluses into
    the sparse grid, grid order) and scatter (restriction back to every grid),
    on hierarchized random grids of the combination set: bitwise vs the oracle."""
    cs = si.combination_set(d, n)
    co = [float(si.combination_coefficient(d, n, lv)) for lv in cs]
    hosts = [oracle.hierarchize(si.fill_uniform(si.num_points(lv), grid_id=g), lv) for g, lv in enumerate(cs)]
    grids = [torch.from_numpy(h).cuda() for h in hosts]
    sp = sgh.gather(grids, cs, co, n)
    want = oracle.gather(hosts, cs, co, n)
    assert sp.numel() == want.size == sgh.sparse_num_points(d, n)
    assert_bitwise(sp.cpu().numpy(), want)
    outs = [torch.full_like(g, float("nan")) for g in grids]
    sgh.scatter(sp, outs, cs, n)
    torch.cuda.synchronize()
    for o, w in zip(outs, oracle.scatter(want, cs, n)):
        assert_bitwise(o.cpu().numpy(), w)


def _bfs_rows_reference(u, levels):
    """x_1 rows in BFS order (layout only, numpy): natural 1-based i -> position
    2^{lam-1} - 1 + j, lam = l_1 - tz(i), j = i >> (tz(i) + 1)."""
    l1 = levels[0]
    n1 = (1 << l1) - 1
    i = np.arange(1, n1 + 1)
    tz = np.array([(int(x) & -int(x)).bit_length() - 1 for x in i])
    pos = (1 << (l1 - tz - 1)) - 1 + (i >> (tz + 1))
    rows = u.reshape(-1, n1)
    out = np.empty_like(rows)
    out[:, pos] = rows
    return out.reshape(-1)


@pytest.mark.parametrize("d,n", [(1, 9), (2, 10), (3, 9), (4, 12), (5, 9), (2, 16), (1, 15), (4, 16)], ids=str)
def test_gather_x1_bfs_bitwise(sgh, d, n):
    """The BFS-row gather (the grids' x_1 rows permuted into BFS order first,
    sgh_permute_x1_bfs, then SGH_FLAG_X1_BFS): the permutation matches the
    layout definition element by element (rows of l_1 <= 12 and of 2^12-index
    segments), and the gather is bitwise the oracle's."""
    cs = si.combination_set(d, n)
    co = [float(si.combination_coefficient(d, n, lv)) for lv in cs]
    hosts = [oracle.hierarchize(si.fill_uniform(si.num_points(lv), grid_id=g), lv) for g, lv in enumerate(cs)]
    grids = [torch.from_numpy(h).cuda() for h in hosts]
    perm = [torch.full_like(g, float("nan")) for g in grids]
    sgh.permute_x1_bfs(grids, perm, cs)
    torch.cuda.synchronize()
    for p_, h, lv in zip(perm, hosts, cs):
        assert_bitwise(p_.cpu().numpy(), _bfs_rows_reference(h, lv))
    sp = sgh.gather(perm, cs, co, n, x1_bfs=True)
    assert_bitwise(sp.cpu().numpy(), oracle.gather(hosts, cs, co, n))


@pytest.mark.parametrize("d,n,split,chunks", [(2, 8, 3, 4), (3, 8, 10, 5), (4, 9, 17, 16), (5, 8, 40, 7)])
def test_gather_ex_chain_bitwise(sgh, d, n, split, chunks):
    """sgh_gather_ex: the grid list split into two CONTIGUOUS blocks, the
    second gathered range by range with SGH_FLAG_ACCUMULATE onto the first's
    sums (what gather_chain does across ranks), equals one gather over all
    grids bitwise; so do range-by-range gathers without accumulation."""
    cs = si.combination_set(d, n)
    co = [float(si.combination_coefficient(d, n, lv)) for lv in cs]
    hosts = [oracle.hierarchize(si.fill_uniform(si.num_points(lv), grid_id=g), lv) for g, lv in enumerate(cs)]
    grids = [torch.from_numpy(h).cuda() for h in hosts]
    want = oracle.gather(hosts, cs, co, n)
    split = min(split, len(cs) - 1)
    sp = sgh.gather(grids[:split], cs[:split], co[:split], n)
    for b, e, lo, hi in sgh.subspace_chunks(d, n, chunks):
        sgh.gather_ex(grids[split:], cs[split:], co[split:], n, sp, b, e, accumulate=True)
    assert_bitwise(sp.cpu().numpy(), want)
    sp2 = torch.full((sgh.sparse_num_points(d, n),), float("nan"), dtype=torch.float64, device="cuda")
    for b, e, lo, hi in sgh.subspace_chunks(d, n, chunks):
        sgh.gather_ex(grids, cs, co, n, sp2, b, e)
    assert_bitwise(sp2.cpu().numpy(), want)


def test_gather_closed_form_c5_subset(sgh):
    """f = prod x(1-x) on the largest members of the C5 set that fit the oracle
    quickly... the full C5 set: every sparse point equals prod 4^-lam exactly
    (coefficients of the grids holding W_lam sum to 1)."""
    d, n = 4, 22
    cs = si.combination_set(d, n)
    free, _ = torch.cuda.mem_get_info()
    if free < 60e9:
        pytest.skip("needs ~50 GB of device memory")
    co = [float(si.combination_coefficient(d, n, lv)) for lv in cs]
    b = sgh.GridBatch(cs)
    for v, lv in zip(b.views, cs):
        v.copy_(torch.from_numpy(si.fill_smooth(lv)))
    b.hierarchize()
    sp = sgh.gather(b.views, cs, co, n)
    # expected: 4^-|lam|_1 per subspace, subspaces in SG order (level sum ascending)
    import math
    off = 0
    for s in range(d, n + 1):
        cnt = math.comb(s - 1, d - 1) << (s - d)
        blk = sp[off:off + cnt]
        assert bool((blk == 4.0 ** -s).all()), s
        off += cnt
    assert off == sp.numel()


@pytest.mark.parametrize("seed", range(int(os.environ.get("SGH_FUZZ_SEEDS", "6"))))
def test_random_shapes_fuzz(sgh, seed):
    """Planner fuzz: random level vectors (d = 1..6, up to ~2 M points) under every
    plan family -- automatic, whole-pole fusion only, per axis, forced two-blocked
    -- hierarchize and dehierarchize, bitwise vs the oracle.  SGH_FUZZ_SEEDS
    widens the seed range for ad-hoc runs."""
    rng = np.random.default_rng(1000 + seed)
    done = 0
    while done < 12:
        d = int(rng.integers(1, 7))
        lv = tuple(int(x) for x in rng.integers(1, 15 - 2 * d if d < 6 else 4, size=d))
        N = si.num_points(lv)
        if N > 2_000_000:
            continue
        done += 1
        u = si.fill_uniform(N, grid_id=done + 100 * seed)
        want_h = oracle.hierarchize(u.copy(), lv)
        want_d = oracle.dehierarchize(u.copy(), lv)
        for fuse in (True, "whole", False):
            assert_bitwise(gpu_transform(sgh, u, lv, fuse=fuse, guard=64), want_h)
            assert_bitwise(gpu_transform(sgh, u, lv, inverse=True, fuse=fuse, guard=64), want_d)
        assert_bitwise(gpu_transform(sgh, u, lv, guard=64, fuse="two_blocked"), want_h)
        assert_bitwise(gpu_transform(sgh, u, lv, inverse=True, guard=64, fuse="two_blocked"), want_d)


# --------------------------------------------- ablation: BFS layout (report only)
@pytest.mark.parametrize("l", [1, 2, 3, 5, 9, 13, 20], ids=str)
def test_bfs_layout_ablation_bitwise(sgh, l):
    """the paper's BFS layout of a 1-D pole.  The
    fill permuted into BFS order, hierarchized there (out of place) and
    permuted back is Alg. 1's result bitwise; the same for the in-place BFS
    dehierarchization; and the permutation round trip is the identity."""
    N = (1 << l) - 1
    u = si.fill_uniform(N, grid_id=l)
    nat = torch.from_numpy(u).cuda()
    bfs = torch.empty_like(nat)
    out = torch.empty_like(nat)
    back = torch.empty_like(nat)
    sgh.bfs_permute_1d(nat, bfs, l, to_bfs=True)
    sgh.bfs_permute_1d(bfs, back, l, to_bfs=False)
    torch.cuda.synchronize()
    assert_bitwise(back.cpu().numpy(), u)
    if l > 1:                                       # the root sits first in BFS order
        assert float(bfs[0]) == u[(1 << (l - 1)) - 1]
    sgh.bfs_hierarchize_1d(bfs, out, l)
    sgh.bfs_permute_1d(out, back, l, to_bfs=False)
    torch.cuda.synchronize()
    assert_bitwise(back.cpu().numpy(), oracle.hierarchize(u.copy(), (l,)))
    sgh.bfs_dehierarchize_1d(bfs, l)
    sgh.bfs_permute_1d(bfs, back, l, to_bfs=False)
    torch.cuda.synchronize()
    assert_bitwise(back.cpu().numpy(), oracle.dehierarchize(u.copy(), (l,)))


# ------------------------------------------- ablation: reduced-op (report only)
REDOP_LIB = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "paper_1309_0392_b200", "lib",
                         "libsgh_redop.so")


@pytest.mark.skipif(not os.path.exists(REDOP_LIB), reason="libsgh_redop.so not built (__graft_entry__.build())")
def test_reduced_op_ablation_normwise(sgh):
    """the paper's reduced-op update x - 0.5 (L + R),
    built as a second library (-DSGH_REDUCED_OP, every update site through one
    macro).  It rounds differently from Alg. 1's two subtractions (reading
    R5), so it is NOT bitwise equal to the oracle, but within the normwise
    1e-13 of reading R10 on every kernel kind the shapes reach."""
    import ctypes
    L = ctypes.CDLL(REDOP_LIB)
    L.sgh_hierarchize.restype = ctypes.c_int
    L.sgh_hierarchize.argtypes = [ctypes.c_void_p, ctypes.POINTER(ctypes.c_int32), ctypes.c_int32, ctypes.c_void_p]
    differs = 0
    for levels in [(5, 5), (12,), (8, 8, 8), (6, 6, 5, 5), (10, 4, 4, 4), (14, 3), (2, 7, 11, 2)]:
        N = si.num_points(levels)
        u = si.fill_uniform(N, grid_id=N % 991)
        g = torch.from_numpy(u).cuda()
        lv = (ctypes.c_int32 * len(levels))(*levels)
        assert L.sgh_hierarchize(ctypes.c_void_p(g.data_ptr()), lv, len(levels),
                                 ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)) == 0
        torch.cuda.synchronize()
        got = g.cpu().numpy()
        want = oracle.hierarchize(u.copy(), levels)
        assert np.max(np.abs(got - want)) / np.max(np.abs(want)) <= 1e-13, levels
        differs += int(np.count_nonzero(_bits(got) != _bits(want)))
    assert differs > 0, "the reduced-op build should round differently from Alg. 1"

