"""CPU-only checks of the C-ABI library: it loads, exports every symbol that
include/sgh.h declares, and its host-only logic (geometry, validation, shard
ranges, workspace sizing) behaves.  No compute call is made here (no GPU)."""
import ctypes
import os
import re

import pytest

import paper_1309_0392_b200 as sgh
import sgh_inputs as si

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared_symbols():
    src = open(os.path.join(ROOT, "include", "sgh.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(sgh_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    names = _declared_symbols()
    assert len(names) >= 20
    L = ctypes.CDLL(sgh.LIB_PATH)
    missing = [n for n in names if not hasattr(L, n)]
    assert not missing, missing
    assert set(names) == set(sgh.EXPORTED)


def test_library_is_sm100a_only():
    out = os.popen(f"cuobjdump --list-elf {sgh.LIB_PATH} 2>&1").read()
    assert "sm_100a" in out
    for bad in ("sm_80", "sm_90", "sm_103"):
        assert bad not in out


def test_num_points():
    assert sgh.num_points([3]) == 7
    assert sgh.num_points([1, 1, 1]) == 1
    assert sgh.num_points([2, 2]) == 9
    assert sgh.num_points([14, 13]) == 134_193_153
    assert sgh.num_points([0]) == -1
    assert sgh.num_points([31]) == -1           # > SGH_MAX_LEVEL
    assert sgh.num_points([30, 30, 30]) == -1   # N*8 overflows int64
    assert sgh.num_points([1] * 17) == -1       # d > SGH_MAX_D


def test_validation_before_enqueue():
    """Invalid arguments are rejected on the host before any CUDA call."""
    i32 = ctypes.c_int32
    lv = (i32 * 2)(5, 0)
    rc = sgh.lib.sgh_hierarchize(ctypes.c_void_p(0x1000), lv, 2, None)
    assert rc == 1 and b"level" in sgh.lib.sgh_last_error()
    lv = (i32 * 2)(5, 5)
    assert sgh.lib.sgh_hierarchize(None, lv, 2, None) == 1
    assert sgh.lib.sgh_hierarchize(ctypes.c_void_p(0x1000), lv, 0, None) == 1
    big = (i32 * 1)(31)
    assert sgh.lib.sgh_hierarchize(ctypes.c_void_p(0x1000), big, 1, None) == 2
    bad_order = (i32 * 2)(0, 0)
    assert sgh.lib.sgh_transform_ex(ctypes.c_void_p(0x1000), lv, 2, bad_order, 0, 0, None) == 1
    assert sgh.lib.sgh_transform_ex(ctypes.c_void_p(0x1000), lv, 2, None, 0, 8, None) == 1   # unknown flag
    # batched: negative count, missing workspace
    ptrs = (ctypes.c_void_p * 1)(0x1000)
    assert sgh.lib.sgh_hierarchize_batched(ptrs, lv, 2, -1, 0, None, 0, None) == 1
    assert sgh.lib.sgh_hierarchize_batched(ptrs, lv, 2, 0, 0, None, 0, None) == 0      # empty batch OK
    assert sgh.lib.sgh_hierarchize_batched(ptrs, lv, 2, 1, 0, None, 0, None) == 5      # workspace
    assert sgh.lib.sgh_status_string(5) == b"SGH_ERR_WORKSPACE"


def test_shard_rows_dyadic():
    """Dyadic row shards of x_d: cover [0, n_d) exactly, rank 0
    one row short, others 2^{l_d - p} rows."""
    for levels in ([14, 13], [5, 4, 6], [3, 3]):
        nd = (1 << levels[-1]) - 1
        for P in (1, 2, 4, 8):
            if (1 << levels[-1]) < P:
                continue
            rows = [sgh.shard_rows(levels, P, r) for r in range(P)]
            assert rows[0][0] == 0 and rows[-1][1] == nd
            for (b0, e0), (b1, e1) in zip(rows, rows[1:]):
                assert e0 == b1
            blk = 1 << (levels[-1] - P.bit_length() + 1)
            assert rows[0][1] - rows[0][0] == blk - 1
            assert all(e - b == blk for b, e in rows[1:])
    with pytest.raises(sgh.SGHError):
        sgh.shard_rows([3, 3], 3, 0)          # not a power of two
    with pytest.raises(sgh.SGHError):
        sgh.shard_rows([3, 2], 8, 0)          # more ranks than 2^{l_d}


def test_workspace_sizing():
    assert sgh.batched_workspace_bytes([]) == 0
    c5 = si.combination_set(4, 22)
    ws = sgh.batched_workspace_bytes(c5)
    assert 0 < ws < 64 << 20
    assert sgh.batched_host_buffer_bytes(c5) >= 8 * sum(si.num_points(l) for l in c5)
    assert sgh.sharded_workspace_bytes([14, 13], 8) >= 2 * 8 * 1024 * 16383


@pytest.mark.parametrize("levels,P", [((14, 13), 8), ((10, 4, 4, 4, 4), 2), ((8, 8, 8), 4), ((6, 5), 1), ((3, 7), 8)],
                         ids=str)
def test_lsa_window_sizing(levels, P):
    """The device-API re-shard's window is one slab n_d x max_q |C_q| (column
    blocks C_q = [C q / P, C (q + 1) / P)); invalid arguments give 0."""
    C = si.num_points(levels[:-1]) if len(levels) > 1 else 1
    nd = (1 << levels[-1]) - 1
    maxc = max(C * (q + 1) // P - C * q // P for q in range(P))
    assert sgh.sharded_lsa_window_bytes(levels, P) == 8 * nd * maxc
    assert sgh.lib.sgh_sharded_lsa_window_bytes(None, 2, P) == 0
    assert sgh.sharded_lsa_window_bytes(levels, 3) == 0            # ranks must be a power of two


def test_no_cpu_fallback():
    import torch
    with pytest.raises(TypeError):
        sgh.hierarchize(torch.zeros(961, dtype=torch.float64), [5, 5])


def _plan_passes(levels, **kw):
    """Parse sgh_plan_describe: list of passes, each a list of (kind, attrs, points)."""
    passes = []
    for line in sgh.plan_describe(levels, **kw).splitlines():
        if line.startswith("pass"):
            passes.append([])
            continue
        kind = line.split()[0]
        attrs = dict(kv.split("=", 1) for kv in line.split()[1:])
        passes[-1].append((kind, attrs, float(attrs["points"])))
    return passes


@pytest.mark.parametrize("levels", [(8, 8, 8), (10, 4, 4, 4, 4), (16, 2, 2, 1), (2, 7, 11, 2), (9, 2, 8, 2),
                                    (1, 3, 12), (14, 1, 3, 4), (5, 3, 3, 3), (14, 13), (1, 10, 10, 1)], ids=str)
@pytest.mark.parametrize("inverse", [False, True], ids=["hier", "dehier"])
def test_plan_blocked_groups_cover_each_point_once(levels, inverse):
    """A fused pass (whole poles, or a BLOCKED group: block tiles + coarse-lattice
    views) writes every point of the grid exactly once; a dehierarchization plan
    with group axes after the blocked one runs its lattice phases in two halves
    split by axes (before / after the tiles), each covering the lattice once."""
    N = si.num_points(levels)
    for ph in _plan_passes(levels, inverse=inverse):
        if ph[0][0] != "FUSED":
            continue
        bt2 = [int(a["bt2"]) for _, a, _ in ph if "bt2" in a]
        if any(b >= 0 for b in bt2):
            # two-blocked: the tiles write the points fine along both axes; the
            # cross phases pass over every other point (some once per axis)
            main = max(p for _, _, p in ph)
            assert main < N <= sum(p for _, _, p in ph)
            continue
        skips = [int(a.get("skip", "0")) for _, a, _ in ph]
        if not any(skips):
            assert sum(p for _, _, p in ph) == N
            continue
        # dehierarchization with axes after the blocked one: the lattice phases
        # run twice, split by axes (split_inverse_lattice): T_k^B .. T_1^B, T_0,
        # T_1^A .. T_k^A; each half with the tiles covers every point once
        assert inverse
        main = max(range(len(ph)), key=lambda i: ph[i][2])
        assert skips[main] == 0
        before, after = ph[:main], ph[main + 1:]
        assert len(before) == len(after)
        assert [p for _, _, p in before] == [p for _, _, p in after][::-1]
        assert ph[main][2] + sum(p for _, _, p in after) == N
        a = ph[main][1]
        gl = [int(x) for x in a["levels"].strip("()").split(",")]
        jb = int(a["special"])
        low = sum(1 << k for k in range(jb + 1))
        high = sum(1 << k for k in range(jb + 1, len(gl)))
        assert all(sk == low for sk in skips[:main])        # B halves: axes <= jb skipped
        assert all(sk == high for sk in skips[main + 1:])   # A halves: axes > jb skipped


def test_plan_c2_c3_use_blocked_fusion():
    """C2 (8,8,8): x_1 whole rows x 2^5-row x_2 blocks in one round trip (+ its
    7-row coarse lattice), then x_3 -- 2.03 HBM passes instead of 3."""
    p = _plan_passes((8, 8, 8))
    assert len(p) == 2 and p[0][0][0] == "FUSED" and p[0][0][1]["special"] == "1" and p[0][0][1]["bt"] == "5"
    assert len(_plan_passes((8, 8, 8), fuse="whole")) == 3
    # C3: the contiguous axis blocked at 2^9 with x_2 whole (513-point runs, the
    # pipelined bulk-copy kernel), then x_3 and x_4..x_5 -- the round-2 cost
    # model prefers 3 passes on fast kernels to 2 passes whose tiles have
    # 33-point runs (97.7 vs 94.7 Gpoints/s, profiles/r02/README.md)
    p3 = _plan_passes((10, 4, 4, 4, 4))
    assert 2 <= len(p3) <= 3 and p3[0][0][0] == "FUSED" and p3[0][0][1]["special"] == "0"
    assert int(p3[0][0][1]["runlen"]) >= 128
    assert all(len(ph) == 1 for ph in _plan_passes((8, 8, 8), fuse=False)[:1])
    assert sgh.plan_describe((8, 8, 8), fuse=False).count("FUSED") == 0


def test_plan_two_blocked_available():
    """Two-blocked plans (SURVEY 8(a) a4 block scheme: both axes of a 2-D grid
    in aligned blocks, one round trip + cross phases) are chosen for C4's
    hierarchization (measured 169.6 vs 157.7 Gpoints/s per-axis) and, with
    its own phase order, for the dehierarchization (191.7 vs 124.2)."""
    p = _plan_passes((14, 13))
    assert len(p) == 1 and int(p[0][0][1]["bt2"]) >= 2
    N = si.num_points((14, 13))
    assert p[0][0][2] < N <= sum(x for _, _, x in p[0]) < 1.06 * N
    q = _plan_passes((14, 13), inverse=True)
    assert len(q) == 1
    tiles = [x for k, a, x in q[0] if a.get("bt2", "-1") != "-1" and a.get("levels") == "(14,13)"]
    assert len(tiles) == 1 and tiles[0] == p[0][0][2]          # the same fine-fine tiles
    assert N <= sum(x for _, _, x in q[0]) < 1.06 * N


@pytest.mark.parametrize("levels", [(5, 7, 9), (2, 2, 9, 9), (1, 5, 7, 9), (5, 1, 7, 9), (4, 6, 8), (2, 10, 10),
                                    (3, 4, 3), (2, 2, 2, 5, 5), (4, 4, 11)], ids=str)
def test_plan_prefix_two_blocked_partition(levels):
    """Prefix two-blocked hierarchization plans (>= 3 non-trivial axes): ONE
    pass whose phases -- the box tiles (fine along both blocked axes), then
    the classes coarse along {a}, {b}, {a, b} -- write every point exactly
    once; the first phase is the largest (the tiles).  The dehierarchization
    plan, where one exists, is six phases emitted in reverse execution order
    ({a}^B, tiles, {a}^A, T^B, {b}, T^A): the classes coarse along a and along
    both run in two halves (by axes), so tiles + {a} + {b} + {a, b} cover
    every point once."""
    N = si.num_points(levels)
    p = _plan_passes(levels, fuse="two_blocked")
    assert len(p) == 1 and int(p[0][0][1]["bt2"]) >= 2
    pts = [x for _, _, x in p[0]]
    assert sum(pts) == N and pts[0] == max(pts)
    sq = [l for l in levels if l > 1]
    assert all(a["levels"].count(",") == len(sq) - 1 for _, a, _ in p[0])
    q = _plan_passes(levels, inverse=True, fuse="two_blocked")
    inv_box = [ph for ph in q if len(ph) == 6 and any(int(a.get("bt2", "-1")) >= 0 for _, a, _ in ph)
               and all(a.get("levels", "").count(",") == len(sq) - 1 for _, a, _ in ph)]
    for ph in inv_box:
        pq = [x for _, _, x in ph]
        assert pq[0] == pq[2] and pq[3] == pq[5]
        assert pq[1] + pq[2] + pq[4] + pq[5] == N and pq[1] == max(pq)
        sk = [int(a.get("skip", "0")) for _, a, _ in ph]
        b_bit = 1 << (len(sq) - 1)
        assert sk[1] == 0 and sk[4] == 0 and sk[2] == sk[5] == b_bit and sk[0] == sk[3] == b_bit - 1


@pytest.mark.parametrize("levels,P", [((14, 13), 2), ((14, 13), 4), ((14, 13), 8), ((8, 8, 8), 2), ((8, 8, 8), 4)],
                         ids=str)
def test_sharded_plan_bytes_fused(levels, P):
    """Sharded paths: the fused halo hierarchization
    plans <= 1.3 x 16 B per point of a rank's shard (one box plan + the coarse
    rows), the unfused one ~2 passes; the all-to-all path's local axes are
    planned like a whole grid (plan_grid_rows), so C2's local part is ~1 pass
    (+ pack / unpack copies and the slab pass)."""
    N = si.num_points(levels)
    per = 16.0 * N / P
    fused = max(sgh.sharded_plan_bytes(levels, P, r, path="halo") for r in range(P))
    unfused = max(sgh.sharded_plan_bytes(levels, P, r, path="halo", fused=False) for r in range(P))
    assert fused <= 1.3 * per < unfused
    assert max(sgh.sharded_plan_bytes(levels, P, r, path="halo", inverse=True) for r in range(P)) == unfused
    a2a = max(sgh.sharded_plan_bytes(levels, P, r, path="a2a") for r in range(P))
    assert a2a <= 1.01 * (3 + (len(levels) - 1 if len(levels) < 3 else 1.1)) * per


def test_plan_w8_tiles_by_axis_count():
    """Cost model (DESIGN 7, "W = 8 column tiles at their measured rate"): runs
    of 8 doubles are fused only in tiles of few axes -- the largest C5 shapes
    fuse their two trailing axes in W = 8 tiles (2 round trips), S10 does not
    take a W = 8 tile of six 3-point axes (measured 1.75 TB/s: three passes)."""
    for levels in [(6, 6, 5, 5), (7, 5, 5, 5), (6, 6, 6, 4)]:
        p = _plan_passes(levels)
        assert len(p) == 2
        (kind, a, _), = p[1]
        assert kind == "FUSED" and a["W"] == "8" and a["levels"].count(",") == 1
    for l1 in (8, 9):
        p = _plan_passes((l1,) + (2,) * 9)
        assert len(p) == 3
        for ph in p:
            for kind, a, _ in ph:
                assert not (kind == "FUSED" and a["W"] == "8" and a["levels"].count(",") >= 3)


def test_plan_c5_single_pass_plans_partition():
    """Every C5 member whose hierarchization plan is ONE pass with a second
    blocked axis (two-blocked / prefix two-blocked) writes each point exactly
    once over its phases; every other FUSED pass without a split inverse does
    too (the planner's in-place invariant over the whole 4,255-grid set)."""
    n_box = 0
    for lv in si.combination_set(4, 22):
        N = si.num_points(lv)
        for ph in _plan_passes(lv):
            if ph[0][0] != "FUSED":
                continue
            if any(int(a.get("bt2", "-1")) >= 0 for _, a, _ in ph):
                if len([l for l in lv if l > 1]) >= 3:      # prefix two-blocked: a partition
                    n_box += 1
                    assert sum(p for _, _, p in ph) == N, lv
                continue
            assert sum(p for _, _, p in ph) == N, lv
    assert n_box >= 100


def test_plan_two_blocked_forced():
    """SGH_FLAG_TWO_BLOCKED (fuse="two_blocked") selects the two-blocked plan
    wherever one exists (how the GPU parity tests exercise it)."""
    for lv in [(14, 13), (10, 10), (11, 8), (1, 1, 11, 9)]:
        p = _plan_passes(lv, fuse="two_blocked")
        assert len(p) == 1 and int(p[0][0][1]["bt2"]) >= 2, lv
        N = si.num_points(lv)
        assert p[0][0][2] < N <= sum(x for _, _, x in p[0])
    assert len(_plan_passes((14, 13), inverse=True, fuse="two_blocked")) == 1


def test_library_reads_no_environment():
    """the default library reads no environment variable.  The only
    getenv in csrc/ is tuning_env()'s, compiled in a -DSGH_TUNING build only
    (experiments); the default build's tuning_env returns NULL.  (The
    statically linked CUDA runtime's own getenv calls are not ours.)"""
    import glob
    import re
    hits = []
    for path in glob.glob(os.path.join(os.path.dirname(sgh.__file__), "csrc", "*")):
        src = open(path).read()
        for m in re.finditer(r"\bgetenv\s*\(", src):
            hits.append((os.path.basename(path), src[:m.start()]))
    assert len(hits) == 1 and hits[0][0] == "sgh_plan.hpp", [h[0] for h in hits]
    before = hits[0][1]
    assert before.rfind("#ifdef SGH_TUNING") > before.rfind("#endif"), "getenv outside #ifdef SGH_TUNING"


@pytest.mark.parametrize("d,n", [(1, 9), (2, 7), (3, 8), (4, 22), (5, 9)])
def test_sparse_subspace_offsets(d, n):
    """sgh_sparse_num_subspaces / sgh_sparse_subspace_offset (host): the SG
    order enumerated directly (level sum ascending, then lexicographic, each
    W_lam of 2^{|lam|-d} points) gives the same offsets; the last is the total."""
    import itertools
    from math import comb
    import paper_1309_0392_b200 as sgh
    nsub = sgh.sparse_num_subspaces(d, n)
    assert nsub == comb(n, d)
    if nsub > 20000:
        idx = [0, 1, nsub // 3, nsub - 1, nsub]
    else:
        idx = list(range(nsub + 1))
    subs = []
    for s in range(d, n + 1):
        subs += sorted(c for c in itertools.product(range(1, s - d + 2), repeat=d) if sum(c) == s) if nsub <= 20000 else []
    if subs:
        off = [0]
        for lam in subs:
            off.append(off[-1] + (1 << (sum(lam) - d)))
        assert [sgh.sparse_subspace_offset(d, n, i) for i in idx] == off
    assert sgh.sparse_subspace_offset(d, n, nsub) == sgh.sparse_num_points(d, n)
    with pytest.raises(sgh.SGHError):
        sgh.sparse_subspace_offset(d, n, nsub + 1)


def test_combi_workspace_rejects_oversized_subspaces():
    """Gather plans are refused (workspace size 0) when a subspace would hold
    more than 2^30 points (n - d > 30) -- more than any grid can hold."""
    import ctypes
    lv = (ctypes.c_int32 * 1)(20)
    assert sgh.lib.sgh_combi_workspace_bytes(lv, 1, 1, 30, 0) > 0
    assert sgh.lib.sgh_combi_workspace_bytes(lv, 1, 1, 32, 0) == 0


def test_plan_two_blocked_inverse_phase_order():
    """Dehierarchization with two-blocked tiles (sgh_capi.cu plan_two_blocked):
    the plan lists, in the order the runner reverses, (5) the coarse-a columns'
    fine-b part (axis a skipped), (4) the tiles, (3) the b-lattice view, (2) the
    fine-a view of the coarse-b rows, (1) the a-lattice: a view for the
    coarse-b rows and the coarse-a-column tiles with axis b skipped."""
    q = _plan_passes((14, 13), inverse=True)
    assert len(q) == 1
    ph = q[0]
    kinds = [(k, a.get("skip"), a.get("bt2")) for k, a, _ in ph]
    assert kinds[0][0] == "FUSED" and kinds[0][1] == "1"                  # (5)
    assert kinds[1][0] == "FUSED" and kinds[1][1] == "0" and kinds[1][2] == "5"   # (4): the 257 x 33 tiles
    assert kinds[-1][0] == "FUSED" and kinds[-1][1] == "2"                # (1), fine-b rows
    assert all(k != "FUSED" for k, _, _ in kinds[2:-1])                   # (3), (2), (1) views
    assert ph[0][2] == ph[-1][2]                                          # same coarse-a columns
