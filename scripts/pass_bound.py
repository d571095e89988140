"""Lower bound on HBM round trips per point for the C5 set with on-chip tiles
of at most T points ("How many passes are possible").

A pass reads and writes a point once.  In one pass a tile can finish a point
only if the tile holds, along every non-trivial axis, either the whole pole
(extent n_k = 2^l_k - 1) or an aligned block with its two ends (extent
2^t_k + 1), and the point is fine along every blocked axis: the fraction of
points a pass can finish is at most max prod_k f_k over tile shapes with
prod_k e_k <= T (f_k = 1 whole, 1 - 2^-t_k blocked).  Every other point needs
at least one more pass, so passes >= 2 - max_fraction per grid.
    python scripts/pass_bound.py [T]"""
import itertools
import sys

sys.path.insert(0, ".")
import sgh_inputs as si  # noqa: E402

T = int(sys.argv[1]) if len(sys.argv) > 1 else 8704
members = si.combination_set(4, 22)
tot = acc = 0.0
by_d = {}
for lv in members:
    N = si.num_points(lv)
    axes = [l for l in lv if l > 1]
    opts = []
    for l in axes:
        o = [((1 << l) - 1, 1.0)]                           # whole pole
        o += [((1 << t) + 1, 1.0 - 2.0 ** -t) for t in range(1, l)]   # blocked, t < l
        opts.append(o)
    best = 0.0
    for combo in itertools.product(*opts):
        e = 1
        for ext, _ in combo:
            e *= ext
        if e <= T:
            f = 1.0
            for _, fr in combo:
                f *= fr
            best = max(best, f)
    bound = 1.0 if best >= 1.0 else 2.0 - best
    tot += N
    acc += N * bound
    de = len(axes)
    a = by_d.setdefault(de, [0.0, 0.0])
    a[0] += N
    a[1] += N * bound
print(f"T = {T} points per tile: passes per point >= {acc / tot:.3f} (point-weighted over C5)")
for de in sorted(by_d):
    print(f"  d_eff = {de}: {by_d[de][0] / tot:6.1%} of the points, bound {by_d[de][1] / by_d[de][0]:.3f}")
