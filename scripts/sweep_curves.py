"""Paper-shaped size sweeps: throughput of
hierarchization vs. grid size for
  S1  -- 1-D grids l = 10..27 (Fig. fig:1DLayouts; "1 GB when
         |l|_1 = 27"), and
  S10 -- 10-D grids (l_1, 2, ..., 2), l_1 = 1..9 (Fig. fig:10D),
with the same timing protocol as bench.py (warm-up, CUDA events on the work
stream, L2 flushed before every step when the grid is < 1 GB) and the
dominant kernel's share and GB/s from a second, per-launch-profiled pass.
One JSON line per size on stdout.

    python scripts/sweep_curves.py [S1|S10|both] [--steps 10] [--inverse]
"""
import argparse
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1309_0392_b200 as sgh  # noqa: E402
import sgh_inputs as si  # noqa: E402


def measure(levels, steps, inverse, peak):
    N = si.num_points(levels)
    g = torch.empty(N, dtype=torch.float64, device="cuda")
    sgh.fill_uniform(g, si.SEED)
    flush = 8 * N < 1e9
    scratch = torch.empty((256 << 20) // 8, dtype=torch.float64, device="cuda") if flush else None
    st = torch.cuda.current_stream()

    def run(k):
        ms = 0.0
        for i in range(k):
            if flush:
                scratch.fill_(float(i))
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(st)
            sgh.transform(g, levels, inverse=inverse)
            b.record(st)
            torch.cuda.synchronize()
            ms += a.elapsed_time(b)
        return ms / k

    run(3)
    ms = run(steps)
    sgh.profile_enable(True)
    ms_p = run(steps)
    recs = sgh.profile_read()
    sgh.profile_enable(False)
    per = {}
    for r in recs:
        a = per.setdefault(r["kernel"], [0.0, 0.0])
        a[0] += r["ms"]
        a[1] += r["bytes"]
    dom = max(per, key=lambda k: per[k][0]) if per else None
    passes = sum(int(x.split("=")[1]) for x in sgh.plan_describe(levels, inverse=inverse).split()
                 if x.startswith("points=")) / N
    out = {"levels": list(levels), "points": N, "bytes": 8 * N, "ms": ms, "Gpoints_s": N / ms / 1e6,
           "passes_per_point": passes, "plan_GBps": 16 * passes * N / ms / 1e6,
           "plan_frac": 16 * passes * N / ms / 1e6 / peak, "l2_flushed": flush}
    if dom:
        out.update(dominant=dom, dominant_share=per[dom][0] / (ms_p * steps),
                   dominant_GBps=per[dom][1] / per[dom][0] / 1e6,
                   dominant_frac=per[dom][1] / per[dom][0] / 1e6 / peak)
    del g, scratch
    torch.cuda.empty_cache()
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("which", nargs="?", default="both", choices=["S1", "S10", "both"])
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--inverse", action="store_true")
    a = ap.parse_args()
    try:
        peak = float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"])
    except Exception:  # noqa: BLE001
        peak = 6650.0
    sizes = []
    if a.which in ("S1", "both"):
        sizes += [("S1", (l,)) for l in range(10, 28)]
    if a.which in ("S10", "both"):
        sizes += [("S10", (l,) + (2,) * 9) for l in range(1, 10)]
    for name, lv in sizes:
        r = measure(lv, a.steps, a.inverse, peak)
        r["sweep"] = name
        r["inverse"] = a.inverse
        print(json.dumps(r), flush=True)


if __name__ == "__main__":
    main()
