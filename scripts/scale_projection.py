"""Multi-GPU projection for C5 on ONE B200 (the pool gives one GPU per call).

C5 shards with no data-path collective: rank r of N
transforms its LPT share of the grids, alone on its GPU, and the job's time
is the slowest rank's.  So timing every rank's share on one GPU, one after the
other, gives each rank's device time on its own GPU exactly (same hardware,
no communication); the projected aggregate is total points / max over ranks.
Not a bench value (bench.py --gpus N on N GPUs is); a planning aid for the
SCALE run.  One JSON line per N.
    python scripts/scale_projection.py [--steps 10] [--ns 1,2,4,8]"""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1309_0392_b200 as sgh  # noqa: E402
import sgh_inputs as si  # noqa: E402


def time_share(members, ids, steps):
    b = sgh.GridBatch(members, grid_ids=ids)
    b.fill_uniform(si.SEED)
    for _ in range(3):
        b.hierarchize()
    torch.cuda.synchronize()
    st = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for _ in range(steps):
        b.hierarchize()
    e1.record(st)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / steps
    del b
    torch.cuda.empty_cache()
    return ms


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--ns", default="1,2,4,8")
    ap.add_argument("--by", default="time", choices=["time", "points"],
                    help="LPT weights: the planner's estimated time (bench.py's partition) or points")
    a = ap.parse_args()
    members = si.combination_set(4, 22)
    sizes = [si.num_points(l) for l in members]
    total = sum(sizes)
    base = None
    weights = [sgh.plan_cost(lv) for lv in members] if a.by == "time" else sizes
    for n in [int(x) for x in a.ns.split(",")]:
        parts = si.lpt_partition(weights, n)
        ms = [time_share([members[i] for i in p], list(p), a.steps) for p in parts]
        worst = max(ms)
        val = total / (worst * 1e-3) / 1e9
        if n == 1:
            base = val
        print(json.dumps({"n_gpus": n, "rank_ms": ms, "max_ms": worst, "mean_ms": sum(ms) / len(ms),
                          "projected_Gpoints_s": val, "efficiency_vs_1": (val / (n * base)) if base else None,
                          "points_per_rank_max_over_mean": max(sum(sizes[i] for i in p) for p in parts) * n / total}),
              flush=True)


if __name__ == "__main__":
    main()
