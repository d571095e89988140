"""SURVEY 8(f) 4 ablation (report only): the paper's BFS layout of a 1-D pole
 vs. the row-major layout the product keeps, on B200.
1-D grids l = 20..27; CUDA events per call, L2 flushed before each timed call
below 1 GB.  BFS hierarchization is out of place (one pass, reading each
point's two predecessors from coarser levels), BFS dehierarchization one
launch per level in place; the row-major path is sgh.transform (FLAT_BLOCKS
tiles + coarse lattice).  One JSON line per (level, layout, direction).
    python scripts/ablation_bfs.py [--steps 10]"""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1309_0392_b200 as sgh  # noqa: E402
import sgh_inputs as si  # noqa: E402


def timed(fn, steps, flush):
    st = torch.cuda.current_stream()
    scratch = torch.empty((256 << 20) // 8, dtype=torch.float64, device="cuda") if flush else None
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    ms = 0.0
    for i in range(steps):
        if flush:
            scratch.fill_(float(i))
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        fn()
        b.record(st)
        torch.cuda.synchronize()
        ms += a.elapsed_time(b)
    return ms / steps


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=10)
    a = ap.parse_args()
    for l in range(20, 28):
        N = (1 << l) - 1
        g = torch.empty(N, dtype=torch.float64, device="cuda")
        sgh.fill_uniform(g, si.SEED)
        bfs = torch.empty_like(g)
        out = torch.empty_like(g)
        sgh.bfs_permute_1d(g, bfs, l, to_bfs=True)
        flush = 8 * N < 1e9
        rows = [("row-major", "hier", lambda: sgh.transform(g, (l,))),
                ("row-major", "dehier", lambda: sgh.transform(g, (l,), inverse=True)),
                ("bfs", "hier", lambda: sgh.bfs_hierarchize_1d(bfs, out, l)),
                ("bfs", "dehier", lambda: sgh.bfs_dehierarchize_1d(bfs, l))]
        for layout, d, fn in rows:
            ms = timed(fn, a.steps, flush)
            print(json.dumps({"level": l, "points": N, "layout": layout, "direction": d, "ms": ms,
                              "Gpoints_s": N / ms / 1e6, "GBps_16B_per_point": 16 * N / ms / 1e6}), flush=True)
        del g, bfs, out
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
