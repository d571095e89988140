"""Repeat the whole C5 set (4,255 grids, 41 GB) through the batched transform
and compare the per-grid digests of every run with the oracle-derived golden
sums (tests/golden): a race in the pipelined kernels (k_fpipe's mbarrier ring,
the grouped launches) would show as a run whose digests differ.  compute-
sanitizer is closed on the GPU pool; this is the stand-in for racecheck at
full load.  Usage: python scripts/stress_c5.py [iters]"""
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1309_0392_b200 as sgh  # noqa: E402
import sgh_inputs as si  # noqa: E402

iters = int(sys.argv[1]) if len(sys.argv) > 1 else 10
GOLD = os.path.join(ROOT, "tests", "golden")
SD = json.load(open(os.path.join(GOLD, "survey_digests.json")))
OD = json.load(open(os.path.join(GOLD, "c5_oracle_digests.json")))
cs = si.combination_set(4, 22)
b = sgh.GridBatch(cs)
bad = 0
first = {}
for it in range(iters):
    b.fill_uniform(SD["seed"])
    b.hierarchize()
    dh = b.digests()
    ok_h = sum(dh) % (1 << 64) == int(SD["C5"]["sum_hierarchized"], 16) and dh == first.setdefault("h", dh)
    b.dehierarchize()
    dr = b.digests()
    ok_r = sum(dr) % (1 << 64) == int(OD["sum_round_trip"], 16) and dr == first.setdefault("r", dr)
    torch.cuda.synchronize()
    if not (ok_h and ok_r):
        bad += 1
        nh = sum(x != y for x, y in zip(dh, first["h"]))
        nr = sum(x != y for x, y in zip(dr, first["r"]))
        print(f"iter {it}: hier ok={ok_h} ({nh} grids differ), round trip ok={ok_r} ({nr} grids differ)", flush=True)
print(f"stress_c5: {iters} iterations x (hierarchize + dehierarchize) over {len(cs)} grids, {bad} bad", flush=True)
sys.exit(1 if bad else 0)
