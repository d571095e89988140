"""Representative cases for compute-sanitizer: every kernel kind, both directions,
fused and per-axis, batched and sharded-loopback, each checked bitwise against
the oracle.  Small sizes so memcheck / racecheck / synccheck finish quickly.

    compute-sanitizer --tool racecheck python scripts/sanitize_cases.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
import paper_1309_0392_b200 as sgh  # noqa: E402
import sgh_inputs as si  # noqa: E402

SHAPES = [(5, 5), (13,), (2, 13), (7, 12), (6, 6, 5, 5), (3, 4, 4, 2), (1, 1, 5, 5), (2, 2, 2, 2), (5, 3, 3),
          (10, 4, 4), (3, 2, 1, 2, 3, 2)]


def same(a, b):
    return np.array_equal(np.asarray(a).view(np.uint64), np.asarray(b).view(np.uint64))


bad = 0
for levels in SHAPES:
    N = si.num_points(levels)
    u = si.fill_uniform(N, grid_id=N % 1000)
    for inv in (False, True):
        for fuse in (True, False):
            g = torch.from_numpy(u).cuda()
            sgh.transform(g, levels, inverse=inv, fuse=fuse)
            want = (oracle.dehierarchize if inv else oracle.hierarchize)(u.copy(), levels)
            if not same(g.cpu().numpy(), want):
                print("MISMATCH", levels, inv, fuse)
                bad += 1
members = [(3, 4, 2), (1, 9, 1), (6, 5, 1), (2, 2, 7), (4, 4, 4)]
b = sgh.GridBatch(members)
b.fill_uniform(si.SEED)
b.hierarchize()
for gid, (lv, v) in enumerate(zip(members, b.views)):
    want = oracle.hierarchize(oracle.fill_uniform(si.num_points(lv), si.SEED, gid), lv)
    if not same(v.cpu().numpy(), want):
        print("MISMATCH batched", lv)
        bad += 1
levels, P = (6, 5), 4
u = si.fill_uniform(si.num_points(levels), grid_id=9)
C = si.num_points(levels) // ((1 << levels[-1]) - 1)
shards = []
for r in range(P):
    b0, e0 = sgh.shard_rows(levels, P, r)
    shards.append(torch.from_numpy(u[b0 * C:e0 * C].copy()).cuda())
ws = torch.empty(P * sgh.sharded_workspace_bytes(levels, P) // 8, dtype=torch.float64, device="cuda")
sgh.transform_sharded_loopback(shards, levels, ws)
if not same(torch.cat(shards).cpu().numpy(), oracle.hierarchize(u.copy(), levels)):
    print("MISMATCH sharded")
    bad += 1
torch.cuda.synchronize()
print("sanitize cases done, mismatches:", bad)
sys.exit(1 if bad else 0)
