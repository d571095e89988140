"""Probe: per-kernel throughput when the grid is L2-resident vs HBM-resident.

Runs the per-axis kernels repeatedly on grids of increasing size and prints the
event-timed GB/s per kernel kind (16 B per point per pass).  A grid well below
the 126 MB L2 stays resident between launches, so its numbers show the L2-bound
throughput of the same kernels.
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1309_0392_b200 as sgh  # noqa: E402
import sgh_inputs as si  # noqa: E402

out = []
for levels in [(6, 6, 6), (7, 7, 7), (8, 7, 7), (8, 8, 7), (8, 8, 8), (9, 9, 9)]:
    b = sgh.GridBatch([levels])
    b.fill_uniform(1)
    for _ in range(3):
        b.hierarchize()
    torch.cuda.synchronize()
    sgh.profile_enable(True)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    reps = 20
    for _ in range(reps):
        b.hierarchize()
    e1.record()
    torch.cuda.synchronize()
    recs = sgh.profile_read()
    sgh.profile_enable(False)
    per = {}
    for r in recs:
        a = per.setdefault(r["kernel"], [0.0, 0.0])
        a[0] += r["bytes"]
        a[1] += r["ms"]
    N = si.num_points(levels)
    step_ms = e0.elapsed_time(e1) / reps
    row = {"levels": levels, "MB": 8 * N / 1e6, "step_ms": step_ms,
           "per_axis_GBps": 16 * 3 * N / (step_ms * 1e-3) / 1e9,
           "kernels": {k: v[0] / (v[1] * 1e-3) / 1e9 for k, v in per.items()},
           "kernel_ms_sum": sum(v[1] for v in per.values()) / reps}
    out.append(row)
    print(json.dumps(row), flush=True)
    del b
    torch.cuda.empty_cache()
json.dump(out, open(sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/l2_probe.json", "w"), indent=1)
