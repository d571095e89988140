"""Timeline of k_fpipe from a -DSGH_PIPE_TRACE build (diagnostic only).
Usage: SGH_LIB_PATH=.../var_trace.so python scripts/pipe_trace.py [C5|C4] [min_tiles]"""
import ctypes
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_1309_0392_b200 as sgh  # noqa: E402
import sgh_inputs as si  # noqa: E402

w = sys.argv[1] if len(sys.argv) > 1 else "C5"
min_tiles = int(sys.argv[2]) if len(sys.argv) > 2 else 100000
f = sgh.lib.sgh_debug_pipe_trace
f.restype = ctypes.c_int64
f.argtypes = [ctypes.c_int64, ctypes.c_void_p, ctypes.c_int64]
if w == "C5":
    b = sgh.GridBatch(si.combination_set(4, 22))
    b.fill_uniform(si.SEED)
    run = b.hierarchize
else:
    g = torch.empty(si.num_points((14, 13)), dtype=torch.float64, device="cuda")
    sgh.fill_uniform(g, si.SEED)
    run = lambda: sgh.hierarchize(g, (14, 13))  # noqa: E731
run()
torch.cuda.synchronize()
n = f(min_tiles, None, 0)
run()
torch.cuda.synchronize()
buf = np.zeros(n, dtype=np.uint64)
f(0, buf.ctypes.data, n)
R = buf.reshape(160, 64, 24)
T = R[:, :, :8].astype(np.float64)
A = R[:, :, 8:16].astype(np.float64)
I = R[:, :, 16:24]
ok = (T > 0).all(axis=2)
print("traced tiles:", int(ok.sum()))
T = T[:, 8:56]                     # skip ramp-up / tail
ok = ok[:, 8:56]
t = T[ok]
d = lambda a, b: (t[:, b] - t[:, a]) / 1000.0   # noqa: E731  (us)
rows = [("desc published -> producer starts", 0, 1), ("producer issue time", 1, 2),
        ("issued -> data ready (seen by consumer)", 2, 4), ("consumer wait (3->4)", 3, 4),
        ("compute (4->5)", 4, 5), ("computed -> stores issued", 5, 6), ("store read drain (6->7)", 6, 7),
        ("producer start -> empty next (1->7)", 1, 7)]
for name, a, b2 in rows:
    x = d(a, b2)
    print(f"{name:42s} median {np.median(x):7.2f} us  p10 {np.percentile(x, 10):7.2f}  p90 {np.percentile(x, 90):7.2f}")
# per-CTA tile period
per = np.diff(T[:, :, 2], axis=1)[ok[:, 1:] & ok[:, :-1]] / 1000.0
print(f"{'tile period (producer issue to issue)':42s} median {np.median(per):7.2f} us")

# per-axis transform time by (axis level, role) over the traced tiles
from collections import defaultdict  # noqa: E402
acc = defaultdict(list)
tiles = defaultdict(list)
T = R[:, :, :8].astype(np.float64)
for c in range(160):
    for k in range(8, 56):
        if not (R[c, k, :8] > 0).all():
            continue
        m = int(I[c, k, 0])
        lv = [(int(I[c, k, 1]) >> (8 * j)) & 255 for j in range(m)]
        bj, bt, bt2 = (np.int64(I[c, k, 2]), np.int64(I[c, k, 3]), np.int64(I[c, k, 4]))
        P, units = int(I[c, k, 5]), int(I[c, k, 6])
        t_prev = T[c, k, 4]
        key = (tuple(lv), int(bj), int(bt), int(bt2))
        tiles[key].append((T[c, k, 5] - T[c, k, 4]) / 1000.0)
        for j in range(m):
            if A[c, k, j] > 0:
                role = "blocked" if (j == bj and bt < lv[j]) or (bt2 >= 0 and j == bj + 1) else "whole"
                acc[(lv[j], role)].append((A[c, k, j] - t_prev) / 1000.0)
                t_prev = A[c, k, j]
print("per-axis time (us) by (level, role): median, count")
for key in sorted(acc):
    x = np.array(acc[key])
    print(f"  l={key[0]:2d} {key[1]:8s} median {np.median(x):6.2f}  n={len(x)}")
print("tile compute (us) by task shape (levels, bj, bt, bt2): top 12 by count")
for key, v in sorted(tiles.items(), key=lambda kv: -len(kv[1]))[:12]:
    print(f"  {key}  median {np.median(v):6.2f}  n={len(v)}")
