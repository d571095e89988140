"""Summarise an ncu --csv launch list (gpu__time_duration + dram bytes) by kernel.

    python scripts/ncu_launches.py <launches.csv> [first_id last_id]
"""
import collections
import csv
import sys

SCALE = {"ns": 1e-9, "us": 1e-6, "ms": 1e-3, "byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3,
         "second": 1}
lines = [ln for ln in open(sys.argv[1]) if ln.startswith('"')]
rows = list(csv.reader(lines))
hdr, data = rows[0], rows[1:]
ix = {k: hdr.index(k) for k in ("ID", "Kernel Name", "Metric Name", "Metric Unit", "Metric Value", "Grid Size")}
launch = collections.OrderedDict()
for r in data:
    d = launch.setdefault(int(r[ix["ID"]]), {"k": r[ix["Kernel Name"]].split("(")[0].replace("void ", "")})
    d[r[ix["Metric Name"]]] = float(r[ix["Metric Value"]].replace(",", "")) * SCALE.get(r[ix["Metric Unit"]], 1)
lo, hi = (int(sys.argv[2]), int(sys.argv[3])) if len(sys.argv) > 3 else (min(launch), max(launch))
tot = collections.defaultdict(lambda: [0, 0.0, 0.0])
T = 0.0
for i, d in launch.items():
    if not lo <= i <= hi:
        continue
    a = tot[d["k"]]
    a[0] += 1
    t = d.get("gpu__time_duration.sum", 0.0)
    a[1] += t
    a[2] += d.get("dram__bytes_read.sum", 0.0) + d.get("dram__bytes_write.sum", 0.0)
    T += t
print(f"launches {lo}..{hi}: total kernel time {T * 1e3:.2f} ms")
print(f"{'kernel':34s} {'n':>4s} {'ms':>9s} {'share':>6s} {'DRAM GB':>9s} {'GB/s':>7s}")
for k, (n, t, b) in sorted(tot.items(), key=lambda x: -x[1][1]):
    print(f"{k:34s} {n:4d} {t * 1e3:9.3f} {100 * t / T:5.1f}% {b / 1e9:9.3f} {b / t / 1e9 if t else 0:7.0f}")
