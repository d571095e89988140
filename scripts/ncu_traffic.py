"""Per-kernel-key DRAM traffic from an ncu launch list, for bench.py's
roofline "traffic" field (profiles/ncu_traffic.json).

  python scripts/ncu_traffic.py launches.csv keys.json [profiles/ncu_traffic.json]

launches.csv: `ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
--csv --log-file launches.csv -k regex:"k_(fused|flat|strided|reg|fpipe)" -s <warmup x launches/step>
-c <launches/step> python bench.py ...` (one step's transform launches, in order);
keys.json: `python bench.py ... --dump-launch-keys keys.json` (the same step's kernel keys, in order).
Each key gets the average dram read + write bytes per launch."""
import csv
import json
import sys
from collections import defaultdict


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr_i = next(i for i, r in enumerate(rows) if "Metric Name" in r)
    hdr = rows[hdr_i]
    iid, iname, imet, ival, iunit = (hdr.index(c) for c in ("ID", "Kernel Name", "Metric Name", "Metric Value",
                                                            "Metric Unit"))
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3}
    out = {}
    for r in rows[hdr_i + 1:]:
        if len(r) <= ival:
            continue
        k = int(r[iid])
        d = out.setdefault(k, {"name": r[iname]})
        d[r[imet]] = float(r[ival].replace(",", "")) * scale.get(r[iunit], 1)
    return [out[k] for k in sorted(out)]


def main():
    L = launches(sys.argv[1])
    K = json.load(open(sys.argv[2]))
    dst = sys.argv[3] if len(sys.argv) > 3 else None
    keys = K["keys"]
    if len(L) != len(keys):
        sys.exit(f"launch count mismatch: ncu {len(L)} vs bench {len(keys)}")
    acc = defaultdict(lambda: {"launches": 0, "dram_bytes": 0.0, "algorithmic_bytes": 0.0, "ncu_ms": 0.0})
    for l, k, ab in zip(L, keys, K["algorithmic_bytes"]):
        a = acc[k]
        a["launches"] += 1
        a["dram_bytes"] += l.get("dram__bytes_read.sum", 0) + l.get("dram__bytes_write.sum", 0)
        a["algorithmic_bytes"] += ab
        a["ncu_ms"] += 1e3 * l.get("gpu__time_duration.sum", 0)
    res = {k: {"traffic_bytes_per_launch": v["dram_bytes"] / v["launches"],
               "algorithmic_bytes_per_launch": v["algorithmic_bytes"] / v["launches"],
               "traffic_over_algorithmic": v["dram_bytes"] / max(1.0, v["algorithmic_bytes"]),
               "launches_per_step": v["launches"], "ncu_ms_per_step": v["ncu_ms"]} for k, v in acc.items()}
    total = sum(v["ncu_ms"] for v in acc.values())
    for k, v in sorted(res.items(), key=lambda kv: -kv[1]["ncu_ms_per_step"]):
        print(f"{k:14s} share {v['ncu_ms_per_step'] / total:6.1%}  traffic/alg {v['traffic_over_algorithmic']:.3f}  "
              f"{v['traffic_bytes_per_launch'] / 1e9:.3f} GB/launch")
    if dst:
        try:
            db = json.load(open(dst))
        except Exception:  # noqa: BLE001
            db = {}
        db[K["workload"] + ("_dehier" if K.get("inverse") else "")] = res
        json.dump(db, open(dst, "w"), indent=1, sort_keys=True)


if __name__ == "__main__":
    main()
