"""One-line summaries of bench JSON files: value, dominant kernel, per-kernel share/GB/s."""
import json
import sys

for f in sys.argv[1:]:
    try:
        d = json.load(open(f))
    except Exception as e:  # noqa: BLE001
        print(f, "unreadable", e)
        continue
    ks = {k: (round(v["share_of_step"], 3), round(v["GBps"])) for k, v in d.get("kernels", {}).items()}
    r = d.get("roofline", {})
    print(f"{f}: {d['value']:.1f} {d['unit']} ms={d['ms_per_step']:.3f} dom={r.get('kernel')} "
          f"frac={r.get('frac', 0):.3f} clocks={d.get('clocks', {}).get('sm_mhz')} {ks}")
