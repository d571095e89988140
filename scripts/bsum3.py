"""Print a bench JSON line's headline, roofline and per-kernel shares."""
import json
import sys

for f in sys.argv[1:]:
    d = json.loads(open(f).read().strip().splitlines()[-1])
    r = d.get("roofline", {})
    print(f, round(d["value"], 1), d["ms_per_step"], r.get("kernel"), round(r.get("frac", 0), 3),
          d.get("model", {}).get("passes_per_point") if isinstance(d.get("model"), dict) else "")
    if "-k" in sys.argv[0:1] or len(sys.argv) == 2:
        for k, v in sorted(d.get("kernels", {}).items(), key=lambda kv: -kv[1]["share_of_step"]):
            print(f"   {k:22s} {v['launches_per_step']:5.1f} {v['share_of_step']:.3f} {v['GBps']:8.0f}")
