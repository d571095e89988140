"""Summarise bench JSON lines: value, ms, roofline frac and the per-kernel table."""
import json, sys
for f in sys.argv[1:]:
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
    except Exception as e:
        print(f, "unreadable", e); continue
    rf = d.get("roofline") or {}
    print(f"{f}: {d['value']:.1f} {d['unit']}  {d['ms_per_step']:.3f} ms  frac={rf.get('frac')}  dom={rf.get('kernel')}")
    for k in (d.get("kernels") or [])[:8]:
        print("   ", k)
