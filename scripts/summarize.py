"""Summarise bench JSON lines: python scripts/summarize.py gpurun_out/<tag>/bench_*.json"""
import json
import sys

for f in sys.argv[1:]:
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
    except Exception as e:  # noqa: BLE001
        print(f, "unreadable:", e)
        continue
    m = d.get("model", {})
    r = d.get("roofline") or {}
    print(f"{f}: {d['value']:.1f} {d['unit']}  {d['ms_per_step']:.3f} ms/step  per-axis {m.get('per_axis_GBps') or 0:.0f} GB/s "
          f"({(m.get('per_axis_frac') or 0)*100:.1f}%)  dom={r.get('kernel')} {r.get('achieved', 0):.0f} GB/s "
          f"({r.get('frac', 0)*100:.1f}%) launches={d.get('gpu_launches')} clk={d.get('clocks', {}).get('sm_mhz')}")
    for k, v in (d.get("kernels") or {}).items():
        print(f"     {k:12s} {v['launches_per_step']:5.1f}/step share {v['share_of_step']*100:5.1f}%  {v['GBps'] or 0:7.0f} GB/s")
    if d.get("e2e"):
        print(f"     e2e {d['e2e']['value']:.2f} {d['e2e']['unit']} ({d['e2e'].get('ms_per_step', 0):.0f} ms/step)")
    if d.get("cpu_baseline"):
        print(f"     cpu {d['cpu_baseline']['value']:.3f} on {d['cpu_baseline']['cores']} cores")
