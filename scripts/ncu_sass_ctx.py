"""SASS context around given instruction indices of an ncu report (source page).
Usage: python scripts/ncu_sass_ctx.py report.ncu-rep kernel-regex idx[,idx..] [radius]"""
import csv, subprocess, sys
rep, rx, idxs = sys.argv[1], sys.argv[2], [int(x) for x in sys.argv[3].split(",")]
rad = int(sys.argv[4]) if len(sys.argv) > 4 else 8
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", f"regex:{rx}", "--launch-count", "1"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = rows[1]
body = [r for r in rows[2:] if len(r) == len(hdr) and r[0] != "Address"]
i_s = hdr.index("Warp Stall Sampling (All Samples)")
i_i = hdr.index("Instructions Executed")
for k in idxs:
    print("----", k)
    for j in range(max(0, k - rad), min(len(body), k + rad + 1)):
        r = body[j]
        print(f"{j:5d} {r[i_s]:>8} {r[i_i]:>10}  {r[1].strip()[:100]}")
