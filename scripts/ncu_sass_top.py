"""Top SASS instructions by warp-stall samples from an ncu report (source page).
Usage: python scripts/ncu_sass_top.py report.ncu-rep [kernel-regex] [launch-index] [N]"""
import csv
import subprocess
import sys

rep = sys.argv[1]
rx = sys.argv[2] if len(sys.argv) > 2 else "."
skip = sys.argv[3] if len(sys.argv) > 3 else "0"
N = int(sys.argv[4]) if len(sys.argv) > 4 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", f"regex:{rx}", "--launch-skip", skip,
                      "--launch-count", "1"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
print(rows[0][:2])
hdr = rows[1]
body = []
for r in rows[2:]:
    if len(r) != len(hdr) or r[0] == "Address":
        if body:
            break                      # next kernel's table
        continue
    body.append(r)
i_s = hdr.index("Warp Stall Sampling (All Samples)")
i_n = hdr.index("Warp Stall Sampling (Not-issued Samples)")
i_i = hdr.index("Instructions Executed")
tot = sum(float(r[i_s] or 0) for r in body)
tin = sum(float(r[i_i] or 0) for r in body)
print(f"samples {tot:.0f}  warp-instructions {tin:.0f}")
for k, r in sorted(enumerate(body), key=lambda kr: -float(kr[1][i_s] or 0))[:N]:
    print(f"{k:5d} {100 * float(r[i_s]) / tot:5.1f}% stall {100*float(r[i_n] or 0)/tot:5.1f}% notiss  inst {r[i_i]:>9}  {r[1].strip()[:90]}")
