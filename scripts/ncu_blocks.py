"""Group an ncu source-page SASS listing into runs of equal execution count
(~basic blocks) and print the heaviest: where a kernel's instructions go.
Usage: python scripts/ncu_blocks.py report.ncu-rep [kernel-regex] [launch-skip] [N]"""
import csv
import subprocess
import sys

rep = sys.argv[1]
rx = sys.argv[2] if len(sys.argv) > 2 else "."
skip = sys.argv[3] if len(sys.argv) > 3 else "0"
N = int(sys.argv[4]) if len(sys.argv) > 4 else 15
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", f"regex:{rx}", "--launch-skip", skip,
                      "--launch-count", "1"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = rows[1]
body = []
for r in rows[2:]:
    if len(r) != len(hdr) or r[0] == "Address":
        if body:
            break
        continue
    body.append(r)
ii = hdr.index("Instructions Executed")
iss = hdr.index("Warp Stall Sampling (All Samples)")
blocks, cur = [], None
for k, r in enumerate(body):
    n = int(float(r[ii] or 0))
    if cur and cur[1] == n:
        cur[2] += 1
        cur[3].append(r[1].strip())
        cur[4] += float(r[iss] or 0)
    else:
        cur = [k, n, 1, [r[1].strip()], float(r[iss] or 0)]
        blocks.append(cur)
tot = sum(b[1] * b[2] for b in blocks)
ts = sum(b[4] for b in blocks) or 1
print(f"{rows[0][1][:80]}  warp-instructions {tot}")
for b in sorted(blocks, key=lambda b: -b[1] * b[2])[:N]:
    print(f"@{b[0]:5d} exec {b[1]:9d} x {b[2]:3d} = {100 * b[1] * b[2] / tot:5.1f}% inst {100 * b[4] / ts:5.1f}% stall"
          f"  {' | '.join(b[3][:5])[:120]}")
