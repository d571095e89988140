"""Per CUDA source line: warp-stall samples and warp instructions of one kernel
in an ncu report (needs -lineinfo).  Usage: python scripts/ncu_lines.py rep [regex] [N]"""
import csv, subprocess, sys
rep = sys.argv[1]
rx = sys.argv[2] if len(sys.argv) > 2 else "."
N = int(sys.argv[3]) if len(sys.argv) > 3 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass", "-k", f"regex:{rx}",
                      "--launch-count", "1"], capture_output=True, text=True).stdout
fname, rows, hdr = None, [], None
for r in csv.reader(out.splitlines()):
    if len(r) == 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr and len(r) == len(hdr) and r[0] not in ("", "-"):
        rows.append((fname, r))
i_s = hdr.index("Warp Stall Sampling (All Samples)")
i_i = hdr.index("Instructions Executed")
tot = sum(float(r[i_s] or 0) for _, r in rows)
tin = sum(float(r[i_i] or 0) for _, r in rows)
print(f"samples {tot:.0f}  warp-instructions {tin:.0f}")
for f, r in sorted(rows, key=lambda fr: -float(fr[1][i_s] or 0))[:N]:
    print(f"{100*float(r[i_s] or 0)/tot:5.1f}%  {100*float(r[i_i] or 0)/tin:5.1f}%i  {f}:{r[0]:<5} {r[1].strip()[:90]}")
