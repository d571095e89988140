"""One-kernel summary of an `ncu --set full --import-source on` report for profiles/:
raw metrics (time, DRAM bytes, launch shape, occupancy, issue rate), warp-stall
reasons, the SASS opcode mix and the hottest source lines.

    python scripts/ncu_summary.py report.ncu-rep [peak_GBps] > profiles/rNN/ncu_<kernel>.txt
"""
import collections
import csv
import re
import subprocess
import sys

rep = sys.argv[1]
peak = float(sys.argv[2]) if len(sys.argv) > 2 else None


def ncu(*args):
    return subprocess.run(["ncu", "-i", rep, *args], capture_output=True, text=True).stdout


rows = list(csv.reader(ncu("--page", "raw", "--csv").splitlines()))
hdr, unit, val = rows[0], rows[1], rows[2]
col = {h: i for i, h in enumerate(hdr)}


def num(name):
    return float(val[col[name]].replace(",", "")) if name in col and val[col[name]] not in ("", "n/a") else None


print(f"# {val[col['Kernel Name']]}  grid {val[col['Grid Size']]} x block {val[col['Block Size']]}")
want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
        "launch__registers_per_thread", "launch__shared_mem_per_block_dynamic", "launch__occupancy_limit_shared_mem",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "smsp__inst_executed.sum", "smsp__inst_executed_op_ldgsts.sum",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum", "l1tex__t_sectors_pipe_lsu_mem_global_op_st.sum"]
for w in want:
    if w in col:
        print(f"  {w:62s} {val[col[w]]:>18s} {unit[col[w]]}")
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-9, "us": 1e-6, "ms": 1e-3, "s": 1,
         "nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3, "second": 1}
try:
    b = sum(num(k) * scale[unit[col[k]]] for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"))
    t = num("gpu__time_duration.sum") * scale[unit[col["gpu__time_duration.sum"]]]
    line = f"  => DRAM {b / 1e9:.2f} GB in {t * 1e3:.3f} ms = {b / t / 1e9:.0f} GB/s"
    if peak:
        line += f" = {b / t / 1e9 / peak:.3f} of the measured copy peak ({peak} GB/s)"
    print(line + "  (under ncu: cold cache, serialised)")
except Exception as e:  # noqa: BLE001
    print("  (no DRAM rate:", e, ")")

# warp-stall reasons (sampled)
st = {}
for h in hdr:
    m = re.match(r"smsp__pcsamp_warps_issue_stalled_(\w+?)(_not_issued)?$", h)
    if m and not m.group(2) and num(h):
        st[m.group(1)] = num(h)
tot = sum(st.values())
if tot:
    print("\nWarp-stall samples by reason:")
    for k, v in sorted(st.items(), key=lambda kv: -kv[1])[:9]:
        print(f"  {100 * v / tot:5.1f} %  {k}")

# SASS opcode mix and source lines
out = ncu("--page", "source", "--csv", "--print-source=cuda,sass")
fname, hdr2, lines = None, None, []
ops = collections.Counter()
for r in csv.reader(out.splitlines()):
    if len(r) == 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":                    # "Line No","Source","Address","Source",<metrics...>
        hdr2 = r
        i_sm = r.index("Warp Stall Sampling (All Samples)")
        i_ex = r.index("Instructions Executed")
        continue
    if not hdr2 or len(r) != len(hdr2):
        continue
    try:
        ex = float(r[i_ex].replace(",", "") or 0)
        sm = float(r[i_sm].replace(",", "") or 0)
    except ValueError:
        continue
    if r[0] == "":                                 # a SASS row: address, instruction
        m = re.match(r"\s*(?:@!?U?P\w+\s+)?([A-Z0-9_]+)", r[3])
        if m:
            ops[m.group(1)] += ex
    else:                                          # a CUDA source row: line number, text
        lines.append((sm, ex, fname, r[0], r[1].strip()))
tot_ops = sum(ops.values())
if tot_ops:
    print("\nSASS warp instructions executed by opcode (top 14):")
    for k, v in ops.most_common(14):
        print(f"  {k:12s} {v:14.0f}  {100 * v / tot_ops:5.2f} %")
    for k in ("UBLKCP", "UTMALDG", "LDGSTS", "SYNCS"):
        if k not in dict(ops.most_common(14)):
            print(f"  {k:12s} {ops.get(k, 0):14.0f}  {100 * ops.get(k, 0) / tot_ops:5.2f} %")
ts = sum(l[0] for l in lines)
te = sum(l[1] for l in lines)
if ts:
    print("\nTop source lines by warp-stall samples (share of samples, share of warp instructions):")
    for sm, ex, f, n, src in sorted(lines, key=lambda l: -l[0])[:12]:
        print(f"  {100 * sm / ts:5.1f}%  {100 * ex / max(te, 1):5.1f}%i  {f}:{n}  {src[:100]}")
