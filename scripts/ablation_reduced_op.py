"""Ablation: the paper's reduced-op update x - 0.5 (L + R)
 vs the reference order x - 0.5 L - 0.5 R, on B200.

Builds nothing: expects paper_1309_0392_b200/lib/libsgh_redop.so
(`python paper_1309_0392_b200/build.py --out .../libsgh_redop.so -DSGH_REDUCED_OP`).
Prints per workload the time of both libraries (bench.py, per-axis and the
default plan) and, for the reduced-op library, the normwise deviation from the
oracle (the default library is bitwise equal to it)."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
VAR = os.path.join(ROOT, "paper_1309_0392_b200", "lib", "libsgh_redop.so")


def bench(lib, w, extra):
    env = dict(os.environ)
    if lib:
        env["SGH_LIB_PATH"] = lib
    out = subprocess.run([sys.executable, "bench.py", "--workload", w, "--steps", "10", "--warmup", "3", "--no-e2e",
                          "--no-cpu-baseline", *extra], cwd=ROOT, env=env, capture_output=True, text=True).stdout
    return json.loads(out.strip().splitlines()[-1])["value"]


ERR = r'''
import numpy as np, torch, sys
sys.path.insert(0, "%s")
import oracle, sgh_inputs as si, paper_1309_0392_b200 as sgh
for lv in [(8, 8, 8), (10, 4, 4, 4, 4), (14, 13)]:
    N = si.num_points(lv); u = si.fill_uniform(N, si.SEED, 0)
    g = torch.from_numpy(u).cuda(); sgh.transform(g, lv, fuse=False); got = g.cpu().numpy()
    want = oracle.hierarchize(u.copy(), lv)
    print(lv, float(np.max(np.abs(got - want)) / np.max(np.abs(want))), int(np.count_nonzero(got != want)), N)
''' % ROOT

if __name__ == "__main__":
    for w in ("C2", "C3", "C4", "C5"):
        for extra in ([], ["--per-axis"]):
            a, b = bench(None, w, extra), bench(VAR, w, extra)
            print(f"{w} {' '.join(extra) or 'default plan':12s} reference order {a:7.1f}  reduced-op {b:7.1f} Gpoints/s")
    env = dict(os.environ, SGH_LIB_PATH=VAR)
    print("reduced-op deviation from the oracle (normwise, differing words, N):")
    print(subprocess.run([sys.executable, "-c", ERR], cwd=ROOT, env=env, capture_output=True, text=True).stdout)
