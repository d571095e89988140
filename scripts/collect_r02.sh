#!/bin/bash
# Copy what one `gpurun -- bash scripts/refresh_r02.sh <tag>` call brought back
# (gpurun_out/<tag>) into the tracked profiles/r02 and rebuild the derived
# files: profiles/ncu_traffic.json (per kernel key, workload and direction) and
# the launch-list summary.  Run here (no GPU needed).
# Usage: bash scripts/collect_r02.sh <tag>
set -e
tag=${1:?tag}; src=gpurun_out/$tag; dst=profiles/r02
mkdir -p $dst/traffic
for f in bench_default bench_reference bench_C2 bench_C3 bench_C4 bench_C5 bench_S1 bench_S10 \
         bench_C2_dehier bench_C3_dehier bench_C4_dehier bench_C5_dehier bench_C5cycle; do
  [ -s $src/$f.json ] && cp $src/$f.json $dst/$f.json
done
cp $src/pytest_gpu.log $src/smoke.log $dst/
cp $src/ncu_launches_default.csv $dst/
[ -s $src/sweep_hier.jsonl ] && cp $src/sweep_hier.jsonl $dst/sweep_S1_S10.jsonl
for w in C2 C3 C4 C5 C4_dehier C5_dehier; do
  [ -s $src/traffic/launches_$w.csv ] || continue
  cp $src/traffic/launches_$w.csv $src/traffic/keys_$w.json $dst/traffic/
  python scripts/ncu_traffic.py $dst/traffic/launches_$w.csv $dst/traffic/keys_$w.json profiles/ncu_traffic.json > /dev/null
done
python scripts/ncu_launches.py $dst/ncu_launches_default.csv > $dst/ncu_launches_default_summary.txt
for f in $dst/bench_*.json; do python scripts/bsum.py $f | cut -c1-150; done
