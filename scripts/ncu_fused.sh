#!/bin/bash
# ncu --set full capture of the FUSED kernels of single-grid workloads (under gpurun).
# Usage: bash scripts/ncu_fused.sh tag [regex] [workloads...]
tag=${1:-prof}; rx=${2:-k_fused}; shift 2
out=gpurun_out/$tag; mkdir -p $out
for w in ${@:-C2 C3}; do
  cmd="python bench.py --workload $w --steps 3 --warmup 3 --no-e2e --no-cpu-baseline"
  $cmd > $out/plain_$w.log 2>&1 &&
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$rx -s 2 -c 4 \
      -o $out/$w $cmd > $out/ncu_$w.log 2>&1
  echo "$w rc=$?"
done
