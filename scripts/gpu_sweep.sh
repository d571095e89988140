#!/bin/bash
# Parity tests, then bench lines of workloads under environment variants (under gpurun).
# Usage: bash scripts/gpu_sweep.sh tag "ENV=.. ENV2=.." "..." ; workloads from $WL (default "C2 C3 C5")
tag=$1; shift
out=gpurun_out/$tag; mkdir -p $out
timeout 900 python -m pytest tests -x -q -m gpu -p no:cacheprovider > $out/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> $out/pytest_gpu.log; tail -2 $out/pytest_gpu.log
i=0
for envs in "" "$@"; do
  for w in ${WL:-C2 C3 C5}; do
    steps=20; [ $w = C5 ] && steps=10
    env $envs timeout 300 python bench.py --workload $w --steps $steps --warmup 3 --no-e2e --no-cpu-baseline \
        > $out/b${i}_$w.json 2> $out/b${i}_$w.err
    echo "[$envs] $w: $(python scripts/bsum.py $out/b${i}_$w.json | cut -c1-200)"
  done
  i=$((i+1))
done
