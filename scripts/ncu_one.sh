#!/bin/bash
# ncu --set full of ONE launch of a kernel in a bench run (under gpurun).
# Usage: bash scripts/ncu_one.sh tag workload regex skip [count]
tag=$1; w=$2; rx=$3; skip=${4:-0}; cnt=${5:-1}
out=gpurun_out/$tag; mkdir -p $out
cmd="python bench.py --workload $w --steps 3 --warmup 3 --no-e2e --no-cpu-baseline"
$cmd > $out/plain_$w.log 2>&1 &&
timeout 900 ncu --set full --clock-control none --import-source on -k regex:$rx -s $skip -c $cnt \
    -o $out/${w}_$rx $cmd > $out/ncu_${w}.log 2>&1
echo "ncu rc=$?"
