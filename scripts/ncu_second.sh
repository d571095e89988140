#!/bin/bash
# ncu --set full of the C5 step's other large launches (under gpurun): the first
# large STRIDED<256> launch (13 % of the step: the 7th k_strided launch of a step) and the
# W = 32 blocked FUSED launch (5 %: the 9th k_fused launch); see profiles/r02/traffic/keys_C5.json.
tag=${1:-r02j}; out=gpurun_out/$tag; mkdir -p $out
cmd="python bench.py --workload C5 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline"
$cmd > $out/plain_C5.log 2>&1 || { echo "plain bench failed"; exit 1; }
timeout 900 ncu --set full --clock-control none --import-source on -k k_strided -s 6 -c 1 \
    -o $out/C5_strided256 $cmd > $out/ncu_strided256.log 2>&1; echo "ncu strided rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k k_fused -s 8 -c 1 \
    -o $out/C5_fused32 $cmd > $out/ncu_fused32.log 2>&1; echo "ncu fused32 rc=$?"
ls -la $out
