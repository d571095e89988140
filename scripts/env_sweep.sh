#!/bin/bash
# A/B environment settings on one workload.
# Usage (under gpurun): bash scripts/env_sweep.sh tag workload "VAR=a VAR=b ..." [extra bench args]
tag=$1; w=$2; settings=$3; shift 3
out=gpurun_out/$tag
mkdir -p $out
for e in NONE=1 $settings; do
  n=${e//=/_}
  env $e timeout 300 python bench.py --workload $w --steps 10 --warmup 3 --no-e2e --no-cpu-baseline "$@" \
    > $out/bench_${w}_$n.json 2> $out/bench_${w}_$n.err
  echo "$e rc=$? $(python -c "import json;d=json.loads(open('$out/bench_${w}_$n.json').read().strip().splitlines()[-1]);print(round(d['value'],1), d['roofline']['kernel'], round(d['roofline']['frac'],3))" 2>/dev/null)"
done
