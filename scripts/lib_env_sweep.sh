#!/bin/bash
# A/B (library variant, environment) pairs on one workload; variants need -DSGH_TUNING for env knobs.
# Usage (under gpurun): bash scripts/lib_env_sweep.sh tag workload "var:ENV=V var2:ENV=V ..." [bench args]
tag=$1; w=$2; pairs=$3; shift 3
out=gpurun_out/$tag; mkdir -p $out
for p in base:NONE=1 $pairs; do
  v=${p%%:*}; e=${p#*:}
  if [ "$v" = base ]; then lib=""; else lib=$PWD/paper_1309_0392_b200/lib/var_$v.so; fi
  n=${v}_${e//=/_}
  env $e SGH_LIB_PATH=$lib timeout 300 python bench.py --workload $w --steps 10 --warmup 3 --no-e2e --no-cpu-baseline "$@" \
    > $out/bench_${w}_$n.json 2> $out/bench_${w}_$n.err
  echo "$v $e rc=$? $(python -c "import json;d=json.loads(open('$out/bench_${w}_$n.json').read().strip().splitlines()[-1]);print(round(d['value'],1), d['roofline']['kernel'], round(d['roofline']['frac'],3), round(d['model']['passes_per_point'],3))" 2>/dev/null)"
done
