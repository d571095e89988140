#!/bin/bash
# A/B the tuning variants built by build_variants.sh on one workload.
# Usage (under gpurun): bash scripts/variant_sweep.sh tag workload "name1 name2 ..." [extra bench args]
tag=$1; w=$2; names=$3; shift 3
out=gpurun_out/$tag
mkdir -p $out
for n in base $names; do
  if [ "$n" = base ]; then lib=""; else lib=$PWD/paper_1309_0392_b200/lib/var_$n.so; fi
  SGH_LIB_PATH=$lib timeout 300 python bench.py --workload $w --steps 10 --warmup 3 --no-e2e --no-cpu-baseline "$@" \
    > $out/bench_${w}_$n.json 2> $out/bench_${w}_$n.err
  echo "$n rc=$? $(python -c "import json;d=json.loads(open('$out/bench_${w}_$n.json').read().strip().splitlines()[-1]);print(round(d['value'],1), d['roofline']['kernel'], round(d['roofline']['frac'],3))" 2>/dev/null)"
done
