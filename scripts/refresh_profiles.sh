#!/bin/bash
# Everything the committed profiles/ summaries come from (under gpurun):
# final_check.sh (tests, smoke, default bench, reference arm, ncu launch list)
# plus every workload's bench line, hierarchization and dehierarchization.
tag=${1:-refresh}; out=gpurun_out/$tag; mkdir -p $out
bash scripts/final_check.sh $tag
for w in C2 C3 C4 C5 S1 S10; do
  timeout 300 python bench.py --workload $w --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > $out/bench_$w.json 2> $out/bench_$w.err
  echo "$w $(python scripts/bsum.py $out/bench_$w.json | cut -c1-110)"
done
for w in C2 C3 C4 C5; do
  timeout 300 python bench.py --workload $w --inverse --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > $out/bench_${w}_dehier.json 2> $out/bench_${w}_dehier.err
  echo "$w inv $(python scripts/bsum.py $out/bench_${w}_dehier.json | cut -c1-110)"
done
timeout 300 python bench.py --workload C5cycle --steps 3 --warmup 3 > $out/bench_C5cycle.json 2> $out/bench_C5cycle.err
echo "C5cycle $(python scripts/bsum.py $out/bench_C5cycle.json | cut -c1-110)"
