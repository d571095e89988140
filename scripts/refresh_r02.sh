#!/bin/bash
# Everything the committed profiles/r02 summaries come from (under gpurun).
tag=${1:-r02}; out=gpurun_out/$tag; mkdir -p $out
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
timeout 600 python scripts/sweep_curves.py both --steps 10 > $out/sweep_hier.jsonl 2> $out/sweep.err; echo "sweep rc=$?"
bash scripts/traffic_capture.sh $tag/traffic "C5 C4 C2 C3"
bash scripts/traffic_capture.sh $tag/traffic "C5 C4" --inverse
bash scripts/ncu_one.sh $tag C5 k_fpipe 0 1
