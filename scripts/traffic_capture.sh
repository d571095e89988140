#!/bin/bash
# DRAM traffic per kernel key (bench roofline "traffic"): one plain bench run that
# dumps the launch keys of a timed step, then an ncu launch list of the same step.
# Usage (under gpurun): bash scripts/traffic_capture.sh tag "C5 C2 C3 C4" [--inverse]
tag=$1; out=gpurun_out/$tag; mkdir -p $out
extra=$3; sfx=${extra:+_dehier}
for w in ${2:-C5}; do
  cmd="python bench.py --workload $w --steps 1 --warmup 3 --no-e2e --no-cpu-baseline $extra"
  $cmd --dump-launch-keys $out/keys_$w$sfx.json > $out/plain_$w$sfx.json 2> $out/plain_$w$sfx.err || { echo "$w plain failed"; continue; }
  L=$(python -c "import json;print(json.load(open('$out/keys_$w$sfx.json'))['launches_per_step'])")
  timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
      -k regex:"k_(fused|flat|strided|reg|fpipe)" -s $((3 * L)) -c $L --csv --log-file $out/launches_$w$sfx.csv \
      $cmd > $out/ncu_$w$sfx.log 2>&1
  echo "$w ncu rc=$? launches/step=$L"
done
