#!/bin/bash
# One GPU round-trip: parity tests, then short benches of every workload.
# Usage (under gpurun): bash scripts/gpu_check.sh [tag]
tag=${1:-run}
out=gpurun_out/$tag
mkdir -p $out
timeout 900 python -m pytest tests -x -q -m gpu -p no:cacheprovider > $out/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> $out/pytest_gpu.log
tail -3 $out/pytest_gpu.log
for w in C2 C3 C4; do
  timeout 300 python bench.py --workload $w --steps 20 --warmup 5 --no-e2e --no-cpu-baseline > $out/bench_$w.json 2> $out/bench_$w.err
done
timeout 600 python bench.py --steps 10 --warmup 3 ${BENCH_EXTRA} > $out/bench_C5.json 2> $out/bench_C5.err
echo "bench rc=$?"
