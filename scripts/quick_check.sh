#!/bin/bash
# Fast GPU iteration: a parity subset, then C5 and C4 benches.
# Usage (under gpurun): bash scripts/quick_check.sh tag [pytest -k expr]
tag=${1:-quick}
kexpr=${2:-"shape_sweep or subnormal or blocked or two_blocked or batched or c5"}
out=gpurun_out/$tag
mkdir -p $out
timeout 400 python -m pytest tests -x -q -m gpu -p no:cacheprovider -k "$kexpr" > $out/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> $out/pytest_gpu.log
tail -3 $out/pytest_gpu.log
for w in C5 C4; do
  timeout 300 python bench.py --workload $w --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > $out/bench_$w.json 2> $out/bench_$w.err
  echo "bench $w rc=$?"
done
