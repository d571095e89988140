#!/bin/bash
# Round-end style check (under gpurun): GPU tests, smoke(), default bench (C5 with
# e2e + cpu baseline), the reference arm, the launch list of the default bench
# command and the per-key DRAM traffic of each workload.
tag=${1:-final}; out=gpurun_out/$tag; mkdir -p $out
timeout 1200 python -m pytest tests -q -m gpu -p no:cacheprovider > $out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $out/pytest_gpu.log
tail -2 $out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $out/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 $out/smoke.log
timeout 900 python bench.py > $out/bench_default.json 2> $out/bench_default.err; echo "bench rc=$?"
python scripts/bsum.py $out/bench_default.json | cut -c1-200
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $out/bench_reference.json 2> $out/bench_reference.err; echo "reference rc=$?"
cat $out/bench_reference.json | cut -c1-300
cmd="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline"
$cmd > $out/plain_launches.json 2>&1 && timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    --clock-control none --csv --log-file $out/ncu_launches_default.csv $cmd > $out/ncu_launches.log 2>&1; echo "ncu launches rc=$?"
