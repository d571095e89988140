#!/bin/bash
# compute-sanitizer (one tool per gpurun call) over scripts/sanitize_cases.py.
# Usage (under gpurun): bash scripts/sanitize.sh <memcheck|racecheck|synccheck|initcheck> <outdir>
tool=${1:-memcheck}
out=${2:-gpurun_out/sanitize}
mkdir -p $out
python scripts/sanitize_cases.py > $out/plain_$tool.log 2>&1 && \
timeout 1500 compute-sanitizer --tool $tool --error-exitcode 99 --print-limit 20 \
  python scripts/sanitize_cases.py > $out/$tool.log 2>&1
echo "sanitizer $tool rc=$?" >> $out/$tool.log
tail -4 $out/$tool.log
