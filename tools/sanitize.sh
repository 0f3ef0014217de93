#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck over every kernel family
# at small sizes (tools/sanitize_case.py).  Logs -> gpurun_out/sanitize_*.log
set -u
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck racecheck synccheck; do
  extra=""
  [ "$tool" = racecheck ] && extra="--racecheck-report analysis"
  timeout 1500 $CS --tool $tool $extra --error-exitcode 9 --print-limit 50 \
    python tools/sanitize_case.py ${SAN_ARGS:-} > gpurun_out/sanitize_$tool.log 2>&1
  echo "$tool rc=$?" | tee -a gpurun_out/sanitize_summary.txt
  tail -3 gpurun_out/sanitize_$tool.log | tee -a gpurun_out/sanitize_summary.txt
done
