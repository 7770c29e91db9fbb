#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck / initcheck over the solve
# kernels (tools/sanitize_case.py). Logs go to gpurun_out/sanitize_<tool>.log;
# summaries are copied to profiles/ by hand. Run on the GPU box:
#   gpurun -- bash tools/sanitize.sh
set -u
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck synccheck racecheck initcheck; do
  size=small
  [ "$tool" = memcheck ] && size=c1
  timeout 1500 $CS --tool $tool --target-processes all --print-limit 50 --error-exitcode 99 \
      python tools/sanitize_case.py $size > gpurun_out/sanitize_$tool.log 2>&1
  echo "$tool rc=$?" | tee -a gpurun_out/sanitize_summary.txt
  grep -E "ERROR SUMMARY|RACECHECK SUMMARY|Program hit|Invalid|Race" gpurun_out/sanitize_$tool.log | sort | uniq -c | head -20 >> gpurun_out/sanitize_summary.txt
done
