#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck over tools/sanitize_cases.py
# (run on a B200 via gpurun); logs -> gpurun_out/sanitize/
set -u
OUT=gpurun_out/sanitize
mkdir -p $OUT
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck synccheck racecheck; do
  timeout 1500 $CS --tool $tool --error-exitcode 9 --print-limit 50 --target-processes all \
      python tools/sanitize_cases.py > $OUT/$tool.log 2>&1
  echo "$tool rc=$?" | tee -a $OUT/summary.txt
  grep -E "ERROR SUMMARY|sanitize case" $OUT/$tool.log | tee -a $OUT/summary.txt
done
