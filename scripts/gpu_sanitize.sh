#!/bin/bash
# compute-sanitizer over every kernel path (scripts/sanitize_cases.py), one tool at a time.
mkdir -p gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
python scripts/sanitize_cases.py > gpurun_out/sanitize_plain.log 2>&1; echo "plain rc=$?" >> gpurun_out/sanitize_plain.log
for tool in memcheck synccheck initcheck racecheck; do
  extra=""
  [ "$tool" = "racecheck" ] && extra="--small"
  [ "$tool" = "memcheck" ] && opts="--leak-check no" || opts=""
  timeout 900 $CS --tool $tool $opts --target-processes all --print-limit 50 \
     python scripts/sanitize_cases.py $extra > gpurun_out/sanitize_$tool.log 2>&1
  echo "rc=$?" >> gpurun_out/sanitize_$tool.log
done
tail -n 5 gpurun_out/sanitize_*.log
