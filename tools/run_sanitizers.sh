#!/bin/bash
# SURVEY.md §4b tier T5: compute-sanitizer memcheck / racecheck / synccheck / initcheck over the
# kernel-coverage workload of tools/sanitize_workload.py (C1, C2, modes, slab group, AOS, 3-D).
# Logs: gpurun_out/sanitize_<tool>.log; summary lines: gpurun_out/sanitize_summary.txt.
set -u
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
: > gpurun_out/sanitize_summary.txt
for tool in memcheck racecheck synccheck initcheck; do
  extra=""
  [ "$tool" = racecheck ] && extra="--racecheck-report all"
  [ "$tool" = memcheck ] && extra="--leak-check full"
  timeout ${SANI_TIMEOUT:-1500} $CS --tool $tool $extra --print-limit 200 --error-exitcode 9 \
      --target-processes all python tools/sanitize_workload.py "$@" > gpurun_out/sanitize_$tool.log 2>&1
  rc=$?
  echo "$tool rc=$rc $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|LEAK SUMMARY' gpurun_out/sanitize_$tool.log | tr '\n' ' ')" \
      >> gpurun_out/sanitize_summary.txt
done
cat gpurun_out/sanitize_summary.txt
