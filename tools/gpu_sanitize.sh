#!/bin/bash
# compute-sanitizer over small launches of every kernel family
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck racecheck synccheck; do
  for part in sem gemm stream generic assembly; do
    timeout 900 $CS --tool $tool --error-exitcode 9 python tools/sanitize_cases.py $part > gpurun_out/sanitize_${tool}_${part}.log 2>&1
    echo "$tool $part rc=$?" >> gpurun_out/sanitize_summary.txt
  done
done
