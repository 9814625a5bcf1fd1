#!/bin/bash
# dgemm: tests, bench line, racecheck / memcheck / synccheck of the gemm cases
cd $GRAFT_REPO_ROOT; O=gpurun_out/dgemm; mkdir -p $O
VARIANTS="${VARIANTS:-0}" bash tools/gpu_dgemm.sh
CS=/usr/local/cuda/bin/compute-sanitizer
: > $O/sanitize_summary.txt
for tool in racecheck memcheck synccheck; do
  timeout 900 $CS --tool $tool --error-exitcode 9 python tools/sanitize_cases.py gemm > $O/sanitize_$tool.log 2>&1
  echo "$tool gemm rc=$?" >> $O/sanitize_summary.txt
done
