#!/bin/bash
# compute-sanitizer over the streaming kernels (fill, matvec split-j and TMA)
cd $GRAFT_REPO_ROOT; O=gpurun_out/san_stream; mkdir -p $O
CS=/usr/local/cuda/bin/compute-sanitizer
: > $O/sanitize_summary.txt
for tool in racecheck memcheck synccheck; do
  timeout 900 $CS --tool $tool --error-exitcode 9 python tools/sanitize_cases.py stream > $O/sanitize_$tool.log 2>&1
  echo "$tool stream rc=$?" >> $O/sanitize_summary.txt
done
