#!/bin/bash
# sanitizers over the gemm and streaming cases (rings that wrap), matvec line
cd $GRAFT_REPO_ROOT; O=gpurun_out/san2; mkdir -p $O
CS=/usr/local/cuda/bin/compute-sanitizer
: > $O/sanitize_summary.txt
for part in stream gemm; do
  for tool in racecheck memcheck synccheck; do
    timeout 900 $CS --tool $tool --error-exitcode 9 python tools/sanitize_cases.py $part > $O/sanitize_${tool}_$part.log 2>&1
    echo "$tool $part rc=$?" >> $O/sanitize_summary.txt
  done
done
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "matvec" > $O/pytest.log 2>&1
timeout 300 python bench.py --workload matvec --no-cpu --steps 10 --warmup 3 2>/dev/null | tail -1 > $O/matvec.json
