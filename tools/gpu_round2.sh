#!/bin/bash
# round-2 evidence: full GPU suite, smoke, default bench (with configs),
# reference arm, ncu launch list of the default bench, sanitizers on the
# new / changed kernels.  Outputs under gpurun_out/r2full/.
cd $GRAFT_REPO_ROOT; O=gpurun_out/r2full; mkdir -p $O
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -rf > $O/pytest_gpu.log 2>&1
timeout 600 python bench.py > $O/bench_default.json 2> $O/bench_default.err
timeout 600 python bench.py --impl reference > $O/bench_reference.json 2> $O/bench_reference.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_default.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu --no-configs > $O/bench_under_ncu.log 2>&1
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck racecheck synccheck; do
  for part in assembly sem gemm; do
    timeout 900 $CS --tool $tool --error-exitcode 9 python tools/sanitize_cases.py $part > $O/sanitize_${tool}_${part}.log 2>&1
    echo "$tool $part rc=$?" >> $O/sanitize_summary.txt
  done
done
