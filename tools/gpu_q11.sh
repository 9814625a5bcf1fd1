#!/bin/bash
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err
timeout 900 python bench.py --workload sweep > gpurun_out/bench_sweep.json 2>> gpurun_out/bench_other.err
timeout 600 python bench.py --workload sem65k --no-e2e > gpurun_out/bench_sem65k.json 2>> gpurun_out/bench_other.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:semlap -s 3 -c 1 -o gpurun_out/prof_sem2m_fma python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --no-verify > gpurun_out/ncu_sem2m_fma.log 2>&1
