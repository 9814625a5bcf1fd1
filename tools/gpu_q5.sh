#!/bin/bash
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 300 python bench.py --workload sgemm --steps 5 > gpurun_out/bench_sgemm.json 2>>gpurun_out/q5.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:sgemm_tc2 -s 1 -c 1 -o gpurun_out/prof_sgemm2 python bench.py --workload sgemm --steps 1 --warmup 3 > gpurun_out/ncu_sgemm2.log 2>&1
for w in matvec fill axpy; do timeout 300 python bench.py --workload $w > gpurun_out/bench_$w.json 2>>gpurun_out/q5.err; done
timeout 300 python bench.py --workload fill --variant 1 > gpurun_out/bench_fill_v1.json 2>>gpurun_out/q5.err
timeout 300 python bench.py --workload matvec --variant 2 > gpurun_out/bench_matvec_v2.json 2>>gpurun_out/q5.err
