#!/bin/bash
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -rf -p no:cacheprovider -k "sgemm" > gpurun_out/pytest_q9.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_q9.log
for v in 0 4; do timeout 300 python bench.py --workload sgemm --variant $v --steps 5 > gpurun_out/bench_sgemm_v$v.json 2>>gpurun_out/q9.err; done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:sgemm_tc2 -s 1 -c 1 -o gpurun_out/prof_sgemm4 python bench.py --workload sgemm --steps 1 --warmup 3 > gpurun_out/ncu_sgemm4.log 2>&1
