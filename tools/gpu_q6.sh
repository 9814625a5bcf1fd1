#!/bin/bash
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -rf -p no:cacheprovider -k "sgemm or matvec" > gpurun_out/pytest_q6.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_q6.log
timeout 300 python bench.py --workload sgemm --steps 5 > gpurun_out/bench_sgemm.json 2>>gpurun_out/q6.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:sgemm_tc2 -s 1 -c 1 -o gpurun_out/prof_sgemm3 python bench.py --workload sgemm --steps 1 --warmup 3 > gpurun_out/ncu_sgemm3.log 2>&1
timeout 300 python bench.py --workload matvec > gpurun_out/bench_matvec.json 2>>gpurun_out/q6.err
