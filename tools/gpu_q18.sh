#!/bin/bash
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_generic.py -m gpu -q -rf -p no:cacheprovider -k "gemm" > gpurun_out/pytest_q18.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_q18.log
timeout 600 python bench.py --workload dgemm --steps 5 > gpurun_out/bench_dgemm.json 2> gpurun_out/bench_dgemm.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:dgemm_dmma -s 1 -c 1 -o gpurun_out/prof_dgemm python bench.py --workload dgemm --gemm-n 4096 --steps 1 --warmup 3 > gpurun_out/ncu_dgemm.log 2>&1
