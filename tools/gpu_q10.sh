#!/bin/bash
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -rf -p no:cacheprovider -k "semlap" > gpurun_out/pytest_q10.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_q10.log
timeout 1200 python tools/sem_sweep.py 4:0,50 5:0,50 6:0,50 7:0,50 8:0,50 9:0,50 10:0,50 11:0,50 12:0,50 13:0,50 14:0,50 15:0,50 16:0,50 > gpurun_out/sweep_q10.jsonl 2> gpurun_out/sweep_q10.err
timeout 300 python bench.py --variant 50 --no-e2e --no-cpu > gpurun_out/bench_fma.json 2> gpurun_out/bench_fma.err
V=50 timeout 300 python tools/exp_timing.py > gpurun_out/exp_timing_fma.json 2>&1
