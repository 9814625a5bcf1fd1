#!/bin/bash
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -rf -p no:cacheprovider -k "semlap" > gpurun_out/pytest_q7.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_q7.log
timeout 900 python bench.py --workload sweep > gpurun_out/bench_sweep.json 2>> gpurun_out/q7.err
timeout 1200 python tools/sem_sweep.py 9:0,9,20,21 10:0,9,20,21 11:0,9,20 12:0,9,30,31 13:0,31 14:0,30,31 15:0,30 16:0,30,31 > gpurun_out/sweep_q7.jsonl 2> gpurun_out/sweep_q7.err
