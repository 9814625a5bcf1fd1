#!/bin/bash
# DMMA SEM kernel: DFMA-mode parity + per-order timing (sweep sizes) + the default line
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -rf -p no:cacheprovider -k "fma_mode" > gpurun_out/pytest_tc2.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_tc2.log
timeout 900 python tools/sem_sweep.py ${SPECS:-8:52 12:52 13:52 14:52 15:52 16:52} > gpurun_out/sweep_tc2.jsonl 2> gpurun_out/sweep_tc2.err
timeout 600 python bench.py --no-e2e --no-cpu > gpurun_out/bench_tc2q.json 2> gpurun_out/bench_tc2q.err
