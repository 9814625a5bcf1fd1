#!/bin/bash
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -rf -p no:cacheprovider -k "fma_mode" > gpurun_out/pytest_q12.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_q12.log
timeout 900 python tools/sem_sweep.py 10:50,51 12:50,51 14:50,51 16:50,51 > gpurun_out/sweep_q12.jsonl 2> gpurun_out/sweep_q12.err
