#!/bin/bash
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -rf -p no:cacheprovider -k "fma_mode" > gpurun_out/pytest_tc2.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_tc2.log
timeout 1500 python tools/sem_sweep.py 12:52,53 13:52,53 14:52,53 15:52,53 16:52,53,54 > gpurun_out/sweep_tc2.jsonl 2> gpurun_out/sweep_tc2.err
