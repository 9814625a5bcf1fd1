#!/bin/bash
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -rf -p no:cacheprovider -k "fma_mode" > gpurun_out/pytest_q15.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_q15.log
timeout 1200 python tools/sem_sweep.py 9:50,51 10:50,51 11:50,51 12:50,51 13:50,51 14:50,51 15:50,51 16:50,51 > gpurun_out/sweep_q15.jsonl 2> gpurun_out/sweep_q15.err
