#!/bin/bash
# SEM order sweep: parity for the new kernels, then timing per variant
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -rf -p no:cacheprovider -k "semlap" > gpurun_out/pytest_sem.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_sem.log
timeout 1200 python tools/sem_sweep.py 4:0,20,21,22,9 5:0,20,21,22,9 6:0,20,21,22,9 7:0,20,21,22,9 8:0,5,20,21,22,9 9:0,20,21,9 10:0,20,21,9 11:0,20,9 12:0,30,31 13:0,31 14:0,30,31 15:0,30 16:0,30,31 > gpurun_out/sem_sweep.jsonl 2> gpurun_out/sem_sweep.err
