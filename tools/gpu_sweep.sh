#!/bin/bash
# SEM order sweep: parity for the new kernels, then timing per variant
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -rf -p no:cacheprovider -k "semlap" > gpurun_out/pytest_sem.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_sem.log
timeout 1200 python tools/sem_sweep.py ${SWEEP:-4:0,23 5:0,20,21 6:0,20,21,22 7:0,20,21,22,23 8:0,22 9:0,20,21 10:0,20,21 11:0,20 12:0,20} > gpurun_out/sem_sweep.jsonl 2> gpurun_out/sem_sweep.err
