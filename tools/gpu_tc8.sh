#!/bin/bash
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -rf -p no:cacheprovider -k "fma_mode" > gpurun_out/pytest_tc8.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_tc8.log
timeout 900 python tools/sem_sweep.py 5:50,52 6:50,52 7:50,52 > gpurun_out/sweep_tc8.jsonl 2> gpurun_out/sweep_tc8.err
