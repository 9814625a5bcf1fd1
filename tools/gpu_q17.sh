#!/bin/bash
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -rf -p no:cacheprovider -k "semlap_gen_variants or fma_mode" > gpurun_out/pytest_q17.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_q17.log
timeout 1200 python tools/sem_sweep.py 7:0,60,50,61 9:0,60,50,61 10:0,60,50,61 11:0,60,50,61 12:0,60,50,61 > gpurun_out/sweep_q17.jsonl 2> gpurun_out/sweep_q17.err
