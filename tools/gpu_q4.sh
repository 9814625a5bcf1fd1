#!/bin/bash
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -rf -p no:cacheprovider -k "sgemm_tensor and 3200 and -2" > gpurun_out/pytest_q4.log 2>&1
