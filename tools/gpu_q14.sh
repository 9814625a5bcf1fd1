#!/bin/bash
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -rf -p no:cacheprovider -k "semlap" > gpurun_out/pytest_q14.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_q14.log
timeout 600 python bench.py --no-e2e --no-cpu > gpurun_out/bench_q14.json 2> gpurun_out/bench_q14.err
V=0 timeout 300 python tools/exp_timing.py > gpurun_out/exp_timing_bw2.json 2>&1
