#!/bin/bash
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -rf -s -p no:cacheprovider -k "sgemm" > gpurun_out/pytest_gemm.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gemm.log
for v in 2 1; do timeout 300 python bench.py --workload sgemm --variant $v --steps 5 > gpurun_out/bench_sgemm_v$v.json 2>&1; done
