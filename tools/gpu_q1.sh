#!/bin/bash
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -rf -p no:cacheprovider -k "fill or matvec" > gpurun_out/pytest_q1.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_q1.log
for v in 0 1; do timeout 300 python bench.py --workload fill --variant $v > gpurun_out/bench_fill_v$v.json 2>>gpurun_out/q1.err; done
timeout 300 python bench.py --workload matvec > gpurun_out/bench_matvec.json 2>>gpurun_out/q1.err
timeout 300 ncu --set full --clock-control none --import-source on -k regex:matvec_split -s 3 -c 1 -o gpurun_out/prof_matvec_split python bench.py --workload matvec --variant 2 --steps 1 --warmup 3 > gpurun_out/ncu_mvs.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:fill_bulk -s 3 -c 1 -o gpurun_out/prof_fill_bulk python bench.py --workload fill --steps 1 --warmup 3 > gpurun_out/ncu_fillb.log 2>&1
