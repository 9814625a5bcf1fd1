#!/bin/bash
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -rf -p no:cacheprovider -k "semlap" > gpurun_out/pytest_q2.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_q2.log
timeout 600 python tools/sem_sweep.py 8:0,39,41,42 --bytes 2 > gpurun_out/sweep_q2.jsonl 2> gpurun_out/sweep_q2.err
timeout 300 python tools/exp_timing.py > gpurun_out/exp_timing_kc.json 2>&1
V=39 timeout 300 python tools/exp_timing.py > gpurun_out/exp_timing_v39.json 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:semlap -s 3 -c 1 -o gpurun_out/prof_sem65k_kc python bench.py --workload sem65k --steps 1 --warmup 3 --no-e2e --no-cpu --no-verify > gpurun_out/ncu_sem65k_kc.log 2>&1
timeout 900 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err
