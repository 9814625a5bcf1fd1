#!/bin/bash
# round-1 (session 3): re-establish state: parity, default bench, sweep, timing experiment
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
(nvidia-smi; nproc; lscpu | grep -E "Model name|Socket|Core|Thread") > gpurun_out/box.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -q -rf -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err
timeout 600 python bench.py --workload sweep > gpurun_out/bench_sweep.json 2>> gpurun_out/bench_other.err
timeout 300 python tools/exp_timing.py > gpurun_out/exp_timing.json 2>&1
for w in fill axpy matvec; do timeout 600 python bench.py --workload $w > gpurun_out/bench_$w.json 2>> gpurun_out/bench_other.err; done
ls -la gpurun_out
