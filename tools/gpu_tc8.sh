#!/bin/bash
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for v in 53 52 50; do V=$v timeout 300 python tools/exp_timing.py > gpurun_out/exp_timing_tc8_$v.json 2>&1; done
for v in 53 52 50; do timeout 600 python bench.py --variant $v --no-e2e --no-cpu --steps 30 > gpurun_out/bench_tc8_$v.json 2> gpurun_out/bench_tc8.err; done
