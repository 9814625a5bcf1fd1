#!/bin/bash
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for wl in sem2m sem65k; do timeout 300 python bench.py --workload $wl --no-e2e --no-cpu --no-verify > gpurun_out/probe_$wl.json 2>&1; done
nvidia-smi -q -d CLOCK,POWER,PERFORMANCE > gpurun_out/smi_q.txt 2>&1
