#!/bin/bash
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
NCU="ncu --set full --clock-control none --import-source on"
for n in 9 10 12; do timeout 600 $NCU -k regex:semlap -s 3 -c 1 -o gpurun_out/prof_fma_n$n python tools/sem_sweep.py $n:50 --bytes 1 > gpurun_out/ncu_fma_n$n.log 2>&1; done
