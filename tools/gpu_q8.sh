#!/bin/bash
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
NCU="ncu --set full --clock-control none --import-source on"
timeout 600 $NCU -k regex:semlap -s 3 -c 1 -o gpurun_out/prof_sem_n16b python tools/sem_sweep.py 16:0 --bytes 1 > gpurun_out/ncu_n16b.log 2>&1
timeout 600 $NCU -k regex:semlap -s 3 -c 1 -o gpurun_out/prof_sem_n12b python tools/sem_sweep.py 12:0 --bytes 1 > gpurun_out/ncu_n12b.log 2>&1
timeout 600 $NCU -k regex:semlap -s 3 -c 1 -o gpurun_out/prof_sem_n10b python tools/sem_sweep.py 10:0 --bytes 1 > gpurun_out/ncu_n10b.log 2>&1
