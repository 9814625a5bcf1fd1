#!/bin/bash
# ncu --set full captures of every workload's dominant kernel (source-level)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
NCU="ncu --set full --clock-control none --import-source on"
timeout 600 $NCU -k regex:semlap -s 3 -c 1 -o gpurun_out/prof_sem65k python bench.py --workload sem65k --steps 1 --warmup 3 --no-e2e --no-cpu --no-verify > gpurun_out/ncu_sem65k.log 2>&1
timeout 300 $NCU -k regex:matvec -s 3 -c 1 -o gpurun_out/prof_matvec python bench.py --workload matvec --steps 1 --warmup 3 > gpurun_out/ncu_matvec.log 2>&1
timeout 300 $NCU -k regex:fill_vec -s 3 -c 1 -o gpurun_out/prof_fill python bench.py --workload fill --steps 1 --warmup 3 > gpurun_out/ncu_fill.log 2>&1
timeout 300 $NCU -k regex:axpy_vec -s 3 -c 1 -o gpurun_out/prof_axpy python bench.py --workload axpy --steps 1 --warmup 3 > gpurun_out/ncu_axpy.log 2>&1
timeout 600 $NCU -k regex:semlap -s 3 -c 1 -o gpurun_out/prof_sem_n12 python tools/sem_sweep.py 12:0 --bytes 1 > gpurun_out/ncu_n12.log 2>&1
timeout 600 $NCU -k regex:semlap -s 3 -c 1 -o gpurun_out/prof_sem_n16 python tools/sem_sweep.py 16:0 --bytes 1 > gpurun_out/ncu_n16.log 2>&1
timeout 600 $NCU -k regex:gemm -s 1 -c 1 -o gpurun_out/prof_sgemm python bench.py --workload sgemm --steps 1 --warmup 3 > gpurun_out/ncu_sgemm.log 2>&1
ls -la gpurun_out
