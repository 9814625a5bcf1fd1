#!/bin/bash
# round-1 run 2: parity tests, benches, ncu captures
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -rf -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err
for w in fill axpy matvec sweep; do timeout 600 python bench.py --workload $w > gpurun_out/bench_$w.json 2>> gpurun_out/bench_other.err; done
timeout 600 python bench.py --workload sgemm --gemm-n 4096 --steps 3 > gpurun_out/bench_sgemm_exact4096.json 2>> gpurun_out/bench_other.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:semlap_kernel -s 3 -c 1 -o gpurun_out/prof_sem65k python bench.py --workload sem65k --steps 1 --warmup 3 --no-e2e --no-cpu --no-verify > gpurun_out/ncu_sem.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_default.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu --no-verify > gpurun_out/ncu_launches.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:matvec_tma -s 3 -c 1 -o gpurun_out/prof_matvec python bench.py --workload matvec --steps 1 --warmup 3 > gpurun_out/ncu_matvec.log 2>&1
ls -la gpurun_out
