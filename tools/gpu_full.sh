#!/bin/bash
# full round checkpoint: parity suite, smoke, every bench line, ncu evidence
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
(nvidia-smi --query-gpu=name,power.limit,clocks.max.sm,clocks.max.mem --format=csv; nproc; lscpu | grep -E "Model name") > gpurun_out/box.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -rf -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_reference.json 2> gpurun_out/bench_reference.err
for w in sem65k fill axpy matvec sgemm dgemm generic sweep; do timeout 900 python bench.py --workload $w > gpurun_out/bench_$w.json 2>> gpurun_out/bench_other.err; done
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_default.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu --no-verify > gpurun_out/ncu_launches.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:semlap -s 3 -c 1 -o gpurun_out/prof_sem2m_kc python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --no-verify > gpurun_out/ncu_sem2m.log 2>&1
ls -la gpurun_out
