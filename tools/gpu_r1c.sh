#!/bin/bash
# round-1 (re-entry): parity tests, default bench, variant sweep, ncu
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
(nvidia-smi; free -g; nproc; lscpu | grep -E "Model name|Socket|Core|Thread") > gpurun_out/box.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -q -rf -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err
timeout 300 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_reference.json 2> gpurun_out/bench_reference.err
for v in 0 5 9 12 14; do
  for wl in sem2m; do
    echo "variant $v $wl: $(timeout 300 python bench.py --workload $wl --variant $v --no-e2e --no-cpu --no-verify 2>&1 | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["value"],2), "GDOF/s", round(d["roofline"]["frac"],4), round(d["roofline"]["stream_probe_gbs"],1), d["clocks"]["sm_mhz"], d["clocks"]["reasons"])' 2>&1)" >> gpurun_out/sem_variants.log
  done
done
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_default.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu --no-verify > gpurun_out/ncu_launches.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:semlap -s 3 -c 1 -o gpurun_out/prof_sem2m python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --no-verify > gpurun_out/ncu_sem.log 2>&1
for w in fill axpy matvec sweep; do timeout 600 python bench.py --workload $w > gpurun_out/bench_$w.json 2>> gpurun_out/bench_other.err; done
timeout 300 python bench.py --workload sgemm --steps 5 > gpurun_out/bench_sgemm.json 2>> gpurun_out/bench_other.err
ls -la gpurun_out
