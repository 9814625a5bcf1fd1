#!/bin/bash
# generic engine: parity tests, bench rows, one ncu capture of the DGEMM
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_generic.py -m gpu -q -rf -p no:cacheprovider > gpurun_out/pytest_generic.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_generic.log
timeout 600 python bench.py --workload generic > gpurun_out/bench_generic.json 2> gpurun_out/bench_generic.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:lfb_gen_dgemm -c 1 -o gpurun_out/prof_gen_dgemm python bench.py --workload generic --steps 1 --warmup 3 > gpurun_out/ncu_gen.log 2>&1
ls gpurun_out | head -5
