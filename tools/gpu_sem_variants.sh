#!/bin/bash
# SEM kernel variant sweep: parity tests + bench per variant (2M and 65K)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -rf -p no:cacheprovider -k "semlap" > gpurun_out/pytest_sem.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_sem.log
for v in ${VARIANTS:-0 5 6 7 10 11 12 13 14 15}; do
  for wl in sem2m sem65k; do
    echo "variant $v $wl: $(timeout 300 python bench.py --workload $wl --variant $v --no-e2e --no-cpu 2>&1 | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["value"],2), "GDOF/s", round(d["roofline"]["frac"],4), d["verify"], d["clocks"]["sm_mhz"], d["clocks"]["reasons"])' 2>&1)" >> gpurun_out/sem_variants.log
  done
done
