#!/bin/bash
# dgemm DMMA kernel variants at 8192^3 (bench line each, no CPU leg):
# 0 default (BK 16 x 4 stages), 3 BK 32 x 3, 4 fragments double-buffered,
# 5 both.  Outputs gpurun_out/dgemm/.
cd $GRAFT_REPO_ROOT; O=gpurun_out/dgemm; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "dgemm" > $O/pytest.log 2>&1
for v in ${VARIANTS:-0 3 4 5}; do
  timeout 300 python bench.py --workload dgemm --variant $v --no-cpu --steps 10 --warmup 3 2>/dev/null | tail -1 > $O/v$v.json
done
