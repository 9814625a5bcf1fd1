#!/bin/bash
# round-2 ncu --set full captures of the changed / headline kernels,
# summarised on the box into gpurun_out/prof_r02/*.md
cd $GRAFT_REPO_ROOT; O=gpurun_out/prof_r02; mkdir -p $O
NCU="ncu --set full --clock-control none --import-source on"
run() {  # key regex cmd...
  local key=$1 re=$2; shift 2
  timeout 900 $NCU -k regex:$re -s ${SKIP:-3} -c 1 -o $O/$key "$@" > $O/ncu_$key.log 2>&1
  python tools/ncu_summary.py $O/$key.ncu-rep $key --round r02 > /dev/null 2>&1
  cp profiles/r02_$key.md $O/ 2>/dev/null
  rm -f $O/$key.ncu-rep
}
run semlap_n8 semlap_tc2 python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --no-verify --no-configs
run semlap_n8_bitwise semlap_kc python bench.py --variant 0 --steps 1 --warmup 3 --no-e2e --no-cpu --no-verify --no-configs
SKIP=2 run dgemm dgemm_ws python bench.py --workload dgemm --no-cpu --steps 1 --warmup 2
run matvec matvec_split python bench.py --workload matvec --no-cpu --steps 1 --warmup 3
run sem_n15_dmma semlap_tc2 python tools/sem_sweep.py 15:52
