#!/bin/bash
# ncu --set full of the high-order SEM kernels (sweep sizes)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for spec in ${SPECS:-16:52 13:52 16:0 13:0}; do
  tag=$(echo $spec | tr ':' '_')
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:semlap -s 3 -c 1 -o gpurun_out/prof_hi_$tag python tools/sem_sweep.py $spec > gpurun_out/ncu_hi_$tag.log 2>&1
done
ls gpurun_out | grep prof_hi
# summarise on the box, bring back only the summaries
for spec in ${SPECS:-16:52 13:52 16:0 13:0}; do
  tag=$(echo $spec | tr ':' '_')
  python tools/ncu_summary.py gpurun_out/prof_hi_$tag.ncu-rep sem_hi_$tag --round r01 > /dev/null 2>&1
  cp profiles/r01_sem_hi_$tag.md gpurun_out/ 2>/dev/null
  rm -f gpurun_out/prof_hi_$tag.ncu-rep
done
