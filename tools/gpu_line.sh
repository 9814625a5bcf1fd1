#!/bin/bash
# line-owner SEM kernel (semlap_line.cu): parity, timing against the
# defaults, ncu of n = 16.  Outputs under gpurun_out/line/.
cd $GRAFT_REPO_ROOT; O=gpurun_out/line; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "line_kernel or (fma_mode and 71)" > $O/pytest.log 2>&1
timeout 900 python tools/sem_sweep.py ${SWEEP:-9:0,50,70,71,72 10:0,50,70,71,72 11:0,50,70,71,72 12:0,50,70,71,72 13:0,50,70,71,72 14:0,50,70,71,72 15:0,50,70,71,72 16:0,50,70,71,72} > $O/sweep.jsonl 2> $O/sweep.err
for spec in ${SPECS:-16:70 16:0}; do
  tag=$(echo $spec | tr ':' '_')
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:semlap -s 3 -c 1 -o $O/prof_$tag python tools/sem_sweep.py $spec > $O/ncu_$tag.log 2>&1
  python tools/ncu_summary.py $O/prof_$tag.ncu-rep sem_hi_$tag --round r02 > /dev/null 2>&1
  cp profiles/r02_sem_hi_$tag.md $O/ 2>/dev/null
  [ -n "$KEEP_REP" ] || rm -f $O/prof_$tag.ncu-rep
done
