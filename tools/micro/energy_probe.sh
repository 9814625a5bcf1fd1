#!/bin/bash
# products per joule: each energy_probe kernel for 3 s under nvidia-smi
# power / clock sampling (10 ms).  Output: gpurun_out/energy_probe.txt
cd $GRAFT_REPO_ROOT; O=gpurun_out; mkdir -p $O
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/energy_probe tools/micro/energy_probe.cu || exit 1
: > $O/energy_probe.txt
for k in 0 1 2 3; do
  nvidia-smi --query-gpu=power.draw,clocks.sm,clocks_throttle_reasons.active --format=csv,noheader,nounits -lms 10 > /tmp/smi_$k.csv &
  P=$!
  sleep 0.5
  /tmp/energy_probe $k 3 >> $O/energy_probe.txt
  kill $P
  python3 - <<PY >> $O/energy_probe.txt
rows=[l.split(', ') for l in open('/tmp/smi_$k.csv') if l.strip()]
rows=rows[60:-20] if len(rows)>100 else rows
pw=sorted(float(r[0]) for r in rows); ck=sorted(float(r[1]) for r in rows)
print({"kernel": $k, "power_median": pw[len(pw)//2], "sm_mhz_median": ck[len(ck)//2], "reasons": sorted(set(r[2] for r in rows))})
PY
  sleep 2
done
