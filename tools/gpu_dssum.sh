#!/bin/bash
# dssum: assembly tests, probe (E = 64, 128; default vs generic kernel),
# ncu of the default kernel.  Outputs under gpurun_out/dssum/.
cd $GRAFT_REPO_ROOT; O=gpurun_out/dssum; mkdir -p $O
timeout 600 python -m pytest tests/test_assembly.py -m gpu -q -x > $O/pytest.log 2>&1
python tools/dssum_probe.py 64 8 ${VARIANTS:-0 1} > $O/probe.jsonl 2>&1
python tools/dssum_probe.py 128 8 ${VARIANTS:-0 1} >> $O/probe.jsonl 2>&1
python tools/dssum_probe.py 32 16 ${VARIANTS:-0 1} >> $O/probe.jsonl 2>&1
python tools/dssum_probe.py 128 4 ${VARIANTS:-0 1} >> $O/probe.jsonl 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:dssum -s 5 -c 1 -o $O/prof_dssum python tools/dssum_probe.py 64 8 0 > $O/ncu.log 2>&1
python tools/ncu_summary.py $O/prof_dssum.ncu-rep dssum_${TAG:-v0} --round r02 > /dev/null 2>&1; cp profiles/r02_dssum_${TAG:-v0}.md $O/
[ -n "$KEEP_REP" ] || rm -f $O/prof_dssum.ncu-rep
