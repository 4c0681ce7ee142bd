#!/bin/bash
# One ncu --set full capture + source counters: KCONF (bench config), KREGEX
# (kernel name regex), KSKIP (launches of it to skip), KPREC (fp32 / fp64).
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
O=${OUT:-gpurun_out/ncu1}; mkdir -p $O; R=/tmp/ncu1; mkdir -p $R
timeout 900 ncu --set full --clock-control none --import-source on -k regex:${KREGEX} -s ${KSKIP:-0} -c 1 \
  -o $R/k -f python tools/prof_run.py --config ${KCONF:-c5} --precision ${KPREC:-fp32} --reps 1 > $O/ncu.log 2>&1
python tools/ncu_summary.py report $R/k.ncu-rep > $O/full.md 2>&1
ncu -i $R/k.ncu-rep --page source --csv --print-source cuda,sass > $O/src.csv 2>&1
ncu -i $R/k.ncu-rep --page source --csv --print-source sass > $O/sass.csv 2>&1
