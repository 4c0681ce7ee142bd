#!/bin/bash
# Source-level counters of the FP64 sampler (c64_sample, C2 FP64), third launch.
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
O=gpurun_out/src64s; mkdir -p $O; R=/tmp/ncu_src; mkdir -p $R
timeout 900 ncu --set full --clock-control none --import-source on -k regex:c64_sample -s 2 -c 1 \
  -o $R/src -f python tools/prof_run.py --config c2 --precision fp64 --reps 1 > $O/ncu.log 2>&1
ncu -i $R/src.ncu-rep --page source --csv --print-source cuda,sass > $O/src.csv 2>&1
ncu -i $R/src.ncu-rep --page source --csv --print-source sass > $O/sass.csv 2>&1
ls -la $O
