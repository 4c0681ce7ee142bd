#!/bin/bash
# ncu captures of the C2 step: launch list + full sets of the pair and sample kernels.
# The launch list runs eagerly (DSMC_NO_GRAPH=1): ncu does not survive replaying
# a CUDA graph whose edges are programmatic (PDL).
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
CFG=${1:-c2}
DSMC_NO_GRAPH=1 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv \
  --log-file gpurun_out/launches_$CFG.csv python tools/prof_run.py --config $CFG --reps 1 > gpurun_out/ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:c32_pair -s 3 -c 1 \
  -o gpurun_out/pair_$CFG -f python tools/prof_run.py --config $CFG --reps 1 > gpurun_out/ncu_full.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:c32_sample -s 3 -c 1 \
  -o gpurun_out/sample_$CFG -f python tools/prof_run.py --config $CFG --reps 1 > gpurun_out/ncu_full2.log 2>&1
echo done
