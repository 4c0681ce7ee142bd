#!/bin/bash
# Launch list (per-kernel device time) of the C2 step with the tc2 pass 1.
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
O=${OUT:-gpurun_out/tc2launch}; mkdir -p $O
DSMC_PAIR_KERNEL=${DSMC_PAIR_KERNEL:-tc2} DSMC_NO_GRAPH=1 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv \
  --log-file $O/launches_c2.csv python tools/prof_run.py --config ${KCONF:-c2} --reps 1 > $O/ncu_launch.log 2>&1
python tools/ncu_summary.py launches $O/launches_c2.csv > $O/launches_c2.md 2>&1
