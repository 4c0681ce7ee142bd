cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
O=gpurun_out/tc2prof; mkdir -p $O; R=/tmp/ncu_tc2; mkdir -p $R
DSMC_PAIR_KERNEL=tc2 timeout 600 ncu --set full --clock-control none --import-source on -k regex:c32_pair_tc2 -s 2 -c 1 \
    -o $R/full -f python tools/prof_run.py --config c2 --reps 1 > $O/ncu_full.log 2>&1
python tools/ncu_summary.py report $R/full.ncu-rep > $O/full.md 2>&1
ncu -i $R/full.ncu-rep --page source --csv --print-source cuda,sass > $O/src.csv 2>&1
ncu -i $R/full.ncu-rep --page source --csv --print-source sass > $O/sass.csv 2>&1
ncu -i $R/full.ncu-rep --page raw --csv > $O/raw.csv 2>&1
