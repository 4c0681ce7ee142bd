cd $GRAFT_REPO_ROOT; O=gpurun_out/wprof; mkdir -p $O
DSMC_NO_GRAPH=1 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file $O/launches_c6.csv python tools/prof_run.py --config c6 --reps 1 > $O/l.log 2>&1
python tools/ncu_summary.py launches $O/launches_c6.csv > $O/launches_c6.md 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:pairw_tc2 -s 3 -c 1 -o /tmp/k -f python tools/prof_run.py --config c6 --reps 1 > $O/n.log 2>&1
python tools/ncu_summary.py report /tmp/k.ncu-rep > $O/full_pairw_tc2.md 2>&1
ncu -i /tmp/k.ncu-rep --page source --csv --print-source cuda,sass > $O/src.csv 2>&1
ncu -i /tmp/k.ncu-rep --page source --csv --print-source sass > $O/sass.csv 2>&1
cat $O/launches_c6.md
