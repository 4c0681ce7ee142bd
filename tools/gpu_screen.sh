#!/bin/bash
# FP64 pass-1 row-max screen: bit-identity tests, then C2 / C5 FP64 timing with
# the screen off and on, and one ncu --set full capture of c64_rows.
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
O=${OUT:-gpurun_out/screen}; mkdir -p $O
timeout 1800 python -m pytest tests/test_gpu_c64_screen.py tests/test_gpu_parity.py tests/test_gpu_stress.py \
  tests/test_gpu_baseline_parity.py -m gpu -q -x --timeout 1200 > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
tail -3 $O/pytest.log
for s in 0 1; do
  DSMC_C64_SCREEN=$s timeout 900 python bench.py --config c2 --precision fp64 --steps 5 --warmup 3 --no-cpu-baseline > $O/c2_fp64_s$s.json 2> $O/c2_fp64_s$s.err
  python tools/show_bench.py $O/c2_fp64_s$s.json 2>/dev/null | head -3
done
DSMC_C64_SCREEN=1 timeout 900 python bench.py --config c5 --precision fp64 --steps 2 --warmup 1 --no-cpu-baseline > $O/c5_fp64_s1.json 2> $O/c5_fp64_s1.err
if [ "$NCU" = "1" ]; then
  R=/tmp/ncu_scr; mkdir -p $R
  DSMC_NO_GRAPH=1 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file $O/launches_c2_fp64.csv python tools/prof_run.py --config c2 --precision fp64 --reps 1 > $O/ncu_launch.log 2>&1
  python tools/ncu_summary.py launches $O/launches_c2_fp64.csv > $O/launches_c2_fp64.md 2>&1
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:c64_rows -s 2 -c 1 \
    -o $R/full_c2_c64_rows -f python tools/prof_run.py --config c2 --precision fp64 --reps 1 > $O/ncu_full.log 2>&1
  python tools/ncu_summary.py report $R/full_c2_c64_rows.ncu-rep > $O/full_c2_c64_rows.md 2>&1
fi
echo done
