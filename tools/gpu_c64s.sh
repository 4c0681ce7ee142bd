#!/bin/bash
# FP64 sampler A/B: parity tests, then C2 FP64 step for the default build and VARIANTS
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
O=${OUT:-gpurun_out/c64s}; mkdir -p $O; P=paper_2202_02264_b200
timeout 1800 python -m pytest tests/test_gpu_c64_screen.py tests/test_gpu_parity.py tests/test_gpu_stress.py \
  tests/test_gpu_baseline_parity.py -m gpu -q -x --timeout 1200 > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
tail -2 $O/pytest.log
cp $P/libdsmc_b200.so /tmp/base.so
for v in base $VARIANTS; do
  [ $v != base ] && cp $P/libdsmc_b200_$v.so $P/libdsmc_b200.so
  timeout 900 python bench.py --config c2 --precision fp64 --steps 5 --warmup 3 --no-cpu-baseline > $O/${v}_c2.json 2> $O/${v}_c2.err
  echo "$v c2 fp64 $(python -c "import json; d=json.load(open('$O/${v}_c2.json')); print(round(d['ms_per_step'],3))" 2>&1 | tail -1)"
  cp /tmp/base.so $P/libdsmc_b200.so
done
DSMC_NO_GRAPH=1 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file $O/launches_c2_fp64.csv python tools/prof_run.py --config c2 --precision fp64 --reps 1 > $O/ncu_launch.log 2>&1
python tools/ncu_summary.py launches $O/launches_c2_fp64.csv > $O/launches_c2_fp64.md 2>&1
echo done
