#!/bin/bash
# Streaming tcgen05 pass 1 (DSMC_PAIR_KERNEL=tc2): tests, C2 / C5 A/B against
# the CUDA-core kernel, and one ncu --set full capture of c32_pair_tc2.
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
O=${OUT:-gpurun_out/tc2}; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_pair_tc.py -m gpu -q -x --timeout 600 > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
tail -3 $O/pytest.log
for c in ${CONFIGS:-c2 c5}; do
  for k in fma tc2; do
    DSMC_PAIR_KERNEL=$k timeout 600 python bench.py --config $c --steps ${STEPS:-5} --warmup 3 --no-cpu-baseline --no-fp64 > $O/${k}_$c.json 2> $O/${k}_$c.err
    python tools/show_bench.py $O/${k}_$c.json | head -2
  done
done
if [ "$NCU" = "1" ]; then
  R=/tmp/ncu_tc2; mkdir -p $R
  DSMC_PAIR_KERNEL=tc2 timeout 600 ncu --set full --clock-control none --import-source on -k regex:c32_pair_tc2 -s 2 -c 1 \
    -o $R/full -f python tools/prof_run.py --config c2 --reps 1 > $O/ncu_full.log 2>&1
  python tools/ncu_summary.py report $R/full.ncu-rep > $O/full_c2_c32_pair_tc2.md 2>&1
  ncu -i $R/full.ncu-rep --page source --csv --print-source cuda,sass > $O/src.csv 2>&1
  ncu -i $R/full.ncu-rep --page source --csv --print-source sass > $O/sass.csv 2>&1
fi
echo done
