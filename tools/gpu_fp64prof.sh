#!/bin/bash
# FP64 parity path profile at C2: launch list + full/source captures of
# c64_rows and c64_sample.
O=gpurun_out/fp64; mkdir -p $O; R=/tmp/ncu_fp64; mkdir -p $R
make -C paper_2202_02264_b200/csrc -j8 > $O/make.log 2>&1
DSMC_NO_GRAPH=1 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv \
  --log-file $O/launches_c2.csv python tools/prof_run.py --config c2 --reps 1 --precision fp64 > $O/ncu_launch.log 2>&1
python tools/ncu_summary.py launches $O/launches_c2.csv > $O/launches_c2.md 2>&1
for k in c64_rows c64_sample; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k -s 2 -c 1 \
    -o $R/$k -f python tools/prof_run.py --config c2 --reps 1 --precision fp64 > $O/ncu_$k.log 2>&1
  python tools/ncu_summary.py report $R/$k.ncu-rep > $O/full_$k.md 2>&1
  ncu -i $R/$k.ncu-rep --page source --csv --print-source cuda,sass > $O/src_$k.csv 2>&1
  ncu -i $R/$k.ncu-rep --page source --csv --print-source sass > $O/sass_$k.csv 2>&1
done
cat $O/launches_c2.md
