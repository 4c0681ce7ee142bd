#!/bin/bash
# Source-level (SASS + CUDA line) counters of one kernel launch: instruction
# counts and stall samples per line, to find where a kernel's issue slots go.
#   KCONF=c5 KREGEX=c32_sample bash tools/gpu_src.sh
set -u
O=gpurun_out/src; mkdir -p $O
R=/tmp/ncu_src; mkdir -p $R
KCONF=${KCONF:-c5}; KREGEX=${KREGEX:-c32_sample}
make -C paper_2202_02264_b200/csrc -j8 > $O/make.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:$KREGEX -s 3 -c 1 \
  -o $R/src -f python tools/prof_run.py --config $KCONF --reps 1 > $O/ncu.log 2>&1
echo "rc=$?" >> $O/ncu.log
ncu -i $R/src.ncu-rep --page source --csv --print-source cuda,sass > $O/src_${KCONF}_${KREGEX}.csv 2>&1
ncu -i $R/src.ncu-rep --page source --csv --print-source sass > $O/sass_${KCONF}_${KREGEX}.csv 2>&1
python tools/ncu_summary.py report $R/src.ncu-rep > $O/full_${KCONF}_${KREGEX}.md 2>&1
ls -la $O
