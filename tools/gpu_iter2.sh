#!/bin/bash
# gpu_iter.sh + a source-level ncu capture of one kernel (KCONF/KREGEX/KPREC)
bash tools/gpu_iter.sh
if [ -n "$KREGEX" ]; then
  O=gpurun_out/it; R=/tmp/ncu_it; mkdir -p $R
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$KREGEX -s ${KSKIP:-2} -c 1 \
    -o $R/k -f python tools/prof_run.py --config $KCONF --reps 1 --precision ${KPREC:-fp32} > $O/ncu.log 2>&1
  python tools/ncu_summary.py report $R/k.ncu-rep > $O/full_${KCONF}_$KREGEX.md 2>&1
  ncu -i $R/k.ncu-rep --page source --csv --print-source cuda,sass > $O/src_k.csv 2>&1
  ncu -i $R/k.ncu-rep --page source --csv --print-source sass > $O/sass_k.csv 2>&1
  head -30 $O/full_${KCONF}_$KREGEX.md
fi
