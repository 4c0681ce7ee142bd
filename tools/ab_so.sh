#!/bin/bash
# A/B of engine builds made by tools/build_variant.sh: swap each variant .so in
# as libdsmc_b200.so and bench C4 / C5 with it (run under gpurun).
cd $GRAFT_REPO_ROOT; P=paper_2202_02264_b200
cp $P/libdsmc_b200.so /tmp/base.so
for v in base s4 s5; do
  if [ $v = base ]; then cp /tmp/base.so $P/libdsmc_b200.so; else cp $P/libdsmc_b200_$v.so $P/libdsmc_b200.so; fi
  for c in c4 c5; do timeout 400 python bench.py --config $c --no-cpu-baseline > gpurun_out/so_${v}_${c}.json 2>/dev/null; done
done
cp /tmp/base.so $P/libdsmc_b200.so
