#!/bin/bash
# A/B of engine builds made by tools/build_variant.sh: swap each variant .so in
# as libdsmc_b200.so and bench the configs with it (run under gpurun).
#   VARIANTS="base ws0 ws2" CONFIGS="c5 c2" bash tools/ab_so.sh
cd $GRAFT_REPO_ROOT; P=paper_2202_02264_b200
mkdir -p gpurun_out/ab
cp $P/libdsmc_b200.so /tmp/base.so
for v in ${VARIANTS:-base}; do
  if [ $v = base ]; then cp /tmp/base.so $P/libdsmc_b200.so; else cp $P/libdsmc_b200_$v.so $P/libdsmc_b200.so; fi
  for c in ${CONFIGS:-c4 c5}; do
    timeout 400 python bench.py --config $c --steps ${STEPS:-10} --warmup 3 --no-cpu-baseline --no-fp64 \
      > gpurun_out/ab/so_${v}_${c}.json 2> gpurun_out/ab/so_${v}_${c}.err
  done
done
cp /tmp/base.so $P/libdsmc_b200.so
