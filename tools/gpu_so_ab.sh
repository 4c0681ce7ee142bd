#!/bin/bash
# Variant .so A/B: bitwise check of each variant against the main build with
# AB_TOOL (tools/lazy_ab.py or tools/dense_ab.py), then bench CONFIGS per variant.
#   VARIANTS="b8 b16" CONFIGS="c3" AB_TOOL=tools/lazy_ab.py bash tools/gpu_so_ab.sh
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
P=paper_2202_02264_b200; O=gpurun_out/soab; rm -rf $O; mkdir -p $O
cp $P/libdsmc_b200.so /tmp/base.so
timeout 600 python ${AB_TOOL:-tools/lazy_ab.py} run /tmp/base.so $O/base.npz > $O/ab_base.log 2>&1
for v in $VARIANTS; do
  timeout 600 python ${AB_TOOL:-tools/lazy_ab.py} run $P/libdsmc_b200_$v.so $O/$v.npz > $O/ab_$v.log 2>&1
  echo "$v: $(python ${AB_TOOL:-tools/lazy_ab.py} cmp $O/base.npz $O/$v.npz | tail -1)"
done
rm -f $O/*.npz
for v in base $VARIANTS; do
  if [ $v = base ]; then cp /tmp/base.so $P/libdsmc_b200.so; else cp $P/libdsmc_b200_$v.so $P/libdsmc_b200.so; fi
  for c in ${CONFIGS:-c3}; do
    timeout 600 python bench.py --config $c --steps ${STEPS:-10} --warmup 3 --no-cpu-baseline --no-fp64 > $O/${v}_$c.json 2> $O/${v}_$c.err
    python -c "
import json; d=json.load(open('$O/${v}_$c.json')); r=d['roofline']
print('$v $c', 'ms %.3f'%d['ms_per_step'], 'levels', r.get('levels_ms'), 'pair', r.get('pair_kernel_ms_per_step'), 'sample', r.get('sample_kernel_ms_per_step'), 'frac', r.get('frac'))" 2>&1 | tail -1
  done
done
cp /tmp/base.so $P/libdsmc_b200.so
