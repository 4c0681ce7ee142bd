#!/bin/bash
# Bitwise + timing A/B of an engine env switch (same build): the dense FP32
# A/B cases (tools/dense_ab.py) with and without the switch, then bench lines.
#   FLAG=DSMC_SAMPLER_WALK CONFIGS="c5 c2 c4" bash tools/env_ab.sh
cd $GRAFT_REPO_ROOT; P=paper_2202_02264_b200; O=gpurun_out/envab; mkdir -p $O
FLAG=${FLAG:-DSMC_SAMPLER_WALK}
make -C $P/csrc -j8 > $O/make.log 2>&1
L=$P/libdsmc_b200.so
env $FLAG=1 timeout 600 python tools/dense_ab.py run $L $O/a.npz > $O/ab_a.log 2>&1
timeout 600 python tools/dense_ab.py run $L $O/b.npz > $O/ab_b.log 2>&1
python tools/dense_ab.py cmp $O/a.npz $O/b.npz > $O/cmp.txt 2>&1
rm -f $O/a.npz $O/b.npz
for c in ${CONFIGS:-c5 c2 c4}; do
  for v in 1 0; do
    env $FLAG=$v timeout 600 python bench.py --config $c --steps ${STEPS:-10} --warmup 3 --no-cpu-baseline --no-fp64 \
      > $O/bench_${c}_$FLAG$v.json 2> $O/bench_${c}_$FLAG$v.err
  done
done
cat $O/cmp.txt
for f in $O/bench_*.json; do python -c "
import json,sys; d=json.load(open('$f')); print('$f', d['ms_per_step'], d['roofline'].get('sample_kernel_ms_per_step'), d['roofline'].get('pair_kernel_ms_per_step'))"; done
