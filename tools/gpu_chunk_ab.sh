#!/bin/bash
# Chunk-size sweep: DSMC_WS_BUDGET_MB (pass-1 sub-block sums per chunk) vs
# the C5 / C2 step and the pair / sampler split.
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
O=gpurun_out/chunk; rm -rf $O; mkdir -p $O
for mb in ${BUDGETS:-1024 256 128 64 32}; do
  for c in ${CONFIGS:-c5}; do
    DSMC_WS_BUDGET_MB=$mb timeout 900 python bench.py --config $c --steps ${STEPS:-5} --warmup 3 --no-cpu-baseline --no-fp64 > $O/${c}_$mb.json 2> $O/${c}_$mb.err
    python -c "
import json; d=json.load(open('$O/${c}_$mb.json')); r=d['roofline']
print('$c $mb MB', 'ms %.3f'%d['ms_per_step'], 'pair', r.get('pair_kernel_ms_per_step'), 'sample', r.get('sample_kernel_ms_per_step'), 'launches', d.get('gpu_launches'))"
  done
done
