#!/bin/bash
# Quarter-sum sampler A/B: statistical GPU tests on the current build, then
# bench lines for: current build, current build with DSMC_SAMPLER_FULL64=1,
# and the previous build (libdsmc_b200_head.so).
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
P=paper_2202_02264_b200; O=gpurun_out/qs; rm -rf $O; mkdir -p $O
timeout 2000 python -m pytest ${PYTEST_FILES:-tests/test_gpu_stat.py tests/test_gpu_c5_law.py tests/test_gpu_invariance.py tests/test_gpu_pgibbs.py} -m gpu -q --timeout 1500 > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log; tail -3 $O/pytest.log
b() { timeout 900 python bench.py --config $1 --steps ${STEPS:-10} --warmup 3 --no-cpu-baseline --no-fp64 > $O/$2_$1.json 2> $O/$2_$1.err
  python -c "
import json; d=json.load(open('$O/$2_$1.json')); r=d['roofline']
print('$2 $1', 'ms %.3f'%d['ms_per_step'], 'pair', r.get('pair_kernel_ms_per_step'), 'sample', r.get('sample_kernel_ms_per_step'))"; }
for c in ${CONFIGS:-c5 c2 c4}; do
  b $c qs
  DSMC_SAMPLER_FULL64=1 b $c full64
done
cp $P/libdsmc_b200.so /tmp/base.so; cp $P/libdsmc_b200_head.so $P/libdsmc_b200.so
for c in ${CONFIGS:-c5 c2 c4}; do b $c head; done
cp /tmp/base.so $P/libdsmc_b200.so
