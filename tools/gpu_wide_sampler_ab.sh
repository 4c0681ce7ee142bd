#!/bin/bash
# Wide-path A/B: wide / large-N GPU tests on the current build, then the
# C6 lines (d = 32 / 16 / 8) for the current build and each VARIANT .so.
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
P=paper_2202_02264_b200; O=gpurun_out/w; rm -rf $O; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_wide.py tests/test_gpu_stat.py -k "wide or large_n" -m gpu -q > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log; tail -2 $O/pytest.log
cp $P/libdsmc_b200.so /tmp/base.so
for v in base $VARIANTS; do
  [ $v != base ] && cp $P/libdsmc_b200_$v.so $P/libdsmc_b200.so
  for c in ${CONFIGS:-c6 c6d16 c6d8}; do
    timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-fp64 > $O/${v}_$c.json 2>$O/${v}_$c.err
    python -c "
import json; d=json.load(open('$O/${v}_$c.json')); r=d['roofline']; print('$v $c', round(d['ms_per_step'],3), 'e2e %.4g'%d['e2e']['value'], 'leaf', round(r.get('leaf_ms'),3), 'pair', round(r.get('pair_kernel_ms_per_step'),3), 'sample', round(r.get('sample_kernel_ms_per_step'),3))"
  done
  cp /tmp/base.so $P/libdsmc_b200.so
done
