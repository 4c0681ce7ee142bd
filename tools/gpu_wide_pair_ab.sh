#!/bin/bash
# Wide pass-1 A/B: wide GPU tests (default kernel), then the C6 lines with
# DSMC_WIDE_PAIR = default (pipelined tcgen05) / tc1 (first tcgen05) / fma.
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
O=gpurun_out/wp; rm -rf $O; mkdir -p $O
make -C paper_2202_02264_b200/csrc -j8 > $O/make.log 2>&1
timeout 900 python -m pytest tests/test_gpu_wide.py -m gpu -q -x > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log; tail -3 $O/pytest.log
for k in tc2 tc1 fma; do
  for c in ${CONFIGS:-c6 c6d16 c6d8}; do
    DSMC_WIDE_PAIR=$k timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-fp64 > $O/${k}_$c.json 2>$O/${k}_$c.err
    python -c "
import json; d=json.load(open('$O/${k}_$c.json')); r=d['roofline']; print('$k $c', round(d['ms_per_step'],3), 'pair', round(r.get('pair_kernel_ms_per_step'),3), 'frac', round(r.get('frac'),3), 'sample', round(r.get('sample_kernel_ms_per_step'),3))" 2>&1 | tail -1
  done
done
