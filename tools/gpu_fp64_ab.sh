#!/bin/bash
# FP64 parity path A/B: the GPU parity tests on the current build, then the
# C2 / C4 bench lines' FP64 records for the current build and each VARIANT.
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
P=paper_2202_02264_b200; O=gpurun_out/f64ab; rm -rf $O; mkdir -p $O
timeout 1500 python -m pytest ${PYTEST_FILES:-tests/test_gpu_parity.py tests/test_gpu_baseline_parity.py} -m gpu -q -x --timeout 1200 > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log; tail -3 $O/pytest.log
cp $P/libdsmc_b200.so /tmp/base.so
for v in base $VARIANTS; do
  if [ $v != base ]; then cp $P/libdsmc_b200_$v.so $P/libdsmc_b200.so; fi
  for c in ${CONFIGS:-c2}; do
    timeout 900 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline > $O/${v}_$c.json 2> $O/${v}_$c.err
    python -c "
import json; d=json.load(open('$O/${v}_$c.json')); print('$v $c', round(d['ms_per_step'],3), (d.get('fp64_parity') or {}).get('ms_per_step'))"
  done
  cp /tmp/base.so $P/libdsmc_b200.so
done
