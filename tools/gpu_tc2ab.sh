#!/bin/bash
# tc2 variants A/B (C2, C5 pass-1 ms): default build vs libdsmc_b200_<v>.so
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
O=${OUT:-gpurun_out/tc2ab}; mkdir -p $O; P=paper_2202_02264_b200
timeout 900 python -m pytest tests/test_gpu_pair_tc.py -m gpu -q -x --timeout 600 > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
tail -2 $O/pytest.log
cp $P/libdsmc_b200.so /tmp/base.so
for v in base $VARIANTS; do
  [ $v != base ] && cp $P/libdsmc_b200_$v.so $P/libdsmc_b200.so
  for c in ${CONFIGS:-c2 c5}; do
    DSMC_PAIR_KERNEL=tc2 timeout 600 python bench.py --config $c --steps ${STEPS:-5} --warmup 3 --no-cpu-baseline --no-fp64 > $O/${v}_$c.json 2> $O/${v}_$c.err
    echo "$v $c $(python -c "import json; d=json.load(open('$O/${v}_$c.json')); r=d['roofline']; print(round(d['ms_per_step'],3), 'pair', round(r['pair_kernel_ms_per_step'],2), 'frac', round(r['frac'],4))" 2>&1 | tail -1)"
  done
  cp /tmp/base.so $P/libdsmc_b200.so
done
echo done
