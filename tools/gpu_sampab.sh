#!/bin/bash
# Bitwise + timing A/B of the FP32 dense path: the default build vs
# libdsmc_b200_base.so (tools/dense_ab.py), then C5 / C2 bench lines of both.
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
O=${OUT:-gpurun_out/sampab}; mkdir -p $O; P=paper_2202_02264_b200
python tools/dense_ab.py run $P/libdsmc_b200.so $O/new.npz > $O/ab.log 2>&1
python tools/dense_ab.py run $P/libdsmc_b200_base.so $O/base.npz >> $O/ab.log 2>&1
python tools/dense_ab.py cmp $O/base.npz $O/new.npz >> $O/ab.log 2>&1
cat $O/ab.log | tail -12
cp $P/libdsmc_b200.so /tmp/new.so
for v in new base; do
  [ $v = base ] && cp $P/libdsmc_b200_base.so $P/libdsmc_b200.so
  for c in ${CONFIGS:-c5 c2}; do
    timeout 600 python bench.py --config $c --steps ${STEPS:-10} --warmup 3 --no-cpu-baseline --no-fp64 > $O/${v}_$c.json 2> /dev/null
    echo "$v $c $(python -c "import json; d=json.load(open('$O/${v}_$c.json')); r=d['roofline']; print(round(d['ms_per_step'],3), 'pair', round(r['pair_kernel_ms_per_step'],2), 'sample', round(r['sample_kernel_ms_per_step'],2))")"
  done
  cp /tmp/new.so $P/libdsmc_b200.so
done
