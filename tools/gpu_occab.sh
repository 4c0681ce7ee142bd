#!/bin/bash
# Occupancy A/B: the default build vs VARIANTS (libdsmc_b200_<v>.so) on CONFIGS
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
P=paper_2202_02264_b200; O=${OUT:-gpurun_out/occab}; mkdir -p $O; cp $P/libdsmc_b200.so /tmp/base.so
for v in base $VARIANTS; do
  [ $v != base ] && cp $P/libdsmc_b200_$v.so $P/libdsmc_b200.so
  for c in ${CONFIGS:-c3 c5}; do
    timeout 600 python bench.py --config $c --steps ${STEPS:-10} --warmup 3 --no-cpu-baseline --no-fp64 > $O/${v}_$c.json 2>/dev/null
    echo "$v $c $(python -c "import json; d=json.load(open('$O/${v}_$c.json')); r=d['roofline']; print(round(d['ms_per_step'],3), 'leaf', round(r.get('leaf_ms') or 0,3), 'levels', round(r.get('levels_ms') or 0,3))")"
  done
  cp /tmp/base.so $P/libdsmc_b200.so
done
