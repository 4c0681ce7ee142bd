#!/bin/bash
# The other BASELINE configs as bench lines (not the driver's default).
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
for c in c1 c3 c4; do
  timeout 900 python bench.py --config $c --steps 5 --warmup 2 --no-cpu-baseline > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err
done
echo done
