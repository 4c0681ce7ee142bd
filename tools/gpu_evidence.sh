#!/bin/bash
# Round-end evidence at the current tree: GPU tests, smoke, the default bench
# line (C5, with the CPU baseline), C1-C4 bench lines, the reference arm, and
# the C5 launch list (eager launches) for kernel shares.
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err
for c in c1 c2 c3 c4; do
  timeout 900 python bench.py --config $c --no-cpu-baseline > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err
done
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
# eager launches: ncu does not survive a graph replay with programmatic edges
DSMC_NO_GRAPH=1 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv \
  --log-file gpurun_out/launches_c5.csv python tools/prof_run.py --config c5 --reps 1 > gpurun_out/ncu_launch.log 2>&1
echo done
