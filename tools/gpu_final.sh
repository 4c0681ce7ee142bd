#!/bin/bash
# Round-end evidence: GPU tests, smoke, default bench, C5 launch list, full
# ncu captures of the pair / sample / leaf kernels (each after its own
# command ran clean without ncu).
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err
bash tools/gpu_prof.sh c5
timeout 900 ncu --set full --clock-control none --import-source on -k regex:leaf32 -c 1 \
  -o gpurun_out/leaf_c5 -f python tools/prof_run.py --config c5 --reps 1 > gpurun_out/ncu_leaf.log 2>&1
echo done
