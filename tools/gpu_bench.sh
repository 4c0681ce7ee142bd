#!/bin/bash
# Bench sweep on one GPU: default (C5) bench, C2 bench, the sharded harness at
# 2 ranks over host-staged gloo (protocol check only), the reference arm.
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err; echo "rc=$?" >> gpurun_out/bench_c5.err
timeout 600 python bench.py --config c2 --no-cpu-baseline > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
if [ "$1" != "quick" ]; then
DSMC_DIST_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
  --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --config c2 --steps 3 --warmup 1 \
  > gpurun_out/bench_c2_gloo2.json 2> gpurun_out/bench_c2_gloo2.err; echo "rc=$?" >> gpurun_out/bench_c2_gloo2.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
fi
echo done
