#!/bin/bash
# A/B of the pass-1 kernels (tensor-core c32_pair_tc vs CUDA-core c32_pair):
# GPU tests on the default kernel, then C2 / C4 / C5 bench lines for both.
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
for k in tc fma; do
  for c in ${CONFIGS:-c2 c4 c5}; do
    DSMC_PAIR_KERNEL=$k timeout 900 python bench.py --config $c --no-cpu-baseline > gpurun_out/ab_${k}_${c}.json 2> gpurun_out/ab_${k}_${c}.err
  done
done
echo done
