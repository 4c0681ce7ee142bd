cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out/q
timeout 900 python -m pytest tests/test_gpu_wide.py -m gpu -q --timeout 600 > gpurun_out/q/pytest_wide.log 2>&1; echo "rc=$?" >> gpurun_out/q/pytest_wide.log
for c in c6 c6d16 c6d8; do
  timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-fp64 > gpurun_out/q/wtc_$c.json 2> gpurun_out/q/wtc_$c.err
  DSMC_WIDE_PAIR=fma timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-fp64 > gpurun_out/q/wfma_$c.json 2> gpurun_out/q/wfma_$c.err
done
