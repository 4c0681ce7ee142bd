cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
P=paper_2202_02264_b200; cp $P/libdsmc_b200.so /tmp/base.so
for v in base sw4; do
  [ $v = sw4 ] && cp $P/libdsmc_b200_sw4.so $P/libdsmc_b200.so
  [ $v = sw4 ] && timeout 600 python -m pytest tests/test_gpu_wide.py -m gpu -q -x --timeout 600 2>&1 | tail -1
  for c in c6 c6d16 c6d8; do
    timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-fp64 > gpurun_out/sw_${v}_$c.json 2>/dev/null
    echo "$v $c $(python -c "import json; d=json.load(open('gpurun_out/sw_${v}_$c.json')); r=d['roofline']; print(round(d['ms_per_step'],3), 'sample', round(r['sample_kernel_ms_per_step'],3))")"
  done
  cp /tmp/base.so $P/libdsmc_b200.so
done
