#!/bin/bash
# A/B: pick4 in the leaf kernels (new, in-tree build) vs libdsmc_b200_base.so
cd "$GRAFT_REPO_ROOT"; P=paper_2202_02264_b200
python tools/dense_ab.py run $P/libdsmc_b200_base.so gpurun_out/dab_base.npz > gpurun_out/dab_cmp.log 2>&1
python tools/dense_ab.py run $P/libdsmc_b200.so gpurun_out/dab_new.npz >> gpurun_out/dab_cmp.log 2>&1
python tools/dense_ab.py cmp gpurun_out/dab_base.npz gpurun_out/dab_new.npz >> gpurun_out/dab_cmp.log 2>&1
python tools/lazy_ab.py run $P/libdsmc_b200_base.so gpurun_out/lab_base.npz > gpurun_out/lab_cmp.log 2>&1
python tools/lazy_ab.py run $P/libdsmc_b200.so gpurun_out/lab_new.npz >> gpurun_out/lab_cmp.log 2>&1
python tools/lazy_ab.py cmp gpurun_out/lab_base.npz gpurun_out/lab_new.npz >> gpurun_out/lab_cmp.log 2>&1
cp $P/libdsmc_b200.so /tmp/new.so
for v in base new; do
  if [ $v = base ]; then cp $P/libdsmc_b200_base.so $P/libdsmc_b200.so; else cp /tmp/new.so $P/libdsmc_b200.so; fi
  for c in c5 c3; do timeout 400 python bench.py --config $c --no-cpu-baseline > gpurun_out/ablf_${v}_${c}.json 2>/dev/null; done
done
cp /tmp/new.so $P/libdsmc_b200.so
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
