#!/bin/bash
# Round-2 GPU session: parity + safety tests, smoke, default bench (C5) with
# its FP64 record and CPU leg, the reference arm, and the C5 FP32/FP64 law.
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out/r02
O=gpurun_out/r02
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > $O/smi.txt 2>&1
nproc >> $O/smi.txt; lscpu | grep "Model name" >> $O/smi.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; rc=$?; echo "smoke rc=$rc" >> $O/smoke.log
[ $rc -ne 0 ] && { echo "smoke failed; stopping"; exit 1; }
timeout 1800 python -m pytest tests -m gpu -q --timeout 600 ${PYTEST_ARGS} > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 900 python bench.py > $O/bench_c5.json 2> $O/bench_c5.err
timeout 900 python tools/c5_law.py c5 16 > $O/c5_law.jsonl 2> $O/c5_law.err
echo done
