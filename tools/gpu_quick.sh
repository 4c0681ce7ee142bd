#!/bin/bash
# Quick GPU iteration: selected pytest files (PYTEST_FILES), the C++ host
# binaries, and short bench lines (C5, C2) without the CPU / FP64 legs.
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
O=gpurun_out/q; mkdir -p $O
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1 || { echo smoke failed; cat $O/smoke.log; exit 1; }
if [ -n "$PYTEST_FILES" ]; then
  timeout 1200 python -m pytest $PYTEST_FILES -m gpu -q --timeout 600 > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
fi
./tests/cpp/test_host > $O/test_host.log 2>&1; echo "rc=$?" >> $O/test_host.log
./tests/cpp/_ref/test_resampling > $O/test_resampling.log 2>&1; echo "rc=$?" >> $O/test_resampling.log
for c in ${BENCH_CONFIGS:-c5 c2}; do
  timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-fp64 > $O/bench_$c.json 2> $O/bench_$c.err
done
echo done
