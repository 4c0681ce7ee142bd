#!/bin/bash
# Iteration run: smoke, selected GPU tests, bench lines with optional extra
# flags per config (BENCH="c2:--no-cpu-baseline c6:--no-cpu-baseline --no-fp64").
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
O=gpurun_out/it; rm -rf $O; mkdir -p $O
make -C paper_2202_02264_b200/csrc -j8 > $O/make.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1 || { echo smoke failed; cat $O/smoke.log; exit 1; }
if [ -n "$PYTEST_FILES" ]; then
  timeout 1500 python -m pytest $PYTEST_FILES -m gpu -q --timeout 900 -x > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
  tail -5 $O/pytest.log
fi
IFS=';' read -ra BS <<< "$BENCH"
for spec in "${BS[@]}"; do
  c=${spec%%:*}; fl=${spec#*:}
  timeout 900 python bench.py --config $c --steps ${STEPS:-10} --warmup 3 $fl > $O/bench_$c.json 2> $O/bench_$c.err
  python - <<PY
import json
d=json.load(open("$O/bench_$c.json")); r=d.get("roofline",{})
print("$c", "ms", round(d["ms_per_step"],3), "val %.4g"%d["value"], "e2e %.4g"%d["e2e"]["value"],
      "pair", r.get("pair_kernel_ms_per_step"), "sample", r.get("sample_kernel_ms_per_step"),
      "fp64", (d.get("fp64_parity") or {}).get("ms_per_step"))
PY
done
echo done
