#!/bin/bash
# Round-2 iteration: tests for the FP64 register fill, the batched MH steps and
# the device wide prep, bitwise lazy A/B against the serial-MH build, timings.
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
P=paper_2202_02264_b200; O=gpurun_out/g; rm -rf $O; mkdir -p $O
make -C $P/csrc -j8 > $O/make.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1 || { echo smoke failed; cat $O/smoke.log; exit 1; }
timeout 2400 python -m pytest ${PYTEST_FILES:-tests/test_gpu_parity.py tests/test_gpu_baseline_parity.py tests/test_gpu_wide.py tests/test_gpu_stat.py tests/test_gpu_safety.py tests/test_gpu_pgibbs.py} -m gpu -q --timeout 1200 > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
tail -4 $O/pytest.log
timeout 600 python tools/lazy_ab.py run $P/libdsmc_b200.so $O/la.npz > $O/lazy_a.log 2>&1
timeout 600 python tools/lazy_ab.py run $P/libdsmc_b200_serial.so $O/lb.npz > $O/lazy_b.log 2>&1
python tools/lazy_ab.py cmp $O/la.npz $O/lb.npz > $O/lazy_cmp.txt 2>&1; rm -f $O/la.npz $O/lb.npz; tail -1 $O/lazy_cmp.txt
b() { timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline "$@"; }
b --config c3 --no-fp64 > $O/c3_batched.json 2> $O/c3_batched.err
cp $P/libdsmc_b200.so /tmp/main.so; cp $P/libdsmc_b200_serial.so $P/libdsmc_b200.so
b --config c3 --no-fp64 > $O/c3_serial.json 2> $O/c3_serial.err
cp /tmp/main.so $P/libdsmc_b200.so
b --config c2 > $O/c2_vpl.json 2> $O/c2_vpl.err
DSMC_C64_REFILL=1 b --config c2 > $O/c2_refill.json 2> $O/c2_refill.err
b --config c6 --no-fp64 > $O/c6.json 2> $O/c6.err
b --config c6d8 --no-fp64 > $O/c6d8.json 2> $O/c6d8.err
for f in $O/*.json; do python - "$f" <<'PY'
import json, sys
f = sys.argv[1]
try:
    d = json.load(open(f))
except Exception as e:
    print(f, "FAILED", e); sys.exit()
r = d.get("roofline", {})
print(f.split("/")[-1], "ms %.3f" % d["ms_per_step"], "val %.4g" % d["value"], "e2e %.4g" % d["e2e"]["value"],
      "levels", r.get("levels_ms"), "fp64", (d.get("fp64_parity") or {}).get("ms_per_step"))
PY
done
