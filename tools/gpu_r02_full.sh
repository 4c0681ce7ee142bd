#!/bin/bash
# Round-2 evidence run: smoke, the whole GPU suite, every bench line (CPU legs
# included), the C5 launch list and ncu --set full captures of the top kernels.
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
O=${OUT:-gpurun_out/r02f}; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > $O/smi.txt 2>&1
nproc >> $O/smi.txt; lscpu | grep "Model name" >> $O/smi.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; rc=$?; echo "smoke rc=$rc" >> $O/smoke.log
[ $rc -ne 0 ] && { echo "smoke failed"; exit 1; }
if [ "$ONLY_NCU" != "1" ]; then
timeout 2400 python -m pytest tests -m gpu -q --timeout 900 -rs > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > $O/bench_ref.json 2> $O/bench_ref.err
timeout 900 python bench.py --steps 20 --warmup 5 > $O/bench_c5.json 2> $O/bench_c5.err
for c in c2 c3 c3r c4 c1 c6; do
  timeout 900 python bench.py --config $c --steps 10 --warmup 3 --no-fp64 > $O/bench_$c.json 2> $O/bench_$c.err
done
for c in c6d8 c6d16; do
  timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-fp64 --no-cpu-baseline > $O/bench_$c.json 2> $O/bench_$c.err
done
fi
if [ "$NCU" = "1" ]; then
  # reports stay on the box (/tmp); only summaries travel back (< 64 MiB)
  R=/tmp/ncu_r02; mkdir -p $R
  make -C paper_2202_02264_b200/csrc -j8 > /dev/null 2>&1
  DSMC_NO_GRAPH=1 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv \
    --log-file $O/launches_c5.csv python tools/prof_run.py --config c5 --reps 1 > $O/ncu_launch.log 2>&1
  python tools/ncu_summary.py launches $O/launches_c5.csv > $O/launches_c5.md 2>&1
  # NCU_SPECS: space-separated config:kernel pairs
  for spec in ${NCU_SPECS:-c5:c32_pair c5:c32_sample c3:lazy32_kernel c6:pairw_tc2_kernel c6:samplew_kernel}; do
    set -- ${spec/:/ }
    timeout 900 ncu --set full --clock-control none --import-source on -k regex:$2 -s 3 -c 1 \
      -o $R/full_$1_$2 -f python tools/prof_run.py --config $1 --reps 1 > $O/ncu_full_$1_$2.log 2>&1
    echo "$1 $2 rc=$?" >> $O/ncu_status.txt
    python tools/ncu_summary.py report $R/full_$1_$2.ncu-rep > $O/full_$1_$2.md 2>&1
    ncu -i $R/full_$1_$2.ncu-rep --page raw --csv > $O/full_$1_$2_raw.csv 2>&1
  done
fi
echo done
