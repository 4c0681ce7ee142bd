#!/bin/bash
# ncu --set full of the top kernels at the current tree: c32_pair / c32_sample /
# leaf32 at C5 and lazy32 at C3 (one launch each, after 3 skipped launches).
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
for spec in "c5 c32_pair" "c5 c32_sample" "c5 leaf32_kernel" "c3 lazy32_kernel"; do
  set -- $spec
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$2 -s 3 -c 1 \
    -o gpurun_out/full_$1_$2 -f python tools/prof_run.py --config $1 --reps 1 > gpurun_out/ncu_full_$1_$2.log 2>&1
  echo "$1 $2 rc=$?"
done
echo done
