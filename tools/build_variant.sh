#!/bin/bash
# build_variant.sh NAME FLAGS... : engine variant as ../libdsmc_b200_NAME.so
set -e
cd /root/repo/paper_2202_02264_b200/csrc
name=$1; shift
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 --expt-relaxed-constexpr \
  -Xcompiler -fPIC -Xcompiler -fvisibility=hidden -I../../include "$@" -c engine.cu -o /tmp/engine_$name.o
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o ../libdsmc_b200_$name.so /tmp/engine_$name.o kalman.o -lcudart
