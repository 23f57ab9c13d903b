#!/bin/bash
# Build libps variants with other far1p tilings (factor elements per staged item, ring stages)
# into ab_libs/ for an A/B on the GPU box:  PS_LIB=ab_libs/libps_CH_NS.so python bench.py ...
set -u
cd "$(dirname "$0")/.."
mkdir -p ab_libs
for v in "$@"; do
  ch=${v%_*}; ns=${v#*_}
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -lineinfo -O3 -std=c++17 -Xcompiler -fPIC --shared \
    -DPS_F1P_CH=$ch -DPS_F1P_NS=$ns paper_2109_04129_b200/csrc/ps_kernels.cu paper_2109_04129_b200/csrc/ps_rcs.cu \
    paper_2109_04129_b200/csrc/ps_host.cpp -o ab_libs/libps_${ch}_${ns}.so -ldl > ab_libs/build_${ch}_${ns}.log 2>&1 &
done
wait
ls -la ab_libs/*.so
