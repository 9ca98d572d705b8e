#!/bin/bash
# build merge-kernel parameter variants into paper_2209_06909_b200/libps_var_*.so
set -e
NV="/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-O2 -shared --expt-relaxed-constexpr -diag-suppress 177,1886"
for v in "$@"; do
  name=$(echo $v | tr ',=' '__')
  flags=$(echo $v | tr ',' ' ' | sed 's/\([A-Z0-9_]*=[0-9]*\)/-D\1/g')
  $NV $flags -o paper_2209_06909_b200/libps_var_$name.so paper_2209_06909_b200/csrc/powersort.cu &
done
wait
ls paper_2209_06909_b200/libps_var_*.so
