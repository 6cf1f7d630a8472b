#!/bin/bash
# builds libsfkv variants with different compile-time switches into exp/
set -e
cd "$(dirname "$0")"; mkdir -p ../../exp
NVCC=/usr/local/cuda/bin/nvcc
FLAGS="-O3 -std=c++17 -lineinfo -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC,-O2 --expt-relaxed-constexpr"
for v in "$@"; do
  name=${v%%:*}; defs=${v#*:}
  D=""; for d in ${defs//,/ }; do D="$D -D$d"; done
  mkdir -p /tmp/var_$name
  for f in abi match commit copy mm_map tracker tokenize metrics; do $NVCC $FLAGS $D -c $f.cu -o /tmp/var_$name/$f.o & done; wait
  $NVCC -gencode arch=compute_100a,code=sm_100a -shared -o ../../exp/libsfkv_$name.so /tmp/var_$name/*.o
  echo built $name
done
