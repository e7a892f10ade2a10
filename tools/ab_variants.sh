#!/bin/bash
# Interleaved attention microbench over prebuilt variants (full JSON lines):
#   tools/ab_variants.sh <out> a qp rf ...   (a = in-tree build, x = libragcache_b200_x.so)
# Each non-default variant first runs the attention parity tests.
cd "$(dirname "$0")/.."
out=$1; shift
for v in "$@"; do
  [ "$v" = a ] && continue
  RCB_LIB_PATH=$PWD/paper_2404_12457_b200/libragcache_b200_$v.so timeout 600 python -m pytest \
    tests/test_gpu_kernels.py -x -q -k "prefix_prefill" > gpurun_out/${out}_tests_$v.txt 2>&1
  echo "rc=$?" >> gpurun_out/${out}_tests_$v.txt
done
for rep in 1 2; do
  for v in "$@"; do
    if [ "$v" = a ]; then unset RCB_LIB_PATH; else export RCB_LIB_PATH=$PWD/paper_2404_12457_b200/libragcache_b200_$v.so; fi
    python tools/microbench.py attn 2>&1 | grep '"prefix_prefill' | sed "s/^/$v$rep /"
  done
done > gpurun_out/${out}.txt
