#!/bin/bash
# A/B of the K/V write's tokens per CTA (RCB_KV_UNITS variants): parity, then interleaved microbench
cd "$(dirname "$0")/.."
for v in u512 u1024 u2048; do
  RCB_LIB_PATH=$PWD/paper_2404_12457_b200/libragcache_b200_$v.so timeout 600 python -m pytest \
    tests/test_gpu_kernels.py -x -q -k "kv_write" > gpurun_out/kvt_tests_$v.txt 2>&1
  echo "rc=$?" >> gpurun_out/kvt_tests_$v.txt
done
for rep in 1 2; do
  for v in a u512 u1024 u2048; do
    if [ "$v" = a ]; then unset RCB_LIB_PATH; else export RCB_LIB_PATH=$PWD/paper_2404_12457_b200/libragcache_b200_$v.so; fi
    for c in llama2 "mistral mixed"; do
      MB_CASE="$c" python tools/microbench.py attn 2>&1 | grep '"kv_write' | sed "s/^/$v$rep /"
    done
  done
done > gpurun_out/kvt.txt
