#!/bin/bash
# Interleaved default-workload bench lines over prebuilt variants: tools/ab_bench.sh <out> a x ...
cd "$(dirname "$0")/.."
out=$1; shift
for rep in 1 2 3; do
  for v in "$@"; do
    if [ "$v" = a ]; then unset RCB_LIB_PATH; else export RCB_LIB_PATH=$PWD/paper_2404_12457_b200/libragcache_b200_$v.so; fi
    timeout 600 python bench.py --no-ttft --no-cpu-baseline --no-hit-sweep --no-model-step 2>/dev/null | tail -1 | \
      python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$v$rep', d['value'], d['ms_per_step'], r['launch_ms_mean'], d['clocks']['sm_mhz'])"
  done
done > gpurun_out/${out}.txt 2>&1
