#!/bin/bash
# Run the attention microbench on prebuilt library variants, interleaved twice:
#   tools/abn.sh a b c   (a = in-tree libragcache_b200.so, x = libragcache_b200_x.so)
# MB_CASE selects the microbench case(s).
cd "$(dirname "$0")/.."
for rep in 1 2; do
  for v in "$@"; do
    if [ "$v" = a ]; then unset RCB_LIB_PATH; else export RCB_LIB_PATH=$PWD/paper_2404_12457_b200/libragcache_b200_$v.so; fi
    python tools/microbench.py attn 2>&1 | grep -v kv_write | sed "s/^/$v$rep /" | cut -c1-150
  done
done
