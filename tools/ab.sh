#!/bin/bash
# A/B kernel variants on one box: tools/ab.sh "<EXTRA flags B>" [microbench args]
# builds variant B into build_b/ -> libragcache_b200_b.so and runs the attention
# microbench on A (the in-tree build) and B alternately, twice.
set -e
cd "$(dirname "$0")/../paper_2404_12457_b200/csrc"
make -s BUILD=build_b OUT=../libragcache_b200_b.so EXTRA="$1" > /dev/null
cd ../..
shift
for rep in 1 2; do
  for v in a b; do
    if [ $v = b ]; then export RCB_LIB_PATH=$PWD/paper_2404_12457_b200/libragcache_b200_b.so; else unset RCB_LIB_PATH; fi
    python tools/microbench.py "${@:-attn}" 2>&1 | grep -v kv_write | sed "s/^/$v$rep /" | cut -c1-140
  done
done
