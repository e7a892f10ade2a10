#!/bin/bash
# tools/ab_multi.sh "<flags v1>" "<flags v2>" ... : build each variant and run the
# attention microbench on the in-tree build (a) and every variant, on one box.
set -e
root="$(cd "$(dirname "$0")/.." && pwd)"
i=0
for flags in "$@"; do
  i=$((i+1))
  (cd "$root/paper_2404_12457_b200/csrc" && make -s BUILD=build_v$i OUT=../libragcache_b200_v$i.so EXTRA="$flags" > /dev/null)
done
cd "$root"
for rep in 1 2; do
  unset RCB_LIB_PATH
  python tools/microbench.py attn 2>&1 | grep -v kv_write | sed "s/^/a$rep /" | cut -c1-120
  for j in $(seq 1 $i); do
    RCB_LIB_PATH=$root/paper_2404_12457_b200/libragcache_b200_v$j.so python tools/microbench.py attn 2>&1 | grep -v kv_write | sed "s/^/v$j.$rep /" | cut -c1-120
  done
done
