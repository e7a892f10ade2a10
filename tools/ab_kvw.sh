# kv_write_rope variants: tools/ab_kvw.sh a t4u1 ...  (MB_CASE selects the attention cases)
cd "$(dirname "$0")/.."
for rep in 1 2; do
  for v in "$@"; do
    if [ "$v" = a ]; then unset RCB_LIB_PATH; else export RCB_LIB_PATH=$PWD/paper_2404_12457_b200/libragcache_b200_$v.so; fi
    python tools/microbench.py attn 2>&1 | grep kv_write | sed "s/^/$v$rep /"
  done
done
