# item-boundary + softmax-phase timelines of CTA 0 (trace builds; under gpurun)
mkdir -p gpurun_out
for lib in tr trns; do
  export RCB_LIB_PATH=$PWD/paper_2404_12457_b200/libragcache_b200_$lib.so
  for c in mistral_long mistral_mixed llama2_miss; do for r in 0 1; do
    TL_CASE=$c TL_ROPE=$r timeout 120 python tools/attn_timeline.py > gpurun_out/tl2_${lib}_${c}_rope$r.txt 2>&1
  done; done
done
