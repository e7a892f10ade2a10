mkdir -p gpurun_out
export RCB_LIB_PATH=$PWD/paper_2404_12457_b200/libragcache_b200_tr.so
for c in llama2_miss mistral_mixed; do for r in 0 1; do
  TL_CASE=$c TL_ROPE=$r timeout 120 python tools/attn_timeline.py > gpurun_out/tl_${c}_rope$r.txt 2>&1
done; done
unset RCB_LIB_PATH
timeout 300 python tools/microbench.py attn > gpurun_out/mb_attn_r2.txt 2>&1
timeout 400 python bench.py --no-ttft --no-cpu-baseline > gpurun_out/r2c_bench.log 2>&1
