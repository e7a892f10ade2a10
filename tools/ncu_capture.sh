#!/bin/bash
# ncu evidence for profiles/ (run under gpurun; one GPU).  Usage: tools/ncu_capture.sh <tag>
TAG=${1:-r1}
set -x
mkdir -p gpurun_out
# 1. launch list of the bench command (cold-cache, serialised: compare SHARES)
ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/${TAG}_bench_launches.csv \
    python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-ttft --no-model-step > gpurun_out/${TAG}_bench_under_ncu.log 2>&1
# 2. one attention launch of the bench step itself (warm-up step 0, layer 5)
ncu --set full --clock-control none --import-source on -k regex:prefix_prefill -s 5 -c 1 \
    -o gpurun_out/${TAG}_attn_bench python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-ttft --no-model-step > /dev/null 2>&1
# 3. full captures of each hot kernel (microbench shapes)
# (the mixed-step case only: 2 plain launches, then the fused-RoPE one is captured)
MB_CASE="mixed step" ncu --set full --clock-control none --import-source on -k regex:prefix_prefill -s 2 -c 1 \
    -o gpurun_out/${TAG}_attn_mixed python tools/microbench.py attn --ncu > /dev/null 2>&1
# MHA (G = 1, LLaMA2 shape) with fused RoPE: the third launch of the case is the RoPE one
MB_CASE="llama2 miss" ncu --set full --clock-control none --import-source on -k regex:prefix_prefill -s 2 -c 1 \
    -o gpurun_out/${TAG}_attn_mha python tools/microbench.py attn --ncu > /dev/null 2>&1
# split-only variant (decode step over a 4096-token context: HBM-bound)
MB_CASE="decode a4096" ncu --set full --clock-control none --import-source on -k regex:prefix_prefill -s 2 -c 1 \
    -o gpurun_out/${TAG}_attn_decode python tools/microbench.py attn --ncu > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:topk_scan -s 0 -c 1 \
    -o gpurun_out/${TAG}_retrieval_scan python tools/microbench.py retrieval --ncu > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:block_copy -s 0 -c 1 \
    -o gpurun_out/${TAG}_block_gather python tools/microbench.py copy --ncu > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:kv_write_rope -s 5 -c 1 \
    -o gpurun_out/${TAG}_kv_write python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-ttft --no-model-step > /dev/null 2>&1
ls -la gpurun_out
