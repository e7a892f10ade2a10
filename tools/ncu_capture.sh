#!/bin/bash
# ncu evidence for profiles/ (run under gpurun; one GPU).
set -x
mkdir -p gpurun_out
# 1. launch list of the bench command (cold-cache, serialised: compare SHARES)
ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/r1_bench_launches.csv \
    python bench.py --steps 2 --warmup 1 --cache-warm-steps 40 --no-cpu-baseline > gpurun_out/r1_bench_under_ncu.log 2>&1
# 2. full captures of each hot kernel (one launch each)
ncu --set full --clock-control none --import-source on -k regex:prefix_prefill -s 4 -c 1 \
    -o gpurun_out/r1_attn_mixed python tools/microbench.py attn --ncu > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:topk_scan -s 0 -c 1 \
    -o gpurun_out/r1_retrieval_scan python tools/microbench.py retrieval --ncu > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:block_copy -s 0 -c 1 \
    -o gpurun_out/r1_block_gather python tools/microbench.py copy --ncu > /dev/null 2>&1
ls -la gpurun_out
