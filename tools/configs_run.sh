#!/bin/bash
# Per-config bench lines + the timed configs[3]/[4] runs (under gpurun, one GPU).
TAG=${1:-r2b}
mkdir -p gpurun_out
timeout 400 python bench.py --no-ttft --no-cpu-baseline > gpurun_out/${TAG}_bench_e2e.log 2>&1
for wl in llama2-7b-top5 llama2-13b-10m mixtral-poisson; do
  timeout 900 python bench.py --workload $wl --no-ttft --no-cpu-baseline > gpurun_out/${TAG}_bench_${wl}.log 2>&1
done
OUT_DIR=gpurun_out timeout 2400 python tools/configs_timed.py 3 4 > gpurun_out/${TAG}_configs_timed.log 2>&1
