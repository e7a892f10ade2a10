# configs[2]/[3] bench lines + LLaMA2 profiles after the MHA O-store change (under gpurun)
TAG=${1:-r2e}
mkdir -p gpurun_out/prof
OUT_DIR=gpurun_out/prof timeout 1200 python tools/measure_profiles.py llama2-7b llama2-13b > gpurun_out/${TAG}_profiles.log 2>&1
for wl in llama2-13b-10m llama2-7b-top5; do
  timeout 900 python bench.py --workload $wl --no-ttft --no-cpu-baseline > gpurun_out/${TAG}_bench_${wl}.log 2>&1
done
