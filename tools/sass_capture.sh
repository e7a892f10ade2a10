# Warp-stall sampling per SASS instruction for the attention launches (under gpurun)
mkdir -p gpurun_out /tmp/reps
for c in "mixed step:mixed" "llama2 miss:mha"; do
  case="${c%%:*}"; tag="${c##*:}"
  MB_CASE="$case" ncu --set full --import-source on --clock-control none -k regex:prefix_prefill -s 2 -c 1 \
      -o /tmp/reps/sass_$tag python tools/microbench.py attn --ncu > /dev/null 2>&1
  ncu -i /tmp/reps/sass_$tag.ncu-rep --page source --csv --print-source sass 2>/dev/null | gzip > gpurun_out/sass_$tag.csv.gz
done
ls -la gpurun_out/sass_*
