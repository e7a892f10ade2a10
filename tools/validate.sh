#!/bin/bash
# Round validation on one B200 (run under gpurun): GPU tests, smoke, bench (both arms), ncu.
# Usage: tools/validate.sh <tag> [skip-tests]
TAG=${1:-r2a}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/${TAG}_smi.txt
if [ "$2" != "skip-tests" ]; then
  timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest.log
  timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/${TAG}_smoke.log 2>&1
fi
timeout 600 python bench.py > gpurun_out/${TAG}_bench.log 2>&1
timeout 600 python bench.py --impl reference > gpurun_out/${TAG}_ref.log 2>&1
timeout 900 bash tools/ncu_capture.sh ${TAG} > gpurun_out/${TAG}_ncu.log 2>&1
PROFILES_DIR=gpurun_out python tools/ncu_summary.py ${TAG} > /dev/null 2>&1
# keep the transfer under gpurun's 64 MiB: raw pages of every capture, the reps themselves
# only for the attention launches when they fit
mkdir -p /tmp/reps
for r in gpurun_out/${TAG}_*.ncu-rep; do
  ncu -i "$r" --page raw --csv > "${r%.ncu-rep}_raw.csv" 2>/dev/null
  mv "$r" /tmp/reps/
done
for k in attn_mha attn_bench; do
  f=/tmp/reps/${TAG}_${k}.ncu-rep
  if [ -f "$f" ] && [ $(du -sm gpurun_out | cut -f1) -lt 30 ] && [ $(du -m "$f" | cut -f1) -lt 15 ]; then cp "$f" gpurun_out/; fi
done
du -sh gpurun_out
