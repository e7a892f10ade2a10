#!/bin/bash
# Final-style validation: sanitizers, GPU tests, smoke, bench (both arms), ncu captures.
TAG=${1:-r2c}
mkdir -p gpurun_out
for t in memcheck racecheck synccheck; do
  timeout 600 compute-sanitizer --tool $t python tools/sanitize_kernels.py > gpurun_out/${TAG}_sanitizer_kernels_$t.log 2>&1
done
bash tools/validate.sh $TAG
