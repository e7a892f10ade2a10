#!/bin/bash
# dynamic work fetch on (planner heuristic) vs off (RCB_DYNAMIC=0): new parity tests, bench x3
cd "$(dirname "$0")/.."
timeout 900 python -m pytest tests/test_gpu_kernels.py -x -q > gpurun_out/dyn_tests.txt 2>&1; echo "rc=$?" >> gpurun_out/dyn_tests.txt
for rep in 1 2 3; do
  for v in off on; do
    if [ $v = off ]; then export RCB_DYNAMIC=0; else unset RCB_DYNAMIC; fi
    timeout 600 python bench.py --no-ttft --no-cpu-baseline --no-hit-sweep --no-model-step 2>/dev/null | tail -1 | \
      python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$v$rep', d['value'], d['ms_per_step'], r['launch_ms_mean'], d['clocks']['sm_mhz'], d['e2e']['value'])"
  done
done > gpurun_out/dyn_bench.txt 2>&1
