timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pdl_tests.txt 2>&1
for rep in 1 2; do for v in a nopdl; do
  if [ $v = a ]; then unset RCB_LIB_PATH; else export RCB_LIB_PATH=$PWD/paper_2404_12457_b200/libragcache_b200_$v.so; fi
  timeout 600 python bench.py --no-ttft --no-cpu-baseline --no-model-step --no-hit-sweep 2>/dev/null | tail -1 | python -c "import json,sys; d=json.load(sys.stdin); print('$v$rep', d['value'], d['ms_per_step'], d['roofline']['launch_ms_mean'], d['e2e']['value'], d['clocks']['sm_mhz'])"
done; done > gpurun_out/ab_pdl.txt 2>&1
