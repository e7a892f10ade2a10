timeout 600 python -m pytest tests/test_gpu_kernels.py -x -q -k "kv_write" > gpurun_out/kvhb_tests.txt 2>&1
MB_CASE="mi" bash tools/ab_kvw.sh a hb0 > gpurun_out/ab_kvhb.txt 2>&1
