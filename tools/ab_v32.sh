timeout 600 python -m pytest tests/test_gpu_kernels.py -x -q -k "kv_write" > gpurun_out/v32_tests.txt 2>&1
MB_CASE="mi" bash tools/ab_kvw.sh a v16 > gpurun_out/ab_v32.txt 2>&1
