RCB_LIB_PATH=$PWD/paper_2404_12457_b200/libragcache_b200_ms.so timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_parity_geometry.py -x -q > gpurun_out/ms_tests.txt 2>&1
MB_CASE=llama2 bash tools/abn.sh a ms > gpurun_out/ab_ms.txt 2>&1
