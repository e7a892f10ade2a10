timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_parity_geometry.py -x -q > gpurun_out/rope_tests.txt 2>&1
MB_CASE=llama2 bash tools/abn.sh base a > gpurun_out/ab_rope.txt 2>&1
MB_CASE=mixed bash tools/abn.sh base a >> gpurun_out/ab_rope.txt 2>&1
