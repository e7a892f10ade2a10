timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_parity_geometry.py tests/test_gpu_model.py -x -q > gpurun_out/mha_tests.txt 2>&1
bash tools/abn.sh base nolf a > gpurun_out/ab_mha.txt 2>&1
