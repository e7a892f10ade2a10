timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_parity_geometry.py -x -q > gpurun_out/stage_tests.txt 2>&1
bash tools/abn.sh s1 s2 a s5 > gpurun_out/ab_stage.txt 2>&1
