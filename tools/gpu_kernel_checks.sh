timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_parity_geometry.py tests/test_gpu_model.py -x -q > gpurun_out/o16_tests.txt 2>&1
timeout 600 compute-sanitizer --tool racecheck python tools/sanitize_kernels.py > gpurun_out/o16_racecheck.txt 2>&1
timeout 600 compute-sanitizer --tool synccheck python tools/sanitize_kernels.py > gpurun_out/o16_synccheck.txt 2>&1
