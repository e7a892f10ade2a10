# A/B of the block-copy kernels: in-tree (TMA bulk) vs libragcache_b200_simt.so
timeout 600 python -m pytest tests/test_gpu_pool.py tests/test_gpu_kernels.py -x -q -k "copy or swap or pool" > gpurun_out/bulk_tests.txt 2>&1
for rep in 1 2; do for v in a simt; do
  if [ $v = a ]; then unset RCB_LIB_PATH; else export RCB_LIB_PATH=$PWD/paper_2404_12457_b200/libragcache_b200_$v.so; fi
  python tools/microbench.py copy swap 2>&1 | sed "s/^/$v$rep /"
done; done > gpurun_out/ab_copy.txt
