# fused tree finish: parity (tree / lists / eval, shards, whole-problem C3-C5) + A/B timing vs the unfused variant
mkdir -p gpurun_out
make -s all > gpurun_out/make.log 2>&1 || { tail gpurun_out/make.log; exit 1; }
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_shards.py tests/test_gpu_fullsize.py tests/test_gpu_nccl_shim.py -x -q -p no:cacheprovider > gpurun_out/pytest_tree.log 2>&1; tail -3 gpurun_out/pytest_tree.log | cut -c1-600
bash scripts/r02_var.sh build/var_tree__DFMM2D_FUSED_FINISH_0/libfmm2d.so
