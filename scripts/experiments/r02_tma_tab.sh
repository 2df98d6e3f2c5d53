# k_near tables by one TMA bulk copy: parity + A/B timing (x2)
mkdir -p gpurun_out
make -s all > gpurun_out/make.log 2>&1 || { tail gpurun_out/make.log; exit 1; }
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_shards.py -x -q -p no:cacheprovider > gpurun_out/pytest_tma.log 2>&1; tail -1 gpurun_out/pytest_tma.log | cut -c1-300
bash scripts/r02_var.sh build/var_near__DFMM2D_NEAR_TMA_TABLES_0/libfmm2d.so
bash scripts/r02_var.sh build/var_near__DFMM2D_NEAR_TMA_TABLES_0/libfmm2d.so
