mkdir -p gpurun_out
make -s all > gpurun_out/make.log 2>&1 || { tail gpurun_out/make.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_shards.py -x -q -p no:cacheprovider > gpurun_out/pytest_m2l.log 2>&1; tail -3 gpurun_out/pytest_m2l.log | cut -c1-400
bash scripts/r02_var.sh build/var_expansions__DFMM2D_M2L_V2_0/libfmm2d.so build/var_expansions__DFMM2D_M2L_CS2_34/libfmm2d.so build/var_expansions__DFMM2D_M2L_CS2_36/libfmm2d.so build/var_expansions__DFMM2D_M2L_CS2_40/libfmm2d.so
