# round 2 call 4: NCCL-shim multi-process tests, near-field timing experiments, bench line
mkdir -p gpurun_out
make -s all > gpurun_out/make.log 2>&1 || { tail gpurun_out/make.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_nccl_shim.py -x -q -p no:cacheprovider --durations=8 > gpurun_out/pytest_shim.log 2>&1; tail -25 gpurun_out/pytest_shim.log | cut -c1-300
bash scripts/r02_var.sh build/var_near__DFMM2D_NEAR_EXP_NOSTAGE/libfmm2d.so build/var_near__DFMM2D_NEAR_EXP_NOL2P/libfmm2d.so build/var_near__DFMM2D_NEAR_EXP_NOSTORE/libfmm2d.so build/var_near__DFMM2D_NEAR_EXP_NOSTAGE__DFMM2D_NEAR_EXP_NOL2P__DFMM2D_NEAR_EXP_NOSTORE/libfmm2d.so
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; tail -1 gpurun_out/bench.log | cut -c1-3000
