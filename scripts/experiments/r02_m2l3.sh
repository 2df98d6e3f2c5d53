# warp-pair M2L: parity of the expansions / eval (in-tree default = pairs, MINB 4) + A/B timing
mkdir -p gpurun_out
make -s all > gpurun_out/make.log 2>&1 || { tail gpurun_out/make.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_shards.py -x -q -p no:cacheprovider > gpurun_out/pytest_m2l.log 2>&1; tail -2 gpurun_out/pytest_m2l.log | cut -c1-600
bash scripts/r02_var.sh build/var_expansions__DFMM2D_M2L2_MINB_3/libfmm2d.so build/var_expansions__DFMM2D_M2L_PAIRS_0/libfmm2d.so
