# M2L with L1 prefetch of the next pair's multipole: parity + A/B timing
mkdir -p gpurun_out
make -s all > gpurun_out/make.log 2>&1 || { tail gpurun_out/make.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_shards.py -x -q -p no:cacheprovider > gpurun_out/pytest_m2l.log 2>&1; tail -2 gpurun_out/pytest_m2l.log | cut -c1-600
bash scripts/r02_var.sh build/var_expansions__DFMM2D_M2L_PREFETCH_0/libfmm2d.so
