# P2M software pipeline: parity + A/B timing (x2)
mkdir -p gpurun_out
make -s all > gpurun_out/make.log 2>&1 || { tail gpurun_out/make.log; exit 1; }
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_shards.py -x -q -p no:cacheprovider > gpurun_out/pytest_p2m.log 2>&1; tail -2 gpurun_out/pytest_p2m.log | cut -c1-600
bash scripts/r02_var.sh build/var_expansions__DFMM2D_P2M_PIPE_0/libfmm2d.so
bash scripts/r02_var.sh build/var_expansions__DFMM2D_P2M_PIPE_0/libfmm2d.so
