# early L2P in k_near: parity + A/B timing
mkdir -p gpurun_out
make -s all > gpurun_out/make.log 2>&1 || { tail gpurun_out/make.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider > gpurun_out/pytest_near.log 2>&1; tail -2 gpurun_out/pytest_near.log | cut -c1-600
bash scripts/r02_var.sh build/var_near__DFMM2D_NEAR_EARLY_L2P_0/libfmm2d.so
