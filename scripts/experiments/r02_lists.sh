# connectivity: thread per box for short parent lists -- parity (structure tests, shards, whole C3/C4/C5-1e7 incl. merge) + A/B timing
mkdir -p gpurun_out
make -s all > gpurun_out/make.log 2>&1 || { tail gpurun_out/make.log; exit 1; }
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_shards.py -x -q -p no:cacheprovider > gpurun_out/pytest_lists.log 2>&1; tail -1 gpurun_out/pytest_lists.log | cut -c1-300
FMM2D_SKIP_FULL_C5=1 timeout 1800 python -m pytest tests/test_gpu_fullsize.py -x -q -p no:cacheprovider > gpurun_out/pytest_lists2.log 2>&1; tail -1 gpurun_out/pytest_lists2.log | cut -c1-300
bash scripts/r02_var.sh build/var_lists__DFMM2D_LISTS_THREAD_0/libfmm2d.so
BENCH_ARGS="--parent-merge" bash scripts/r02_var.sh build/var_lists__DFMM2D_LISTS_THREAD_0/libfmm2d.so
