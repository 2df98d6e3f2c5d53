mkdir -p gpurun_out
make -s all > gpurun_out/make.log 2>&1 || { tail gpurun_out/make.log; exit 1; }
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_shards.py tests/test_gpu_nccl_shim.py -x -q -p no:cacheprovider > gpurun_out/pytest_rr.log 2>&1; tail -2 gpurun_out/pytest_rr.log | cut -c1-600
