mkdir -p gpurun_out
make -s all > gpurun_out/make.log 2>&1 || { tail gpurun_out/make.log; exit 1; }
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_shards.py tests/test_gpu_nccl_shim.py -x -q -p no:cacheprovider > gpurun_out/pytest_chk.log 2>&1; tail -1 gpurun_out/pytest_chk.log | cut -c1-300
bash scripts/r02_var.sh
