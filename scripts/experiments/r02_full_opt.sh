mkdir -p gpurun_out
make -s all > gpurun_out/make.log 2>&1 || { tail gpurun_out/make.log; exit 1; }
timeout 2400 python -m pytest tests/test_gpu_fullsize.py -x -q -p no:cacheprovider -k "rr_exchange or parent_merge" -s > gpurun_out/pytest_full_opt.log 2>&1; tail -30 gpurun_out/pytest_full_opt.log | cut -c1-400
