# build_eval: upward pass concurrent with the list construction -- parity + bench timing
mkdir -p gpurun_out
make -s all > gpurun_out/make.log 2>&1 || { tail gpurun_out/make.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_shards.py -x -q -p no:cacheprovider > gpurun_out/pytest_up.log 2>&1; tail -2 gpurun_out/pytest_up.log | cut -c1-600
bash scripts/r02_var.sh
