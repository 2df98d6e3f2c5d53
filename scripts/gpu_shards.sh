mkdir -p gpurun_out
make -s all > gpurun_out/make.log 2>&1 || { tail gpurun_out/make.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_shards.py -m gpu -q -x -p no:cacheprovider > gpurun_out/pt.log 2>&1; tail -25 gpurun_out/pt.log
