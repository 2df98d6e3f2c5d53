mkdir -p gpurun_out
make -s all > gpurun_out/make.log 2>&1 || { tail gpurun_out/make.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_shards.py -m gpu -q -x -p no:cacheprovider 2>&1 | tail -2
for R in 8 2; do FMM2D_TREE_TRACE=1 timeout 900 python tools/shard_build_model.py --ranks $R 2>&1 | tail -12; done
