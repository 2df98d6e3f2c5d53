mkdir -p gpurun_out
make -s all > gpurun_out/make.log 2>&1 || { tail gpurun_out/make.log; exit 1; }
export FMM2D_SKIP_FULL_C5=1
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider --durations=5 > gpurun_out/pytest_all.log 2>&1; tail -12 gpurun_out/pytest_all.log | cut -c1-600
timeout 600 python bench.py --steps 3 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/bench.log 2>&1; tail -1 gpurun_out/bench.log | cut -c1-300
python tools/shard_build_model.py > gpurun_out/shard_model.log 2>&1; tail -5 gpurun_out/shard_model.log
python tools/shard_memory.py > gpurun_out/shard_memory.json 2> gpurun_out/shard_memory.err; cat gpurun_out/shard_memory.json; tail -3 gpurun_out/shard_memory.err
