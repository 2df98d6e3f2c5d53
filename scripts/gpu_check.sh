mkdir -p gpurun_out
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
lscpu | grep -E 'Model name|^CPU\(s\)'
./build/fp64_peak > gpurun_out/fp64_peak.json 2>&1; cat gpurun_out/fp64_peak.json
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -3 gpurun_out/smoke.log
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; tail -30 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --config C2 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c2.log 2>&1; tail -5 gpurun_out/bench_c2.log
timeout 900 python bench.py --steps 3 --warmup 3 > gpurun_out/bench_c5.log 2>&1; tail -5 gpurun_out/bench_c5.log
