mkdir -p gpurun_out
make -s all > gpurun_out/make.log 2>&1 || { tail gpurun_out/make.log; exit 1; }
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o build/dmma_peak tools/dmma_peak.cu && ./build/dmma_peak | tee gpurun_out/dmma_peak.json
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_shards.py -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; tail -2 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/plain.log 2>&1; tail -1 gpurun_out/plain.log | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']/1e6,1), 'Mpts/s step', round(d['ms_per_step'],1), {k: round(v,2) for k,v in d['phases_ms'].items()})"
