mkdir -p gpurun_out
make -s all > gpurun_out/make.log 2>&1 || { tail gpurun_out/make.log; exit 1; }
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider -k "build_eval or host_pointer or reusable" 2>&1 | tail -2
timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_e2e.log 2>&1; tail -1 gpurun_out/bench_e2e.log | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']/1e6,1), 'Mpts/s', 'e2e', d['e2e'])"
