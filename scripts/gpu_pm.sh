mkdir -p gpurun_out
make -s all > gpurun_out/make.log 2>&1 || { tail gpurun_out/make.log; exit 1; }
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_shards.py -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
for A in "" "--parent-merge"; do
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e $A > gpurun_out/b.log 2>&1; tail -1 gpurun_out/b.log > gpurun_out/bench_pm$A.json; python -c "
import json; d=json.loads(open('gpurun_out/b.log').read().strip().splitlines()[-1])
print('$A', round(d['value']/1e6,1), 'Mpts/s step', round(d['ms_per_step'],2), {k: round(v,2) for k,v in d['phases_ms'].items()}, d['stats']['weak_pairs'])"
done
