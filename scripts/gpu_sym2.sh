mkdir -p gpurun_out
make -s all > gpurun_out/make.log 2>&1 || { tail gpurun_out/make.log; exit 1; }
for A in "" "--symmetric-p2p"; do
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e $A > gpurun_out/b.log 2>&1; tail -3 gpurun_out/b.log | cut -c1-200; python -c "
import json; d=json.loads(open('gpurun_out/b.log').read().strip().splitlines()[-1])
print('$A', round(d['value']/1e6,1), 'Mpts/s step', round(d['ms_per_step'],2), {k: round(v,2) for k,v in d['phases_ms'].items()})"
done
