# r/R exchange effect on the non-uniform configurations (C3 clusters 1e6, C4 curve 1e7)
mkdir -p gpurun_out
make -s all > gpurun_out/make.log 2>&1 || { tail gpurun_out/make.log; exit 1; }
for C in C3 C4; do for RR in "" "--rr-exchange"; do
  timeout 900 python bench.py --config $C --steps 3 --warmup 3 --no-cpu-baseline --no-e2e $RR > gpurun_out/b.log 2>&1 || { tail -3 gpurun_out/b.log; continue; }
  tail -1 gpurun_out/b.log > gpurun_out/bench_${C}${RR}.json
  python -c "
import json; d=json.loads(open('gpurun_out/b.log').read().strip().splitlines()[-1])
print('$C', '$RR', round(d['value']/1e6,2), 'Mpts/s step', round(d['ms_per_step'],2), 'ms', {k: round(v,2) for k,v in d['phases_ms'].items()}, 'p2p', d['stats']['p2p_pairs'])"
done; done
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider > gpurun_out/pt.log 2>&1; tail -2 gpurun_out/pt.log
