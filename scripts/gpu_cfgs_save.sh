# C3 / C4 (with and without r/R exchange): bench lines saved under gpurun_out/
mkdir -p gpurun_out
make -s all > gpurun_out/make.log 2>&1 || { tail gpurun_out/make.log; exit 1; }
for c in C3 C4; do for rr in "" "--rr-exchange"; do
  name=bench_${c}$(echo $rr | tr -d '-')
  timeout 600 python bench.py --steps 5 --warmup 3 --config $c $rr > gpurun_out/$name.log 2>&1 || { tail -3 gpurun_out/$name.log; continue; }
  tail -1 gpurun_out/$name.log > gpurun_out/$name.json
  python -c "
import json; d=json.loads(open('gpurun_out/$name.json').read())
print('$name', round(d['value']/1e6,2), 'Mpts/s', round(d['ms_per_step'],2), 'ms', {k: round(v,2) for k,v in d['phases_ms'].items() if k!='launches'}, 'frac', round(d['roofline']['frac'],3), 'pairs', '%.3g' % d['roofline']['pairs_per_launch'], 'e2e', '%.3g' % d['e2e']['value'])"
done; done
