# bench lines of the other configurations and the optional steps (saved under gpurun_out/)
mkdir -p gpurun_out
make -s all > gpurun_out/make.log 2>&1 || { tail gpurun_out/make.log; exit 1; }
run() {  # name, args
  timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline $2 > gpurun_out/$1.log 2>&1 || { echo "$1 FAILED"; tail -3 gpurun_out/$1.log; return; }
  tail -1 gpurun_out/$1.log > gpurun_out/$1.json
  python -c "
import json; d=json.loads(open('gpurun_out/$1.json').read())
print('$1', round(d['value']/1e6,2), 'Mpts/s', round(d['ms_per_step'],2), 'ms', {k: round(v,2) for k,v in d['phases_ms'].items() if k!='launches'}, 'frac', round(d['roofline']['frac'],3), 'pairs', '%.3g' % d['roofline']['pairs_per_launch'], 'e2e', '%.3g' % d['e2e']['value'])"
}
run bench_c5_rr "--rr-exchange"
run bench_c5_pm "--parent-merge"
run bench_c5_rr_pm "--rr-exchange --parent-merge"
for c in C3 C4; do run bench_${c} "--config $c"; run bench_${c}_rr "--config $c --rr-exchange"; done
