# C3 / C4 (with and without r/R exchange) for the in-tree library and every build/var_* variant
mkdir -p gpurun_out
make -s all > gpurun_out/make.log 2>&1 || { tail gpurun_out/make.log; exit 1; }
for lib in paper_1006_2269_b200/libfmm2d.so $(ls build/var_*/libfmm2d.so 2>/dev/null); do
  echo "== $lib"
  for c in "--config C3" "--config C3 --rr-exchange" "--config C4" "--config C4 --rr-exchange"; do
    FMM2D_LIB=$lib timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e $c > gpurun_out/bench_cfg.log 2>&1 || { tail -3 gpurun_out/bench_cfg.log; continue; }
    python -c "
import json; d=json.loads(open('gpurun_out/bench_cfg.log').read().strip().splitlines()[-1])
print('$c', round(d['value']/1e6,2), 'Mpts/s', round(d['ms_per_step'],2), 'ms', {k: round(v,2) for k,v in d['phases_ms'].items() if k!='launches'}, 'frac', round(d['roofline']['frac'],3))"
  done
done
