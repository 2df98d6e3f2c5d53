mkdir -p gpurun_out
make -s all > gpurun_out/make.log 2>&1 || { tail gpurun_out/make.log; exit 1; }
for lib in paper_1006_2269_b200/libfmm2d.so $(ls build/var_*/libfmm2d.so 2>/dev/null); do
  echo "== $lib"
  FMM2D_LIB=$lib timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider -k "${TESTK:-tree}" > gpurun_out/pt_var.log 2>&1; tail -1 gpurun_out/pt_var.log
  FMM2D_LIB=$lib timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_var.log 2>&1 || { tail -5 gpurun_out/bench_var.log; continue; }
  python -c "
import json; d=json.loads(open('gpurun_out/bench_var.log').read().strip().splitlines()[-1])
print(round(d['value']/1e6,1), 'Mpts/s step', round(d['ms_per_step'],1), 'ms', {k: round(v,2) for k,v in d['phases_ms'].items()})"
done
