mkdir -p gpurun_out
for e in 1 0 1 0; do
FMM2D_EARLY_UPWARD=$e timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/b.log 2>&1
python -c "
import json; d=json.loads([l for l in open('gpurun_out/b.log') if l.startswith('{')][-1]); print('early=$e', round(d['ms_per_step'],2), d['phases_ms']['build_ms'])"
done
FMM2D_TREE_TRACE=1 timeout 300 python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/trace.log 2>&1; grep "fmm2d tree" gpurun_out/trace.log | tail -24
