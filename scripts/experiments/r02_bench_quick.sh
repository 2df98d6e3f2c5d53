mkdir -p gpurun_out
make -s all > gpurun_out/make.log 2>&1 || { tail gpurun_out/make.log; exit 1; }
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench_q.log 2>&1; tail -1 gpurun_out/bench_q.log | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step']); print(json.dumps(d['optional_steps'])); print(json.dumps(d['roofline_build'])[:400]); print(d['e2e'])"
