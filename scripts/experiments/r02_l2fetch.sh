# cudaLimitMaxL2FetchGranularity 32 / 64 / 128: C5 phase times (tools/l2_fetch_probe.py)
mkdir -p gpurun_out
for g in 32 64 128; do
  timeout 600 python tools/l2_fetch_probe.py $g --steps 3 --warmup 2 --no-cpu-baseline --no-e2e --no-optional > gpurun_out/l2f_$g.log 2> gpurun_out/l2f_$g.err
  grep l2_fetch_probe gpurun_out/l2f_$g.err
  python - $g <<'PY'
import json, sys
l=[x for x in open(f"gpurun_out/l2f_{sys.argv[1]}.log") if x.startswith("{")]
if not l: print("FAILED"); sys.exit()
d=json.loads(l[-1]); ph=d["phases_ms"]
print(f"granularity {sys.argv[1]}: step {d['ms_per_step']:.2f} build {ph['build_ms']:.2f} up {ph['upward_ms']:.2f} m2l {ph['m2l_ms']:.2f} near {ph['near_ms']:.2f}")
PY
done
