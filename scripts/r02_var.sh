# time the C5 phases for the in-tree library and each variant library given as arguments
mkdir -p gpurun_out
for lib in paper_1006_2269_b200/libfmm2d.so "$@"; do
  FMM2D_LIB=$PWD/$lib timeout 600 python bench.py --steps 3 --warmup 2 --no-cpu-baseline --no-e2e --no-optional $BENCH_ARGS > gpurun_out/var.log 2>&1
  python - "$lib" <<'PY'
import json, sys
line = [l for l in open("gpurun_out/var.log") if l.startswith("{")]
if not line:
    print(sys.argv[1], "FAILED"); print(open("gpurun_out/var.log").read()[-1500:]); sys.exit()
d = json.loads(line[-1]); ph = d["phases_ms"]
import os
print(f"{sys.argv[1]:60s} {os.environ.get('BENCH_ARGS',''):10s} step {d['ms_per_step']:.2f} build {ph['build_ms']:.2f} up {ph['upward_ms']:.2f} m2l {ph['m2l_ms']:.2f} down {ph['downward_ms']:.2f} near {ph['near_ms']:.2f}")
PY
done
