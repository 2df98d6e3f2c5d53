mkdir -p gpurun_out
timeout 900 python tools/overlap_probe.py > gpurun_out/overlap_probe.log 2>&1; tail -5 gpurun_out/overlap_probe.log
