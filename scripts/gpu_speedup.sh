mkdir -p gpurun_out
make -s all > gpurun_out/make.log 2>&1 || { tail gpurun_out/make.log; exit 1; }
timeout 1800 python tools/speedup_study.py --out gpurun_out/speedup > gpurun_out/speedup.log 2>&1; tail -16 gpurun_out/speedup.log
