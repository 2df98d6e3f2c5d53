mkdir -p gpurun_out
make -s all > gpurun_out/make.log 2>&1 || { tail gpurun_out/make.log; exit 1; }
timeout 1800 python tools/error_study.py --out gpurun_out/error_study > gpurun_out/error_study.log 2>&1; tail -8 gpurun_out/error_study.log
