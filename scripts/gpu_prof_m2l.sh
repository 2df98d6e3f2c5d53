mkdir -p gpurun_out
make -s all > gpurun_out/make.log 2>&1 || { tail gpurun_out/make.log; exit 1; }
CMD1="python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e"
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base mangled -k "regex:5k_m2lI" -c 1 -o gpurun_out/prof_m2l $CMD1 > gpurun_out/ncu_m2l.log 2>&1; tail -2 gpurun_out/ncu_m2l.log
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base mangled -k "regex:8k_finish" -c 1 -o gpurun_out/prof_finish $CMD1 > gpurun_out/ncu_fin.log 2>&1; tail -2 gpurun_out/ncu_fin.log
