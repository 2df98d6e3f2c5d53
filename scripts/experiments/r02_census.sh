mkdir -p gpurun_out
make -s all > /dev/null 2>&1
M=sm__sass_thread_inst_executed_op_dfma_pred_on.sum,sm__sass_thread_inst_executed_op_dadd_pred_on.sum,sm__sass_thread_inst_executed_op_dmul_pred_on.sum,smsp__inst_executed.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,gpu__time_duration.sum,smsp__thread_inst_executed.sum
timeout 900 ncu --metrics $M --csv --kernel-name-base demangled -k "regex:k_near<|k_m2l<" -c 2 python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e --no-optional > gpurun_out/ncu_census_c5.csv 2>&1
grep -c k_near gpurun_out/ncu_census_c5.csv
