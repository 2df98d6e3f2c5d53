mkdir -p gpurun_out
CMD="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e"
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launches.log 2>&1
SMALL="python bench.py --n 4000000 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e"
$SMALL > gpurun_out/plain_small.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:'k_near|k_m2l' -s 2 -c 2 \
    --metrics sm__sass_thread_inst_executed_op_dfma_pred_on.sum,sm__sass_thread_inst_executed_op_dmul_pred_on.sum,sm__sass_thread_inst_executed_op_dadd_pred_on.sum \
    -o gpurun_out/prof3 $SMALL > gpurun_out/ncu_full.log 2>&1
tail -1 gpurun_out/ncu_full.log
