mkdir -p gpurun_out
SMALL="python bench.py --n 4000000 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e"
$SMALL > gpurun_out/plain_small.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:'k_near' -s 2 -c 2 \
    --metrics sm__sass_thread_inst_executed_op_dfma_pred_on.sum,sm__sass_thread_inst_executed_op_dmul_pred_on.sum,sm__sass_thread_inst_executed_op_dadd_pred_on.sum \
    -o gpurun_out/prof_sym $SMALL > gpurun_out/ncu_full.log 2>&1
tail -1 gpurun_out/ncu_full.log
