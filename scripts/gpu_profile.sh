# ncu launch list of the default bench command + one full capture of the top kernels.
mkdir -p gpurun_out
CMD="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e"
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launches.log 2>&1
SMALL="python bench.py --n 4000000 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e"
$SMALL > gpurun_out/plain_small.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:'k_near|k_m2l' -s 2 -c 2 -o gpurun_out/prof_near_m2l $SMALL > gpurun_out/ncu_full.log 2>&1
tail -3 gpurun_out/ncu_launches.log gpurun_out/ncu_full.log
