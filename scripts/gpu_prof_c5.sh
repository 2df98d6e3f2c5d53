# C5 (bench workload): launch list of the default bench command + one full ncu capture
# of the top kernels (k_near, k_m2l, k_partition) at the bench size (for roofline.traffic).
mkdir -p gpurun_out
make -s all > gpurun_out/make.log 2>&1 || { tail gpurun_out/make.log; exit 1; }
CMD="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e"
timeout 600 $CMD > gpurun_out/plain.log 2>&1; tail -1 gpurun_out/plain.log | cut -c1-400
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launches.log 2>&1
python tools/ncu_launch_summary.py gpurun_out/launches.csv > gpurun_out/launches_summary.txt 2>&1; head -20 gpurun_out/launches_summary.txt
CMD1="python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k_near|k_m2l|k_partition' -c 3 -o gpurun_out/prof_c5 $CMD1 > gpurun_out/ncu_full.log 2>&1
tail -3 gpurun_out/ncu_full.log
