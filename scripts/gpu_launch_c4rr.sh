mkdir -p gpurun_out
make -s all > gpurun_out/make.log 2>&1 || { tail gpurun_out/make.log; exit 1; }
CMD="python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e --config C4 --rr-exchange"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c4rr.csv $CMD > gpurun_out/ncu_c4rr.log 2>&1
python tools/ncu_launch_summary.py gpurun_out/launches_c4rr.csv > gpurun_out/launches_c4rr_summary.txt 2>&1; head -16 gpurun_out/launches_c4rr_summary.txt
