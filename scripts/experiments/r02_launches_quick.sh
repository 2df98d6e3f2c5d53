mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_q.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-optional > gpurun_out/ncu_q.log 2>&1
python tools/ncu_launch_summary.py gpurun_out/launches_q.csv | head -8
