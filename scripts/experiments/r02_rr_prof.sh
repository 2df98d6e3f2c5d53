mkdir -p gpurun_out
for c in C4 C3; do
CMD="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --rr-exchange --config $c"
timeout 600 ncu --metrics gpu__time_duration.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,sm__warps_active.avg.pct_of_peak_sustained_active,launch__grid_size,launch__registers_per_thread --clock-control none -k "regex:k_rr|k_l2l" --csv --log-file gpurun_out/rr_launches_$c.csv $CMD > gpurun_out/rr_ncu_$c.log 2>&1
done
