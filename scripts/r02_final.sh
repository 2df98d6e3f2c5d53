# Round-2 measurement pass: smoke, every GPU test (whole-problem parity at C3/C4/C5 included),
# default bench (CPU baseline + e2e), reference arm, ncu launch list of the bench command,
# ncu --set full of the top kernels at C5.  Outputs under gpurun_out/ (summaries copied to profiles/r02).
mkdir -p gpurun_out
make -s all > gpurun_out/make.log 2>&1 || { tail gpurun_out/make.log; exit 1; }
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -1 gpurun_out/smoke.log
[ -z "$SKIP_TESTS" ] && timeout 2700 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=10 > gpurun_out/pytest_gpu.log 2>&1; tail -16 gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; tail -1 gpurun_out/bench.log | cut -c1-300
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.log 2>&1; tail -1 gpurun_out/bench_ref.log | cut -c1-300
CMD1="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-optional"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD1 > gpurun_out/ncu_launches.log 2>&1
python tools/ncu_launch_summary.py gpurun_out/launches.csv > gpurun_out/launches_summary.txt 2>&1; head -14 gpurun_out/launches_summary.txt
for K in 6k_nearI 5k_m2lI 11k_partitionI 12k_tree_local 8k_finish 5k_p2m; do
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base mangled -k "regex:$K" -c 1 -o /tmp/prof_$K $CMD1 > gpurun_out/ncu_full_$K.log 2>&1
tail -1 gpurun_out/ncu_full_$K.log
python tools/ncu_brief.py /tmp/prof_$K.ncu-rep > gpurun_out/brief_$K.txt 2>&1
ncu -i /tmp/prof_$K.ncu-rep --page source --csv --print-source sass > gpurun_out/source_$K.csv 2>/dev/null; gzip -f gpurun_out/source_$K.csv
done
# FP64 census of k_near / k_m2l (executed DFMA/DADD/DMUL per pair, FP64 pipe) for profiles/r02/fp64_census.json
M=sm__sass_thread_inst_executed_op_dfma_pred_on.sum,sm__sass_thread_inst_executed_op_dadd_pred_on.sum,sm__sass_thread_inst_executed_op_dmul_pred_on.sum,smsp__inst_executed.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,gpu__time_duration.sum,smsp__thread_inst_executed.sum
timeout 900 ncu --metrics $M --csv --kernel-name-base demangled -k "regex:k_near<|k_m2l<" -c 2 python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e --no-optional > gpurun_out/ncu_census_c5.csv 2>&1
