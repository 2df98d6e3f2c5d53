# round 2, call 2: NCCL-shim multi-process tests, Fig. 3 tests + full study, FP64 census.
mkdir -p gpurun_out
make -s all > gpurun_out/make.log 2>&1 || { tail gpurun_out/make.log; exit 1; }
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -o build/p2p_census tools/p2p_census.cu
timeout 900 python -m pytest tests/test_gpu_nccl_shim.py tests/test_gpu_error_study.py -q -p no:cacheprovider --durations=8 > gpurun_out/pytest_shim_err.log 2>&1; tail -15 gpurun_out/pytest_shim_err.log
./build/p2p_census > gpurun_out/p2p_census_time.json; cat gpurun_out/p2p_census_time.json
python tools/dgemm_peak.py > gpurun_out/dgemm_peak.json; cat gpurun_out/dgemm_peak.json
M=sm__sass_thread_inst_executed_op_dfma_pred_on.sum,sm__sass_thread_inst_executed_op_dadd_pred_on.sum,sm__sass_thread_inst_executed_op_dmul_pred_on.sum,smsp__inst_executed.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,gpu__time_duration.sum,smsp__thread_inst_executed.sum
timeout 300 ncu --metrics $M --csv ./build/p2p_census 1 > gpurun_out/ncu_census_libdevice.csv 2>&1
timeout 900 ncu --metrics $M --csv -k regex:"k_near|k_m2l" -c 2 python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > gpurun_out/ncu_census_c5.csv 2>&1
tail -5 gpurun_out/ncu_census_c5.csv | cut -c1-300
timeout 1500 python tools/error_study.py --out gpurun_out/error_study > gpurun_out/error_study.log 2>&1; tail -12 gpurun_out/error_study.log
