mkdir -p gpurun_out
make -s all > gpurun_out/make.log 2>&1 || { tail gpurun_out/make.log; exit 1; }
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "overlap" > gpurun_out/pytest_ov.log 2>&1; tail -2 gpurun_out/pytest_ov.log | cut -c1-300
for w in 1 2 3 4 6; do
FMM2D_OVERLAP_M2L_WARPS=$w BENCH_ARGS=--overlap bash scripts/r02_var.sh
done
