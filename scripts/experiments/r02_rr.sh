# r/R exchange kernels, warp per leaf: parity (rr tests) + A/B timing at C5 / C4 / C3 with --rr-exchange
mkdir -p gpurun_out
make -s all > gpurun_out/make.log 2>&1 || { tail gpurun_out/make.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "rr" > gpurun_out/pytest_rr.log 2>&1; tail -2 gpurun_out/pytest_rr.log | cut -c1-600
for a in "--rr-exchange" "--config C4 --rr-exchange" "--config C3 --rr-exchange"; do
BENCH_ARGS="$a" bash scripts/r02_var.sh build/var_rr__DFMM2D_RR_WARP_0/libfmm2d.so
done
