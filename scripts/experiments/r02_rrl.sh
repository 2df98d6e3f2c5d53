# r/R list split: thread per short list -- parity (rr tests, whole-problem C3/C5 rr) + timing
mkdir -p gpurun_out
make -s all > gpurun_out/make.log 2>&1 || { tail gpurun_out/make.log; exit 1; }
timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "rr" > gpurun_out/pytest_rrl.log 2>&1; tail -1 gpurun_out/pytest_rrl.log | cut -c1-300
timeout 1200 python -m pytest tests/test_gpu_fullsize.py -x -q -p no:cacheprovider -k "rr_exchange" > gpurun_out/pytest_rrl2.log 2>&1; tail -1 gpurun_out/pytest_rrl2.log | cut -c1-300
for a in "--rr-exchange" "--rr-exchange --parent-merge" "--config C4 --rr-exchange" "--config C3 --rr-exchange"; do
BENCH_ARGS="$a" bash scripts/r02_var.sh
done
