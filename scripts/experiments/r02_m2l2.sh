mkdir -p gpurun_out
make -s all > gpurun_out/make.log 2>&1 || { tail gpurun_out/make.log; exit 1; }
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "eval or expansions" > gpurun_out/pytest_m2l.log 2>&1; tail -2 gpurun_out/pytest_m2l.log | cut -c1-400
bash scripts/r02_var.sh build/var_*/libfmm2d.so
