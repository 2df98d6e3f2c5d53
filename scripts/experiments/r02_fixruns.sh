# k_fix_runs with 8 keys per thread: tree parity (presort paths) + timing
mkdir -p gpurun_out
make -s all > gpurun_out/make.log 2>&1 || { tail gpurun_out/make.log; exit 1; }
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_shards.py -x -q -p no:cacheprovider > gpurun_out/pytest_fr.log 2>&1; tail -1 gpurun_out/pytest_fr.log | cut -c1-300
bash scripts/r02_var.sh; bash scripts/r02_var.sh
