# parity subset + C5 phase times of the in-tree library (and variant libraries given as arguments)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_error_study.py -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_quick.log 2>&1; tail -3 gpurun_out/pytest_quick.log
bash scripts/r02_var.sh "$@"
