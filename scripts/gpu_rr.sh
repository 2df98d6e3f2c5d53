mkdir -p gpurun_out
make -s all > gpurun_out/make.log 2>&1 || { tail gpurun_out/make.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_shards.py -m gpu -q -x -p no:cacheprovider -k "rr or overlapped" 2>&1 | tail -2
bash scripts/gpu_cfgs.sh 2>&1 | grep "==\|rr-exchange"
