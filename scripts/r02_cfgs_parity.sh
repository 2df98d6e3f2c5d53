# C3 / C4 bench lines (with and without the r/R exchange) and the one-off whole-problem parity log at C5
# with the final kernels (profiles/r02/full_parity_C5.json is rewritten from gpurun_out/)
bash scripts/gpu_cfgs_save.sh
timeout 1500 python tools/full_parity.py C5 > gpurun_out/full_parity_C5.log 2>&1; tail -5 gpurun_out/full_parity_C5.log
cp profiles/r02/full_parity_C5.json gpurun_out/full_parity_C5.json 2>/dev/null
