mkdir -p gpurun_out
bash scripts/r02_var.sh build/var_expansions__*/libfmm2d.so
