# k_near occupancy variants (9 / 10 CTAs per SM by register cap)
mkdir -p gpurun_out
bash scripts/r02_var.sh build/var_near__*/libfmm2d.so
