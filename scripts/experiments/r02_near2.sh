# k_near timing experiments (not parity-valid variants): no L2P, leaf-order stores, no staging
mkdir -p gpurun_out
bash scripts/r02_var.sh build/var_near__*/libfmm2d.so
