# k_partition variants: two-pass (count, scan, scatter) and 512-thread tiles -- tree parity + timing
mkdir -p gpurun_out
for lib in build/var_tree__*/libfmm2d.so; do
  FMM2D_LIB=$PWD/$lib timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "tree" > gpurun_out/pytest_part.log 2>&1; echo "$lib $(tail -1 gpurun_out/pytest_part.log | cut -c1-200)"
done
bash scripts/r02_var.sh build/var_tree__*/libfmm2d.so
