bash scripts/r02_quick.sh
FMM2D_NEAR_THREADS=128 bash scripts/r02_var.sh | sed 's/^/T128 /'
FMM2D_NEAR_THREADS=64 bash scripts/r02_var.sh | sed 's/^/T64 /'
