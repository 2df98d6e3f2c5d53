# phase trace of the C5 build (FMM2D_TREE_TRACE=1: CUDA-event times per build phase on stderr)
mkdir -p gpurun_out
FMM2D_TREE_TRACE=1 timeout 600 python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-optional > gpurun_out/tree_trace.log 2>&1
grep -i -E "trace|phase|ms" gpurun_out/tree_trace.log | tail -60
