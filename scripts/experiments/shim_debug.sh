mkdir -p gpurun_out/shim
make -s all > gpurun_out/make.log 2>&1 || { tail gpurun_out/make.log; exit 1; }
ID=$(python -c "import os;print((os.urandom(8).hex().encode()+bytes(112)).hex())")
CHILD=$(python - <<'PY'
import re
src=open('tests/test_gpu_nccl_shim.py').read()
print(re.search(r'CHILD = r"""(.*?)"""', src, re.S).group(1))
PY
)
for r in 0 1; do
  FMM2D_NCCL_LIB=$PWD/tests/ncclshim/libncclshim.so FMM2D_NCCLSHIM_DEBUG=1 FMM2D_NCCLSHIM_MB=128 timeout 120 python -c "$CHILD" $PWD C2 100000 2 $r $ID gpurun_out/shim/r$r.npz 0 0 > gpurun_out/shim/r$r.log 2>&1 &
done
wait
tail -20 gpurun_out/shim/r0.log gpurun_out/shim/r1.log
M=sm__sass_thread_inst_executed_op_dfma_pred_on.sum,sm__sass_thread_inst_executed_op_dadd_pred_on.sum,sm__sass_thread_inst_executed_op_dmul_pred_on.sum,smsp__inst_executed.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,gpu__time_duration.sum,smsp__thread_inst_executed.sum,sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active
timeout 900 ncu --metrics $M --csv -k regex:"^k_near|^k_m2l$|^k_m2l<" -c 2 python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > gpurun_out/ncu_census_c5.csv 2>&1
grep -v "^==" gpurun_out/ncu_census_c5.csv | awk -F'","' '{print $5, $13, $15}' | cut -c1-200 | tail -20
