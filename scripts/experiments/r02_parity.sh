# round 2: GPU tests (new level-1 / whole-problem tests), the one-off C5 whole-problem parity
# log, a default bench line.  Host facts first (cores / RAM decide the oracle's C5 time).
mkdir -p gpurun_out
(nproc; free -g; lscpu | grep -i "model name\|^CPU(s)\|Thread\|Socket") > gpurun_out/host.txt 2>&1
make -s all > gpurun_out/make.log 2>&1 || { tail gpurun_out/make.log; exit 1; }
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -1 gpurun_out/smoke.log
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=12 > gpurun_out/pytest_gpu.log 2>&1; tail -18 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/bench.log 2>&1; tail -1 gpurun_out/bench.log | cut -c1-400
MEM=$(awk '/MemTotal/ {print int($2/1048576)}' /proc/meminfo)
if [ "$MEM" -ge 80 ]; then
  timeout 2400 python tools/full_parity.py C5 --out gpurun_out/full_parity_C5.json > gpurun_out/full_parity_c5.log 2>&1; echo "full_parity rc=$?"
  tail -8 gpurun_out/full_parity_c5.log | cut -c1-400
else
  echo "host RAM ${MEM} GB: C5 whole-problem parity skipped"
fi
