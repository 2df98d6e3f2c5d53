mkdir -p gpurun_out
make -s all > gpurun_out/make.log 2>&1 || { tail gpurun_out/make.log; exit 1; }
CMD="python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e --config C4 --rr-exchange"
for K in k_rr_m2p k_rr_p2l k_m2l_long; do
timeout 900 ncu --set full --clock-control none --kernel-name-base demangled -k "regex:$K" -c 1 -o /tmp/prof_$K $CMD > gpurun_out/ncu_$K.log 2>&1; tail -1 gpurun_out/ncu_$K.log
python tools/ncu_brief.py /tmp/prof_$K.ncu-rep > gpurun_out/brief_$K.txt 2>&1
done
