# ncu --set full of k_near at C5: every raw metric (csv) and the source page (gz) into gpurun_out/
mkdir -p gpurun_out
CMD1="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-optional"
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base mangled -k "regex:6k_nearI" -c 1 -o /tmp/prof_near $CMD1 > gpurun_out/ncu_full_near.log 2>&1
tail -1 gpurun_out/ncu_full_near.log
ncu -i /tmp/prof_near.ncu-rep --page raw --csv > gpurun_out/raw_k_near.csv 2>/dev/null
python tools/ncu_brief.py /tmp/prof_near.ncu-rep > gpurun_out/brief_k_near.txt 2>&1
ncu -i /tmp/prof_near.ncu-rep --page source --csv --print-source sass > gpurun_out/source_k_near.csv 2>/dev/null; gzip -f gpurun_out/source_k_near.csv
cat gpurun_out/brief_k_near.txt
