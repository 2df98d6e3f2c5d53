# ncu --set full of k_m2l at C5: raw metrics (csv) and the source page (gz) into gpurun_out/
mkdir -p gpurun_out
CMD1="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-optional"
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base mangled -k "regex:5k_m2lI" -c 1 -o /tmp/prof_m2l $CMD1 > gpurun_out/ncu_full_m2l.log 2>&1
tail -1 gpurun_out/ncu_full_m2l.log
ncu -i /tmp/prof_m2l.ncu-rep --page raw --csv > gpurun_out/raw_k_m2l.csv 2>/dev/null
python tools/ncu_brief.py /tmp/prof_m2l.ncu-rep > gpurun_out/brief_k_m2l.txt 2>&1
ncu -i /tmp/prof_m2l.ncu-rep --page source --csv --print-source sass > gpurun_out/source_k_m2l.csv 2>/dev/null; gzip -f gpurun_out/source_k_m2l.csv
cat gpurun_out/brief_k_m2l.txt
