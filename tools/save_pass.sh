# copy the outputs of scripts/r02_final.sh (gpurun_out/) into profiles/r02 under a version tag
# usage: bash tools/save_pass.sh v5
V=$1; G=gpurun_out; P=profiles/r02
cp $G/ncu_census_c5.csv $P/ncu_census_c5.csv && python tools/census_update.py $G/ncu_census_c5.csv
cp $G/launches.csv $P/launches_c5_$V.csv; cp $G/launches_summary.txt $P/launches_c5_${V}_summary.txt
cp $G/pytest_gpu.log $P/pytest_gpu_$V.log
for k in 6k_nearI:k_near 5k_m2lI:k_m2l 11k_partitionI:k_partition 12k_tree_local:k_tree_local 8k_finish:k_finish 5k_p2m:k_p2m; do a=${k%%:*}; b=${k##*:}; cp $G/brief_$a.txt $P/ncu_full_${b}_c5_$V.txt; done
cp $G/source_6k_nearI.csv.gz $P/ncu_source_k_near_c5_$V.csv.gz; cp $G/source_5k_m2lI.csv.gz $P/ncu_source_k_m2l_c5_$V.csv.gz
grep '^{' $G/bench.log | tail -1 > $P/bench_c5_$V.json; grep '^{' $G/bench_ref.log | tail -1 > $P/bench_ref_$V.json
python - $V <<'PY'
import json, re, sys
v = sys.argv[1]
t = open("profiles/r02/ncu_full_k_near_c5_%s.txt" % v).read()
rd = float(re.search(r"dram__bytes_read.sum\s+([\d.]+) Gbyte", t).group(1)) * 1e9
wr = float(re.search(r"dram__bytes_write.sum\s+([\d.]+) Gbyte", t).group(1)) * 1e9
tm = re.search(r"gpu__time_duration.sum\s+([\d.]+ ms)", t).group(1)
json.dump({"k_near": {"dram_bytes_per_launch": rd + wr, "dram_read": rd, "dram_write": wr, "ncu_time": tm,
                      "source": "profiles/r02/ncu_full_k_near_c5_%s.txt (ncu --set full, C5 bench command, 1 launch)" % v}},
          open("profiles/traffic.json", "w"), indent=1)
PY
