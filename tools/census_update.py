"""Recompute the k_near / k_m2l entries of profiles/r02/fp64_census.json from an ncu census
capture of the C5 bench command (executed FP64 instructions per ordered P2P / M2L pair and the
FP64-pipe utilisation).  usage: python tools/census_update.py gpurun_out/ncu_census_c5.csv"""
import csv
import io
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PAIRS = {"k_near": 26222201312.0, "k_m2l": 201012410.0}      # C5 (bench stats: p2p_pairs, weak_pairs)
lines = open(sys.argv[1]).read().splitlines()
i = [k for k, l in enumerate(lines) if l.startswith('"ID"')][0]
rows = list(csv.DictReader(io.StringIO("\n".join(lines[i:]))))
by = {}
for r in rows:
    name = r["Kernel Name"]
    key = "k_near" if "k_near<" in name else ("k_m2l" if "k_m2l<" in name else None)
    if key is None or key in by and r["Metric Name"] in by[key]:
        continue
    by.setdefault(key, {})[r["Metric Name"]] = float(r["Metric Value"].replace(",", ""))
path = os.path.join(ROOT, "profiles", "r02", "fp64_census.json")
cen = json.load(open(path))
for key, m in by.items():
    n = PAIRS[key]
    dfma = m["sm__sass_thread_inst_executed_op_dfma_pred_on.sum"] / n
    dadd = m["sm__sass_thread_inst_executed_op_dadd_pred_on.sum"] / n
    dmul = m["sm__sass_thread_inst_executed_op_dmul_pred_on.sum"] / n
    e = cen.setdefault(key, {})
    e.update({"pairs": n, "dfma_per_pair": dfma, "dadd_per_pair": dadd, "dmul_per_pair": dmul,
              "flops_per_pair": 2 * dfma + dadd + dmul, "fp64_inst_per_pair": dfma + dadd + dmul,
              "thread_inst_per_pair": m["smsp__thread_inst_executed.sum"] / n,
              "fp64_pipe_pct": m["sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"],
              "source": "profiles/r02/ncu_census_c5.csv (C5 bench command, one launch)"})
    if key == "k_m2l":
        e["flops_per_pair"] = round(e["flops_per_pair"])
    print(key, json.dumps({k: e[k] for k in ("flops_per_pair", "fp64_inst_per_pair", "thread_inst_per_pair",
                                             "fp64_pipe_pct")}))
json.dump(cen, open(path, "w"), indent=1)
