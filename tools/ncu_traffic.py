"""Write profiles/traffic.json: dram__bytes_read.sum + dram__bytes_write.sum per launch of
the bench's dominant kernel, from one `ncu --set full` capture (bench.py reads it into
roofline.traffic).
    python tools/ncu_traffic.py <report.ncu-rep> <kernel> <source-label>"""
import csv
import io
import json
import os
import subprocess
import sys

UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}


def main(rep, kernel, label):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    tot = 0.0
    for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
        i = hdr.index(k)
        tot += float(vals[i].replace(",", "")) * UNIT[units[i]]
    t = hdr.index("gpu__time_duration.sum")
    out = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles", "traffic.json")
    d = json.load(open(out)) if os.path.exists(out) else {}
    d[kernel] = {"dram_bytes_per_launch": tot, "ncu_time": vals[t] + " " + units[t], "source": label}
    json.dump(d, open(out, "w"), indent=1)
    print(kernel, tot)


if __name__ == "__main__":
    main(*sys.argv[1:4])
