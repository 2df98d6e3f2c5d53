"""Summarise an ncu --csv launch list (gpu__time_duration.sum) by kernel: total ms, share."""
import collections
import csv
import io
import sys


def load(path):
    lines = open(path).read().splitlines()
    start = next(i for i, l in enumerate(lines) if l.startswith('"ID"'))
    return list(csv.DictReader(io.StringIO("\n".join(lines[start:]))))


def main(path, top=25):
    rows = load(path)
    agg = collections.defaultdict(lambda: [0, 0.0])
    scale = {"nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0, "second": 1e3, "ns": 1e-6, "us": 1e-3, "ms": 1.0, "s": 1e3}
    for r in rows:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        name = r["Kernel Name"]
        name = name.split("(")[0][:70]
        v = float(r["Metric Value"].replace(",", "")) * scale[r["Metric Unit"]]
        agg[name][0] += 1
        agg[name][1] += v
    tot = sum(v[1] for v in agg.values())
    print(f"{'ms':>10} {'share':>6} {'launches':>8}  kernel   (total {tot:.1f} ms, {sum(v[0] for v in agg.values())} launches)")
    for k, v in sorted(agg.items(), key=lambda x: -x[1][1])[:top]:
        print(f"{v[1]:10.2f} {100 * v[1] / tot:5.1f}% {v[0]:8d}  {k}")


if __name__ == "__main__":
    main(sys.argv[1])
