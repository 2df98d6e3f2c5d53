"""One-off whole-problem parity run (GPU path vs the oracle) at a BASELINE config, with the
log written to profiles/r02/full_parity_<cfg>.json.  Needs a B200 (run under gpurun).

    python tools/full_parity.py C5            # N = 1e8, all 12 levels, all outputs
    python tools/full_parity.py C5 --n 10000000
"""
import argparse
import json
import os
import platform
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import workloads as W  # noqa: E402
from fullparity import compare  # noqa: E402


def host_info():
    cpu = ""
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                cpu = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    mem = 0
    try:
        for line in open("/proc/meminfo"):
            if line.startswith("MemTotal"):
                mem = int(line.split()[1]) // (1024 * 1024)
    except OSError:
        pass
    return {"cpu": cpu, "cores": os.cpu_count(), "mem_gb": mem, "host": platform.node()}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("cfg")
    ap.add_argument("--n", type=int, default=None)
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    import oracle
    c = W.CONFIGS[a.cfg]
    z, m = W.make_config(a.cfg, n=a.n)
    L = oracle.nlevels(len(z), c.leaf_target)
    t0 = time.time()
    res = compare(z, m, c.theta, c.p, L, real=(c.strengths == "real"),
                  log=lambda s: print(f"[{time.time() - t0:7.1f}s] {s}", flush=True))
    res.update({"cfg": a.cfg, "recipe": c.dist, "seed": W.SEED_BASE + list(W.CONFIGS).index(a.cfg),
                "host": host_info(), "wall_s": time.time() - t0,
                "git": subprocess.run(["git", "rev-parse", "--short", "HEAD"], cwd=ROOT, capture_output=True,
                                      text=True).stdout.strip() or None,
                "bar": "perm/offsets/discs/strong/weak of every level bit-exact; Phi, Phi' normwise and "
                       "pointwise (floor 1e-3 max|ref|) <= 1e-12 over all N"})
    ok = all(res[k]["norm"] <= 1e-12 and res[k]["point"] <= 1e-12 for k in ("phi", "dphi"))
    res["pass"] = bool(ok)
    out = a.out or os.path.join(ROOT, "profiles", "r02", f"full_parity_{a.cfg}{'' if a.n is None else '_' + str(a.n)}.json")
    os.makedirs(os.path.dirname(out), exist_ok=True)
    json.dump(res, open(out, "w"), indent=1)
    print(json.dumps(res))
    sys.exit(0 if ok else 1)


if __name__ == "__main__":
    main()
