"""Fig. 4 analogue: speedup of the asymmetric adaptive FMM
(median splits) over the uniform midpoint tree (FMM2D_MIDPOINT, same engine) as the
sources cluster.  N = 200,000 points, harmonic (log) potential, "normal" (N(0, sigma^2)
per coordinate) and "layer" (x uniform, y ~ N(0, sigma^2)) distributions forced by
rejection into the unit square; theta = 0.5, p = 20 (the paper's ~1e-6 tolerance), ~20
sources per box, both trees of the same depth.  Time = build + eval on one B200 (median
of 5 after 2 warm-ups, CUDA events).  The paper's absolute "<~15 %" refers to a separate
optimised uniform code (absent), so only the crossover versus sigma is comparable.

    python tools/speedup_study.py [--out profiles/r01]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import workloads as W  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=200_000)
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r01"))
    args = ap.parse_args()
    import torch
    from paper_1006_2269_b200 import Fmm2d
    stream = torch.cuda.current_stream()
    rows = []
    for kind in ("normal", "layer"):
        for sig in (1.0, 0.3, 0.1, 0.03, 0.01, 0.003, 0.001):
            z, m = W.make(f"{kind}:{sig}", args.n, "real", seed=W.SEED_BASE + 500)
            zt, mt = torch.from_numpy(z).cuda(), torch.from_numpy(m).cuda()
            times = {}
            stats = {}
            for pol in ("median", "midpoint"):
                ts = []
                for it in range(7):
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    e0.record(stream)
                    plan = Fmm2d(zt, theta=0.5, p=20, leaf_target=20, real_strengths=True,
                                 midpoint=(pol == "midpoint"))
                    plan.eval(mt)
                    e1.record(stream)
                    torch.cuda.synchronize()
                    if it >= 2:
                        ts.append(e0.elapsed_time(e1))
                    if it == 6:
                        st = plan.stats()
                        stats[pol] = {"p2p_pairs": st["p2p_pairs"], "weak_pairs": st["weak_pairs"],
                                      "max_leaf": st["max_leaf"], "levels": st["L"] + 1}
                    plan.close()
                times[pol] = float(np.median(ts))
            row = {"dist": kind, "sigma": sig, "t_median_ms": times["median"], "t_midpoint_ms": times["midpoint"],
                   "speedup": times["midpoint"] / times["median"], **{f"{k}_{p}": v for p, d in stats.items()
                                                                       for k, v in d.items()}}
            rows.append(row)
            print(kind, sig, round(times["median"], 3), round(times["midpoint"], 3), "speedup",
                  round(row["speedup"], 2), flush=True)
    os.makedirs(args.out, exist_ok=True)
    with open(os.path.join(args.out, "speedup_study.json"), "w") as f:
        json.dump({"n": args.n, "theta": 0.5, "p": 20, "leaf_target": 20, "rows": rows}, f, indent=1)


if __name__ == "__main__":
    main()
