"""Fig. 3 study at full scale: relative error of the force
F_i = -Phi'(z_i) = sum_j -m_j / (z_i - z_j) (the paper's G) as a function of p for
theta in {0.25, 0.5, sqrt(0.5)}, for a million sources of total mass 1 in the unit
disc, (i) uniform and (ii) radial density ~ 1/r under both readings: R24 (areal density
~ 1/r, radius uniform: "disc_r") and SPEC's (radius log-uniform on [1e-8, 1]: "disc_logr"),
about 20 sources per box.  The error is measured on a seeded random sample of M = 1000 points
 against the oracle's direct sum (long double) at exactly those points;
normwise: max |F_fmm - F_dir| / max |F_dir| over the sample (reading R3).

GPU FMM through the C ABI (paper_1006_2269_b200); the oracle only for the sampled
direct sums.  Writes profiles/<round>/error_study.csv and .json (fitted slope of
log10(err) vs p over p in [6, 18] per (dist, theta); the theta^{p+1} law says log10 theta).

    python tools/error_study.py [--n 1000000] [--out profiles/r01]
"""
import argparse
import json
import math
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import oracle  # noqa: E402
import workloads as W  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=1_000_000)
    ap.add_argument("--M", type=int, default=1000)
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r02"))
    ap.add_argument("--dists", default="disc,disc_r,disc_logr")
    args = ap.parse_args()
    import torch
    from paper_1006_2269_b200 import Fmm2d
    thetas = [0.25, 0.5, math.sqrt(0.5)]
    ps = list(range(2, 31, 2))
    rows, fits = [], {}
    for dist in args.dists.split(","):
        z, m = W.make(dist, args.n, "mass", seed=W.SEED_BASE + 300)
        tg = W.sample_targets(args.n, args.M)
        _, dphi_d = oracle.direct(z, m, tg)
        F_d = -dphi_d
        zt, mt = torch.from_numpy(z).cuda(), torch.from_numpy(m).cuda()
        for th in thetas:
            errs = []
            for p in ps:
                plan = Fmm2d(zt, theta=th, p=p, leaf_target=20, real_strengths=True)
                _, dphi = plan.eval(mt, want_phi=False)
                torch.cuda.synchronize()
                F = -dphi.cpu().numpy()[tg]
                e = float(np.abs(F - F_d).max() / np.abs(F_d).max())
                if not np.isfinite(F).all():
                    e = float("nan")
                errs.append(e)
                rows.append((dist, th, p, plan.L, e, oracle.error_bound(th, p)))
                plan.close()
            sel = [(p, e) for p, e in zip(ps, errs) if 6 <= p <= 18 and np.isfinite(e) and e > 1e-14]
            slope = float(np.polyfit([q for q, _ in sel], [math.log10(e) for _, e in sel], 1)[0]) if len(sel) > 2 else None
            fits[f"{dist}/theta={th:.4f}"] = {"slope_log10_err_per_p": slope, "log10_theta": math.log10(th),
                                             "errors": dict(zip(ps, errs))}
            print(dist, round(th, 4), "slope", slope, "vs", round(math.log10(th), 4), flush=True)
    os.makedirs(args.out, exist_ok=True)
    with open(os.path.join(args.out, "error_study.csv"), "w") as f:
        f.write("dist,theta,p,levels,rel_err_force,apriori_bound\n")
        for r in rows:
            f.write(f"{r[0]},{r[1]:.6f},{r[2]},{r[3] + 1},{r[4]:.6e},{r[5]:.6e}\n")
    with open(os.path.join(args.out, "error_study.json"), "w") as f:
        json.dump({"n": args.n, "M": args.M, "leaf_target": 20, "strengths": "1/N each (total mass 1)",
                   "error": "max |F_fmm - F_dir| / max |F_dir| over the sample, F = -Phi'", "fits": fits}, f, indent=1)


if __name__ == "__main__":
    main()
