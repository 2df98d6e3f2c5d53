"""Fig. 3's claims pinned on the GPU path at reduced N (the full-scale study is
tools/error_study.py, profiles/r02/error_study.*): for sources of total mass 1 in the unit
disc, the relative force error (F = -Phi', the paper's G) decays geometrically in p at
least as fast as the theta^{p+1} law -- fitted slope of log10(err) over p in [6, 18] at most
log10(theta) + 0.12 -- and is strictly ordered in theta at every p."""
import math

import numpy as np
import pytest
import torch

import workloads as W

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("dist", ["disc", "disc_r", "disc_logr"])
def test_error_decay_slope_and_theta_order(orc, dist):
    from paper_1006_2269_b200 import Fmm2d
    n, M = 100_000, 300
    z, m = W.make(dist, n, "mass", seed=W.SEED_BASE + 310)
    tg = W.sample_targets(n, M, seed=311)
    _, dd = orc.direct(z, m, tg)
    zt, mt = torch.from_numpy(z).cuda(), torch.from_numpy(m).cuda()
    ps = list(range(6, 19, 2))
    errs = {}
    for th in (0.25, 0.5, math.sqrt(0.5)):
        errs[th] = []
        for p in ps:
            plan = Fmm2d(zt, theta=th, p=p, leaf_target=20, real_strengths=True)
            _, d = plan.eval(mt, want_phi=False)
            torch.cuda.synchronize()
            d = d.cpu().numpy()[tg]
            assert np.isfinite(d).all()
            errs[th].append(float(np.abs(d - dd).max() / np.abs(dd).max()))
            plan.close()
    for th, e in errs.items():
        sel = [(p, v) for p, v in zip(ps, e) if v > 1e-14]
        slope = np.polyfit([p for p, _ in sel], [math.log10(v) for _, v in sel], 1)[0]
        assert slope <= math.log10(th) + 0.12, (dist, th, slope, e)
    for k in range(len(ps)):
        if errs[0.25][k] > 1e-14:
            assert errs[0.25][k] < errs[0.5][k] < errs[math.sqrt(0.5)][k], (dist, ps[k])
