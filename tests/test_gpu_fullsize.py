"""GPU parity at BASELINE.json's full sizes, in the launch configuration bench.py times.

Full-size outputs cannot all be recomputed by the oracle, so:
  - C3 (1e6, clusters) and C4 (1e7, curve): tree, discs and lists bit-exact against the
    oracle's tree/list builder (cheap at these sizes), plus sampled outputs against the
    oracle's long-double direct sum;
  - C5 (1e8, the metric's workload): sampled outputs against the direct sum, and
    properties that hold at any size (perm is a bijection, leaf sizes floor/ceil(N/4^L),
    finite outputs).
The direct-sum gate is BJ's: Re Phi (real m) within 1e-6 normwise and Phi' within the
paper's a-priori law theta^{p+1}/(1-theta)^2 over the sampled targets.
"""
import numpy as np
import pytest
import torch

import workloads as W

pytestmark = pytest.mark.gpu


def _nerr(a, b):
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-300))


def _run(cfg_name, n=None):
    from paper_1006_2269_b200 import Fmm2d
    c = W.CONFIGS[cfg_name]
    z, m = W.make_config(cfg_name, n=n)
    zt = torch.from_numpy(z).cuda()
    plan = Fmm2d(zt, theta=c.theta, p=c.p, leaf_target=c.leaf_target, real_strengths=(c.strengths == "real"))
    phi, dphi = plan.eval(torch.from_numpy(m).cuda())
    torch.cuda.synchronize()
    return c, z, m, plan, phi, dphi


def _sampled_direct(orc, z, m, phi, dphi, theta, p, M, seed):
    t = W.sample_targets(len(z), M, seed=seed)
    ti = torch.from_numpy(t).cuda()
    phs = phi[ti].cpu().numpy()
    dps = dphi[ti].cpu().numpy()
    assert np.isfinite(phs).all() and np.isfinite(dps).all()
    phd, dpd = orc.direct(z, m, targets=t)
    e_phi = _nerr(phs.real, phd.real)
    e_dphi = _nerr(dps, dpd)
    assert e_phi <= 1e-6, e_phi
    assert e_dphi <= orc.error_bound(theta, p), e_dphi
    return e_phi, e_dphi


def _structure_equal(gp, op, L, levels):
    np.testing.assert_array_equal(gp.perm(), op.perm())
    for l in levels:
        np.testing.assert_array_equal(gp.offsets(l), op.offsets(l))
        for a, b in zip(gp.discs(l), op.discs(l)):
            np.testing.assert_array_equal(a, b)
        for kind in ("strong", "weak"):
            go, gi = gp.list(l, kind)
            oo, oi = op.list(l, kind)
            np.testing.assert_array_equal(go, oo)
            np.testing.assert_array_equal(gi, oi)


def test_c3_full_structure_and_sampled(orc):
    c, z, m, plan, phi, dphi = _run("C3")
    assert plan.L == orc.nlevels(len(z), c.leaf_target) == 7
    op = orc.plan(z, c.theta, plan.L)
    _structure_equal(plan, op, plan.L, range(plan.L + 1))
    _sampled_direct(orc, z, m, phi, dphi, c.theta, c.p, M=64, seed=301)


def test_c4_full_structure_and_sampled(orc):
    c, z, m, plan, phi, dphi = _run("C4")
    assert plan.L == 9
    op = orc.plan(z, c.theta, plan.L)
    _structure_equal(plan, op, plan.L, [0, 3, 6, plan.L])
    _sampled_direct(orc, z, m, phi, dphi, c.theta, c.p, M=32, seed=401)


def test_c5_full_sampled_and_properties(orc):
    c, z, m, plan, phi, dphi = _run("C5")
    n = len(z)
    assert plan.L == 11                                    # 12 levels (BJ configs[4])
    perm = plan.perm()
    assert np.array_equal(np.sort(perm), np.arange(n, dtype=np.uint32))
    sizes = np.diff(plan.offsets(plan.L))
    assert sizes.min() == n // 4 ** plan.L and sizes.max() == -(-n // 4 ** plan.L)
    assert torch.isfinite(torch.view_as_real(phi)).all() and torch.isfinite(torch.view_as_real(dphi)).all()
    _sampled_direct(orc, z, m, phi, dphi, c.theta, c.p, M=16, seed=501)
