"""Pins for the oracle's direct sum (O0) and the theta-criterion (O4 predicate).

Direct sum: P:57-60 (Eq. 1).  Pinned by the two-body closed form (golden), a
50-digit mpmath brute force on small N, and antisymmetry of the derivative.
Criterion: P:115-150.  Pinned by worked examples (golden), its geometric
meaning in exact rational arithmetic, symmetry, the
consequences (2)-(3) and monotonicity in theta.
"""
import json
import math
import os
from fractions import Fraction

import mpmath
import numpy as np
import pytest

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _load(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


def _c(a):
    return np.array([complex(x, y) for x, y in a])


def test_direct_two_body_closed_form(orc):
    g = _load("two_body.json")
    phi, dphi = orc.direct(_c(g["z"]), _c(g["m"]))
    np.testing.assert_allclose(phi, _c(g["phi"]), atol=1e-15)
    np.testing.assert_allclose(dphi, _c(g["dphi"]), atol=1e-15)


def test_direct_equal_masses_antisymmetric(orc):
    # equal masses at +-1: dPhi(+1) = 1/2 = -dPhi(-1) (S:400 analogue)
    phi, dphi = orc.direct(np.array([1.0 + 0j, -1.0 + 0j]), np.array([1.0 + 0j, 1.0 + 0j]))
    assert dphi[0] == pytest.approx(0.5) and dphi[1] == pytest.approx(-0.5)
    assert phi[0].real == pytest.approx(math.log(2.0))
    assert phi[1] == pytest.approx(complex(math.log(2.0), math.pi))   # Log(-2)


@pytest.mark.parametrize("seed", [1, 2])
def test_direct_vs_mpmath_bruteforce(orc, seed):
    rng = np.random.default_rng(seed)
    n = 9
    z = rng.random(n) + 1j * rng.random(n)
    z[3] = z[3].real + 0j        # a point with y = 0: exercises Arg near the axis
    z[4] = complex(z[4].real, z[3].imag)   # same y as z[3]: dy = +0 exactly
    m = (2 * rng.random(n) - 1) + 1j * (2 * rng.random(n) - 1)
    phi, dphi = orc.direct(z, m)
    mpmath.mp.dps = 50
    for i in range(n):
        s = mpmath.mpc(0)
        ds = mpmath.mpc(0)
        for j in range(n):
            if j == i:
                continue
            dz = mpmath.mpc(mpmath.mpf(z[i].real) - mpmath.mpf(z[j].real),
                            mpmath.mpf(z[i].imag) - mpmath.mpf(z[j].imag))
            mj = mpmath.mpc(m[j].real, m[j].imag)
            s += mj * mpmath.log(dz)
            ds += mj / dz
        assert abs(complex(s) - phi[i]) <= 1e-15 * max(1.0, abs(complex(s)))
        assert abs(complex(ds) - dphi[i]) <= 1e-15 * max(1.0, abs(complex(ds)))


def test_direct_target_subset_matches_full(orc):
    rng = np.random.default_rng(3)
    z = rng.random(300) + 1j * rng.random(300)
    m = rng.random(300) + 0j
    phi, dphi = orc.direct(z, m)
    t = np.array([0, 17, 299], np.int64)
    p2, d2 = orc.direct(z, m, targets=t)
    assert np.array_equal(p2, phi[t]) and np.array_equal(d2, dphi[t])


def test_direct_negative_zero_canonicalised(orc):
    # DESIGN R6: -0 is mapped to +0, so Arg(z_i - z_j) with equal y is +pi not -pi
    z = np.array([complex(0.0, -0.0), complex(1.0, 0.0)])
    phi, _ = orc.direct(z, np.array([1.0 + 0j, 1.0 + 0j]))
    assert phi[0].imag == pytest.approx(math.pi)


# ---------------------------------------------------------------- criterion

def test_criterion_examples(orc):
    g = _load("criterion_examples.json")
    for c in g["cases"]:
        got = orc.well_separated(complex(*c["cb"]), c["rb"], complex(*c["cc"]), c["rc"], c["theta"])
        assert got == c["well_separated"], c["why"]


def test_separation_ratios_example():
    g = _load("criterion_examples.json")["separation_ratios"]
    d = abs(complex(*g["cb"]) - complex(*g["cc"]))
    R, r = max(g["rb"], g["rc"]), min(g["rb"], g["rc"])
    assert r / (d - R) == pytest.approx(g["r_over_d_minus_R"])
    assert R / (d - r) == pytest.approx(g["R_over_d_minus_r"])
    assert (d + r + R) / (d - R) == pytest.approx(g["d_plus_r_plus_R_over_d_minus_R"])


def _rand_discs(rng, k):
    c1 = rng.uniform(-2, 2, (k, 2))
    c2 = rng.uniform(-2, 2, (k, 2))
    r1 = rng.uniform(0, 1, k)
    r2 = rng.uniform(0, 1, k)
    return c1, r1, c2, r2


def test_criterion_geometric_meaning_and_symmetry(orc):
    """well separated <=> the bigger disc dilated by 1/theta about its
    centre does not reach the other disc: R/theta + r <= d.  Checked in exact
    rational arithmetic (d^2 compared, no sqrt) away from the boundary."""
    rng = np.random.default_rng(11)
    c1, r1, c2, r2 = _rand_discs(rng, 20000)
    agree = 0
    for k in range(c1.shape[0]):
        theta = [0.3, 0.5, 0.7][k % 3]
        a, b = complex(*c1[k]), complex(*c2[k])
        got = orc.well_separated(a, r1[k], b, r2[k], theta)
        assert got == orc.well_separated(b, r2[k], a, r1[k], theta)          # P:130 symmetry
        R, r = Fraction(max(r1[k], r2[k])), Fraction(min(r1[k], r2[k]))
        th = Fraction(theta)
        dx, dy = Fraction(c1[k][0]) - Fraction(c2[k][0]), Fraction(c1[k][1]) - Fraction(c2[k][1])
        d2 = dx * dx + dy * dy
        lhs = R / th + r                                                    # dilated reach
        margin = float(abs(lhs * lhs - d2)) / max(float(d2), 1e-300)
        if margin < 1e-9:
            continue                                                        # too close to call
        assert got == (lhs * lhs <= d2)
        agree += 1
    assert agree > 19000


def test_criterion_consequences_eq2_eq3_and_monotone(orc):
    """Eq. (2)-(3), over random well-separated pairs; monotone in theta."""
    rng = np.random.default_rng(12)
    c1, r1, c2, r2 = _rand_discs(rng, 20000)
    n_ws = 0
    for k in range(c1.shape[0]):
        theta = [0.3, 0.5, 0.7][k % 3]
        a, b = complex(*c1[k]), complex(*c2[k])
        if not orc.well_separated(a, r1[k], b, r2[k], theta):
            continue
        n_ws += 1
        d = abs(a - b)
        R, r = max(r1[k], r2[k]), min(r1[k], r2[k])
        tol = 1e-12
        assert (d + r + R) / (d - R) <= 2.0 / (1.0 - theta) * (1 + tol)
        assert r / (d - R) <= R / (d - r) * (1 + tol)
        assert R / (d - r) <= theta * (1 + tol)
        assert orc.well_separated(a, r1[k], b, r2[k], min(0.99, theta + 0.1))
    assert n_ws > 1000


def test_error_bound_values(orc):
    g = _load("error_bound.json")
    for c in g["cases"]:
        assert orc.error_bound(c["theta"], c["p"]) == pytest.approx(c["bound"], rel=1e-14), c["why"]
    # ratio bound(theta, p+1)/bound(theta, p) = theta
    for p in range(0, 30):
        assert orc.error_bound(0.3, p + 1) / orc.error_bound(0.3, p) == pytest.approx(0.3)
    # theta^-2 log^-2 theta is minimised at exp(-1)
    f = lambda t: t ** -2 * math.log(t) ** -2
    t0 = g["optimal_theta"]["value"]
    assert all(f(t0) <= f(t) for t in np.linspace(0.05, 0.95, 181))
