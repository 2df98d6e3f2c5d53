"""Pins for the oracle's r/R exchange (O7), the optional finest-level step:
for strongly coupled leaves of radii r < R that satisfy Criterion 1 with the roles of r
and R exchanged (r + theta R <= theta d), the larger box's sources are converted into a
local expansion of the smaller box (P2L) and the smaller box's multipole is evaluated
at the larger box's points (M2P) instead of the direct sum.

Pinned by: worked examples of the predicate (golden), its geometric meaning in exact
rationals, closed forms (P2L of a unit charge = the log series about 4; M2P of a single
charge), the identity P2L = M2L o P2M for a source at the multipole centre, truncation
within the a-priori law against the direct sum, the conversion-list audit, exactly-once
pair coverage, and the whole pass against the direct sum.
"""
import json
import math
import os
from fractions import Fraction

import numpy as np
import pytest

import workloads as W

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _nerr(a, b):
    return np.abs(a - b).max() / np.abs(b).max()


def test_predicate_worked_examples(orc):
    with open(os.path.join(GOLD, "rr_exchange_examples.json")) as f:
        cases = json.load(f)["cases"]
    for c in cases:
        cb, cc = complex(*c["cb"]), complex(*c["cc"])
        assert orc.well_separated(cb, c["rb"], cc, c["rc"], c["theta"]) == c["criterion"], c
        assert orc.rr_exchange(cb, c["rb"], cc, c["rc"], c["theta"]) == c["exchanged"], c


def test_predicate_geometric_meaning_exact():
    """r + theta R <= theta d  <=>  the smaller disc dilated by 1/theta and the larger
    disc do not overlap (r/theta + R <= d), checked in exact rationals; and it is the
    weaker of the two criteria for r < R (it holds whenever Criterion 1 does)."""
    rng = np.random.default_rng(3)
    for _ in range(2000):
        r, R = sorted(Fraction(int(v), 1000) for v in rng.integers(1, 1000, 2))
        d = Fraction(int(rng.integers(1, 4000)), 1000)
        th = Fraction(int(rng.integers(1, 999)), 1000)
        ex = r + th * R <= th * d
        assert ex == (r / th + R <= d)
        if R + th * r <= th * d:
            assert ex


def test_predicate_equal_radii_never(orc):
    rng = np.random.default_rng(4)
    for _ in range(500):
        r = float(rng.random())
        d = float(rng.random()) * 4
        assert not orc.rr_exchange(0j, r, complex(d, 0), r, 0.5)


def test_p2l_unit_charge_closed_form(orc):
    """log(z) about 4: ln 4 + sum_l (-1)^{l+1} (z-4)^l / (l 4^l)."""
    p = 17
    b = orc.p2l([0j], [1.0 + 0j], 4.0, p)
    ref = np.array([math.log(4.0)] + [(-1) ** (l + 1) / (l * 4.0 ** l) for l in range(1, p + 1)])
    assert np.abs(b - ref).max() <= 1e-15 * np.abs(ref).max()


def test_p2l_equals_m2l_of_p2m_at_centre(orc):
    rng = np.random.default_rng(5)
    for _ in range(20):
        cs = complex(*rng.normal(size=2))
        ct = cs + complex(*rng.normal(size=2)) * 3
        mm = complex(*rng.normal(size=2))
        p = int(rng.integers(3, 25))
        a = orc.p2m([cs], [mm], cs, p)
        b1 = orc.m2l(a, cs, ct, p)
        b2 = orc.p2l([cs], [mm], ct, p)
        assert np.abs(b1 - b2).max() <= 1e-13 * np.abs(b2).max()


def test_m2p_single_charge(orc):
    a = orc.p2m([1.5 + 0.5j], [1.0 + 0j], 1.5 + 0.5j, 10)
    phi, dphi = orc.m2p(a, 1.5 + 0.5j, 10, [3.5 + 0.5j])
    assert abs(phi[0] - math.log(2.0)) <= 1e-15 and abs(dphi[0] - 0.5) <= 1e-15


@pytest.mark.parametrize("theta", [0.3, 0.5, 0.7])
def test_p2l_and_m2p_truncation_within_bound(orc, theta):
    """A small disc (radius r) and a large one (radius R) at the exchanged criterion's
    boundary, r + theta R = theta d: P2L of the large box's sources evaluated in the
    small box, and M2P of the small box's multipole at the large box's points, agree
    with the direct sum within theta^{p+1}/(1-theta)^2."""
    rng = np.random.default_rng(7)
    r, R = 0.05, 0.6
    d = (r + theta * R) / theta
    cb, cc = 0j, complex(d, 0)
    zb = cb + r * np.sqrt(rng.random(40)) * np.exp(2j * np.pi * rng.random(40))
    zc = cc + R * np.sqrt(rng.random(60)) * np.exp(2j * np.pi * rng.random(60))
    mb, mc = rng.uniform(-1, 1, 40) + 0j, rng.uniform(-1, 1, 60) + 0j
    for p in (8, 17):
        bound = orc.error_bound(theta, p)
        # P2L: sources of c into a local about cb, evaluated at the points of b
        loc = orc.p2l(zc, mc, cb, p)
        f, df = orc.l2p(loc, cb, p, zb)
        fd = np.array([np.sum(mc * np.log(zi - zc)) for zi in zb])
        dfd = np.array([np.sum(mc / (zi - zc)) for zi in zb])
        assert _nerr(f.real, fd.real) <= bound and _nerr(df, dfd) <= bound
        # M2P: multipole of b evaluated at the points of c
        a = orc.p2m(zb, mb, cb, p)
        g, dg = orc.m2p(a, cb, p, zc)
        gd = np.array([np.sum(mb * np.log(zi - zb)) for zi in zc])
        dgd = np.array([np.sum(mb / (zi - zb)) for zi in zc])
        assert _nerr(g.real, gd.real) <= bound and _nerr(dg, dgd) <= bound


def _leaf_of(P, n, L):
    perm, offL = P.perm(), P.offsets(L)
    leaf_of = np.empty(n, np.int64)
    for b in range(4 ** L):
        leaf_of[perm[offL[b]:offL[b + 1]]] = b
    return leaf_of


@pytest.mark.parametrize("dist,n,L,theta", [("clusters", 3000, 4, 0.5), ("curve", 3000, 4, 0.5),
                                            ("clusters", 2000, 3, 0.3)])
def test_conversion_lists_audit_and_coverage(orc, dist, n, L, theta):
    z, _ = W.make(dist, n, seed=21)
    P = orc.plan(z, theta, L, rr_exchange=True)
    cx, cy, r = P.discs(L)
    so, si = P.list(L, "strong")
    lists = {k: P.list(L, k) for k in ("near", "p2l", "m2p")}
    nconv = 0
    for t in range(4 ** L):
        strong = si[so[t]:so[t + 1]].tolist()
        rows = {k: v[1][v[0][t]:v[0][t + 1]].tolist() for k, v in lists.items()}
        assert sorted(rows["near"] + rows["p2l"] + rows["m2p"]) == strong     # a split of the strong list
        assert t in rows["near"]                                              # self stays direct
        for s in rows["p2l"] + rows["m2p"]:
            ct, cs = complex(cx[t], cy[t]), complex(cx[s], cy[s])
            assert orc.rr_exchange(ct, r[t], cs, r[s], theta)
            assert not orc.well_separated(ct, r[t], cs, r[s], theta)
        for s in rows["p2l"]:
            assert r[t] < r[s]
            mo, mi = lists["m2p"]
            assert t in mi[mo[s]:mo[s + 1]].tolist()                          # s evaluates t's multipole
        for s in rows["m2p"]:
            assert r[s] < r[t]
        for s in rows["near"]:
            if s != t:
                assert not orc.rr_exchange(complex(cx[t], cy[t]), r[t], complex(cx[s], cy[s]), r[s], theta)
        nconv += len(rows["p2l"])
    assert nconv > 0
    # exactly-once coverage: ancestor weak pairs + near + conversions (both directions)
    leaf_of = _leaf_of(P, n, L)
    count = np.zeros((n, n), np.int32)
    for l in range(L + 1):
        anc = leaf_of >> (2 * (L - l))
        kinds = ("weak",) if l < L else ("weak", "near", "p2l", "m2p")
        for kind in kinds:
            off, idx = P.list(l, kind)
            M = np.zeros((4 ** l, 4 ** l), np.int32)
            for b in range(4 ** l):
                M[b, idx[off[b]:off[b + 1]]] += 1
            count += M[np.ix_(anc, anc)]
    np.fill_diagonal(count, 1)
    assert (count == 1).all()


def test_rr_off_keeps_the_strong_list(orc):
    z, _ = W.make("clusters", 2000, seed=22)
    P = orc.plan(z, 0.5, 3)
    so, si = P.list(3, "strong")
    no, ni = P.list(3, "near")
    assert np.array_equal(so, no) and np.array_equal(si, ni)
    assert P.list(3, "p2l")[1].size == 0 and P.list(3, "m2p")[1].size == 0


@pytest.mark.parametrize("dist,n", [("clusters", 6000), ("curve", 6000)])
def test_fmm_with_rr_exchange_within_gate(orc, dist, n):
    """The pass with the conversions against the direct sum: BASELINE's gate on Re Phi and
    the a-priori law on Phi'; against the pass without them: within the same law."""
    z, m = W.make(dist, n, seed=23)
    L = orc.nlevels(n, 35)
    phi_d, dphi_d = orc.direct(z, m)
    on = orc.plan(z, 0.5, L, rr_exchange=True)
    assert on.list(L, "p2l")[1].size > 0
    phi, dphi = on.eval(m, 17)
    phi0, dphi0 = orc.plan(z, 0.5, L).eval(m, 17)
    bound = orc.error_bound(0.5, 17)
    assert _nerr(phi.real, phi_d.real) <= 1e-6 and _nerr(dphi, dphi_d) <= bound
    assert _nerr(phi.real, phi0.real) <= bound and _nerr(dphi, dphi0) <= bound
