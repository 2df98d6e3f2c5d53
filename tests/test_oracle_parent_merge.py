"""Pins for the oracle's parent merge (O8): "a box weakly coupled to all
children of a parent box can often interact via the latter instead (whenever the
theta-criterion with respect to that parent is true)".  With the option on, box b of
level l >= 2 gets a cross-level entry q (level l-1) in place of q's four children when
all four are weak to b and Criterion 1 holds for (b, q); M2L then shifts q's multipole
into b's local.

Pinned by: the list audit (each cross entry replaces exactly four weak children, is well
separated, and is a strong partner of b's parent; and the merge is maximal), exactly-once
pair coverage with the cross pairs, and the pass against the direct sum.
"""
import numpy as np
import pytest

import workloads as W


def _nerr(a, b):
    return np.abs(a - b).max() / np.abs(b).max()


@pytest.mark.parametrize("dist,n,L,theta", [("uniform", 3000, 4, 0.5), ("clusters", 3000, 4, 0.5),
                                            ("curve", 2000, 3, 0.3), ("uniform", 2000, 3, 0.7)])
def test_merge_audit_and_coverage(orc, dist, n, L, theta):
    z, _ = W.make(dist, n, seed=31)
    P = orc.plan(z, theta, L, parent_merge=True)
    off_ = orc.plan(z, theta, L)
    nmerged = 0
    for l in range(1, L + 1):
        cx, cy, r = P.discs(l)
        pcx, pcy, pr = P.discs(l - 1)
        wo, wi = P.list(l, "weak")
        so, si = P.list(l, "strong")
        xo, xi = P.list(l, "xweak")
        wo0, wi0 = off_.list(l, "weak")
        so0, si0 = off_.list(l, "strong")
        np.testing.assert_array_equal(so, so0)                      # strong lists unchanged
        np.testing.assert_array_equal(si, si0)
        po, pi = P.list(l - 1, "strong")
        for b in range(4 ** l):
            cross = xi[xo[b]:xo[b + 1]].tolist()
            weak = set(wi[wo[b]:wo[b + 1]].tolist())
            weak0 = set(wi0[wo0[b]:wo0[b + 1]].tolist())
            if l < 2:
                assert not cross
            cb = complex(cx[b], cy[b])
            for q in cross:
                kids = {4 * q + k for k in range(4)}
                assert kids <= weak0 and not (kids & weak)          # replaces exactly its 4 children
                assert orc.well_separated(cb, r[b], complex(pcx[q], pcy[q]), pr[q], theta)
                assert q in pi[po[b >> 2]:po[(b >> 2) + 1]].tolist()
            assert weak | {4 * q + k for q in cross for k in range(4)} == weak0
            for q in pi[po[b >> 2]:po[(b >> 2) + 1]].tolist():    # maximal
                if {4 * q + k for k in range(4)} <= weak:
                    assert not orc.well_separated(cb, r[b], complex(pcx[q], pcy[q]), pr[q], theta)
            nmerged += len(cross)
    assert nmerged > 0
    # exactly-once coverage: weak (same level), cross (target level l, source level l-1), leaf strong
    perm, offL = P.perm(), P.offsets(L)
    leaf_of = np.empty(n, np.int64)
    for b in range(4 ** L):
        leaf_of[perm[offL[b]:offL[b + 1]]] = b
    count = np.zeros((n, n), np.int32)
    for l in range(L + 1):
        anc = leaf_of >> (2 * (L - l))
        kinds = ["weak", "xweak"] + (["strong"] if l == L else [])
        for kind in kinds:
            off, idx = P.list(l, kind)
            src_l = l - 1 if kind == "xweak" else l
            if kind == "xweak" and l == 0:
                continue
            M = np.zeros((4 ** l, 4 ** src_l), np.int32)
            for b in range(4 ** l):
                M[b, idx[off[b]:off[b + 1]]] += 1
            anc_s = leaf_of >> (2 * (L - src_l))
            count += M[np.ix_(anc, anc_s)]
    np.fill_diagonal(count, 1)
    assert (count == 1).all()


def test_merge_off_has_no_cross_lists(orc):
    z, _ = W.make("uniform", 2000, seed=32)
    P = orc.plan(z, 0.5, 3)
    for l in range(4):
        assert P.list(l, "xweak")[1].size == 0


@pytest.mark.parametrize("dist", ["uniform", "clusters"])
def test_fmm_with_parent_merge_within_gate(orc, dist):
    z, m = W.make(dist, 6000, seed=33)
    L = orc.nlevels(6000, 35)
    phi_d, dphi_d = orc.direct(z, m)
    on = orc.plan(z, 0.5, L, parent_merge=True)
    off = orc.plan(z, 0.5, L)
    pairs_on = sum(on.list(l, "weak")[1].size + on.list(l, "xweak")[1].size for l in range(L + 1))
    pairs_off = sum(off.list(l, "weak")[1].size for l in range(L + 1))
    assert pairs_on < pairs_off
    phi, dphi = on.eval(m, 17)
    phi0, dphi0 = off.eval(m, 17)
    bound = orc.error_bound(0.5, 17)
    assert _nerr(phi.real, phi_d.real) <= 1e-6 and _nerr(dphi, dphi_d) <= bound
    assert _nerr(phi.real, phi0.real) <= bound and _nerr(dphi, dphi0) <= bound
