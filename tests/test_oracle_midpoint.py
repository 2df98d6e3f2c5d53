"""Pins for the oracle's midpoint split policy (O9; Fig. 2 "standard midpoint adaptivity",
the uniform baseline of Fig. 4; reading DESIGN R26): the bounding
square subdivided at geometric midpoints to a uniform depth, empty boxes allowed.

Pinned by: equality with the median tree on an aligned lattice (both are the uniform
quadtree there), containment of every point in its geometric cell (brute force), the box
sizes as brute-force cell counts at every level, exactly-once pair coverage with empty
boxes, and the pass against the direct sum.
"""
import numpy as np
import pytest

import workloads as W


def _nerr(a, b):
    return np.abs(a - b).max() / np.abs(b).max()


def test_lattice_equals_median_tree(orc):
    """On a (K 2^L)^2 lattice the median splits fall between columns, exactly at the
    geometric midpoints: both policies give the same boxes and discs."""
    z = W.lattice(4, 3, h=1.0, shuffle_seed=3)
    a = orc.plan(z, 0.5, 3, midpoint=True)
    b = orc.plan(z, 0.5, 3)
    for l in range(4):
        np.testing.assert_array_equal(a.offsets(l), b.offsets(l))
        for u, v in zip(a.discs(l), b.discs(l)):
            np.testing.assert_array_equal(u, v)
        pa, pb = a.perm(), b.perm()
        off = a.offsets(l)
        for k in range(4 ** l):                   # same sets (in-leaf order may differ)
            assert set(pa[off[k]:off[k + 1]]) == set(pb[off[k]:off[k + 1]])
        for kind in ("strong", "weak"):
            np.testing.assert_array_equal(a.list(l, kind)[1], b.list(l, kind)[1])


@pytest.mark.parametrize("dist,n,L", [("clusters", 3000, 4), ("curve", 2000, 4), ("uniform", 1000, 3)])
def test_cells_containment_and_counts(orc, dist, n, L):
    z, _ = W.make(dist, n, seed=41)
    P = orc.plan(z, 0.5, L, midpoint=True)
    x, y = z.real, z.imag
    x0, y0 = x.min(), y.min()
    side = max(x.max() - x0, y.max() - y0)
    perm = P.perm()
    for l in range(L + 1):
        off = P.offsets(l)
        cx, cy, r = P.discs(l)
        h = side / 2 ** l
        for b in range(4 ** l):
            ix = iy = 0
            for j in range(l):                    # decode the child digits (x-high first)
                q = (b >> (2 * (l - 1 - j))) & 3
                ix = 2 * ix + (q >> 1)
                iy = 2 * iy + (q & 1)
            pts = perm[off[b]:off[b + 1]]
            inside = ((x >= x0 + ix * h - 1e-12) & (x <= x0 + (ix + 1) * h + 1e-12) &
                      (y >= y0 + iy * h - 1e-12) & (y <= y0 + (iy + 1) * h + 1e-12))
            assert inside[pts].all()
            if off[b + 1] == off[b]:
                assert r[b] == -1.0
            else:
                assert r[b] >= 0.0
        assert off[-1] == n
    if dist != "uniform":
        assert any((np.diff(P.offsets(L)) == 0))  # clustered / curve data leave empty leaves


@pytest.mark.parametrize("dist", ["clusters", "curve"])
def test_coverage_with_empty_boxes(orc, dist):
    n, L = 1500, 4
    z, _ = W.make(dist, n, seed=42)
    P = orc.plan(z, 0.5, L, midpoint=True)
    perm, offL = P.perm(), P.offsets(L)
    leaf_of = np.empty(n, np.int64)
    for b in range(4 ** L):
        leaf_of[perm[offL[b]:offL[b + 1]]] = b
    count = np.zeros((n, n), np.int32)
    for l in range(L + 1):
        anc = leaf_of >> (2 * (L - l))
        for kind in (("weak",) if l < L else ("weak", "strong")):
            off, idx = P.list(l, kind)
            M = np.zeros((4 ** l, 4 ** l), np.int32)
            for b in range(4 ** l):
                M[b, idx[off[b]:off[b + 1]]] += 1
            count += M[np.ix_(anc, anc)]
    np.fill_diagonal(count, 1)
    assert (count == 1).all()


@pytest.mark.parametrize("dist", ["uniform", "clusters"])
def test_fmm_midpoint_within_gate(orc, dist):
    z, m = W.make(dist, 5000, seed=43)
    L = orc.nlevels(5000, 35)
    phi_d, dphi_d = orc.direct(z, m)
    phi, dphi = orc.plan(z, 0.5, L, midpoint=True).eval(m, 17)
    assert _nerr(phi.real, phi_d.real) <= 1e-6 and _nerr(dphi, dphi_d) <= orc.error_bound(0.5, 17)
