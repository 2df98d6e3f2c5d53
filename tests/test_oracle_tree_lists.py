"""Pins for the oracle's tree (O1/O2), discs (O3) and connectivity (O4).

Tree: P:333-341 median splits; pinned by a rank-counting brute force (a
different algorithm from the oracle's sorts), box sizes as a pure function of
N, the regular-lattice special case (leaves = K x K blocks of a uniform
quadtree) and the leaf-internal (y, idx) order.  Discs: tight-bbox identities and
the lattice closed form r = (K-1) h / sqrt(2).  Lists: P:343-353; pinned by the
exactly-once pair-coverage audit, symmetry, weak => criterion, strong
(non-self) => not criterion, and the lattice stencil closed form (9 strong,
27 weak interior at theta = 0.5).
"""
import json
import math
import os

import numpy as np
import pytest

import workloads as W

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def test_depth_rule_golden(orc):
    with open(os.path.join(GOLD, "depth_rule.json")) as f:
        g = json.load(f)
    for c in g["cases"]:
        assert orc.nlevels(c["n"], c["leaf_target"]) == c["L"]


def _sizes(n, L):
    """Box sizes per level from the split rule alone: x-low gets ceil(n/2), then
    each half's y-low gets ceil(h/2) (DESIGN R5)."""
    out = [[n]]
    for _ in range(L):
        nxt = []
        for s in out[-1]:
            h0 = (s + 1) // 2
            h1 = s - h0
            nxt += [(h0 + 1) // 2, h0 // 2, (h1 + 1) // 2, h1 // 2]
        out.append(nxt)
    return out


def _bruteforce_children(x, y, members):
    """Rank-count the definition: point i is x-low iff fewer than ceil(n/2) points
    of the box precede it in (x, idx) order; then inside each half the same in y."""
    members = list(members)
    n = len(members)

    def rank(i, key, pool):
        return sum(1 for j in pool if (key[j], j) < (key[i], i))

    xlow = [i for i in members if rank(i, x, members) < (n + 1) // 2]
    xhigh = [i for i in members if i not in set(xlow)]
    kids = []
    for half in (xlow, xhigh):
        h = len(half)
        ylow = [i for i in half if rank(i, y, half) < (h + 1) // 2]
        yhigh = [i for i in half if i not in set(ylow)]
        kids += [set(ylow), set(yhigh)]
    return kids


@pytest.mark.parametrize("dist,n,L", [("uniform", 150, 2), ("clusters", 200, 2), ("curve", 130, 3)])
def test_tree_matches_rank_bruteforce(orc, dist, n, L):
    z, _ = W.make(dist, n, seed=5)
    # inject ties in x and y and a -0 coordinate to exercise the (coord, idx) order
    z[10] = complex(z[11].real, z[10].imag)
    z[20] = complex(z[20].real, z[21].imag)
    z[30] = complex(-0.0, z[30].imag)
    z[31] = complex(0.0, z[31].imag)
    P = orc.plan(z, 0.5, L)
    perm = P.perm()
    x = [v + 0.0 for v in z.real]
    y = [v + 0.0 for v in z.imag]
    sizes = _sizes(n, L)
    for l in range(L):
        off = P.offsets(l)
        offc = P.offsets(l + 1)
        assert list(np.diff(off)) == sizes[l]
        for b in range(4 ** l):
            kids = _bruteforce_children(x, y, perm[off[b]:off[b + 1]])
            for q in range(4):
                c = 4 * b + q
                assert set(perm[offc[c]:offc[c + 1]].tolist()) == kids[q]
    # permutation is a bijection; leaves internally ascending in (y, idx) (DESIGN R13)
    assert sorted(perm.tolist()) == list(range(n))
    offL = P.offsets(L)
    for b in range(4 ** L):
        seg = perm[offL[b]:offL[b + 1]].tolist()
        assert seg == sorted(seg, key=lambda i: (y[i], i))


def test_tree_sizes_differ_by_at_most_one(orc):
    z, _ = W.make("clusters", 5000, seed=7)
    P = orc.plan(z, 0.5, 4)
    for l in range(5):
        s = np.diff(P.offsets(l))
        assert s.max() - s.min() <= 1
        assert s.min() == 5000 // 4 ** l and s.max() == -(-5000 // 4 ** l)


def _morton_xy(b, L):
    """leaf index -> (bx, by) block coordinates with child digit 2*xbit + ybit."""
    bx = by = 0
    for lev in range(L):
        d = (b >> (2 * (L - 1 - lev))) & 3
        bx = 2 * bx + (d >> 1)
        by = 2 * by + (d & 1)
    return bx, by


@pytest.mark.parametrize("K,L", [(4, 3), (5, 2)])
def test_tree_lattice_is_uniform_quadtree(orc, K, L):
    h = 0.25
    z = W.lattice(K, L, h=h, shuffle_seed=3)
    P = orc.plan(z, 0.5, L)
    perm = P.perm()
    off = P.offsets(L)
    cx, cy, r = P.discs(L)
    for b in range(4 ** L):
        bx, by = _morton_xy(b, L)
        pts = z[perm[off[b]:off[b + 1]]]
        ix = np.round(pts.real / h).astype(int)
        iy = np.round(pts.imag / h).astype(int)
        assert set(zip(ix.tolist(), iy.tolist())) == {(bx * K + a, by * K + c) for a in range(K) for c in range(K)}
        assert cx[b] == h * (bx * K + (K - 1) / 2) and cy[b] == h * (by * K + (K - 1) / 2)
        assert r[b] == pytest.approx((K - 1) * h / math.sqrt(2), rel=2e-16)


def test_discs_tight_bbox_and_containment(orc):
    z, _ = W.make("clusters", 3000, seed=9)
    L = 3
    P = orc.plan(z, 0.5, L)
    perm = P.perm()
    for l in range(L + 1):
        off = P.offsets(l)
        cx, cy, r = P.discs(l)
        for b in range(4 ** l):
            pts = z[perm[off[b]:off[b + 1]]]
            assert cx[b] == 0.5 * (pts.real.min() + pts.real.max())
            assert cy[b] == 0.5 * (pts.imag.min() + pts.imag.max())
            dist = np.abs(pts - complex(cx[b], cy[b]))
            assert r[b] >= dist.max() * (1 - 1e-15) and r[b] <= dist.max() * (1 + 1e-15)


def _ancestor(leaf_of, l, L):
    return leaf_of >> (2 * (L - l))


@pytest.mark.parametrize("dist,n,L,theta", [
    ("uniform", 1500, 3, 0.5), ("clusters", 1500, 3, 0.3), ("curve", 1500, 3, 0.7),
    ("uniform", 700, 4, 0.5), ("corners", 1200, 3, 0.5)])
def test_lists_exactly_once_coverage(orc, dist, n, L, theta):
    """Every ordered pair (i, j), i != j, is accounted for exactly once: by one
    ancestor weak pair or by the leaf strong pair."""
    z, _ = W.make(dist, n, seed=13)
    P = orc.plan(z, theta, L)
    perm = P.perm()
    offL = P.offsets(L)
    leaf_of = np.empty(n, np.int64)
    for b in range(4 ** L):
        leaf_of[perm[offL[b]:offL[b + 1]]] = b
    count = np.zeros((n, n), np.int32)
    for l in range(L + 1):
        nb = 4 ** l
        anc = _ancestor(leaf_of, l, L)
        for kind in (("weak",) if l < L else ("weak", "strong")):
            off, idx = P.list(l, kind)
            M = np.zeros((nb, nb), np.int32)
            for b in range(nb):
                M[b, idx[off[b]:off[b + 1]]] += 1
            count += M[np.ix_(anc, anc)]
    np.fill_diagonal(count, 1)
    assert (count == 1).all()


@pytest.mark.parametrize("dist,theta", [("uniform", 0.5), ("clusters", 0.5), ("curve", 0.3)])
def test_lists_symmetric_and_criterion_consistent(orc, dist, theta):
    z, _ = W.make(dist, 4000, seed=17)
    L = 4
    P = orc.plan(z, theta, L)
    for l in range(L + 1):
        cx, cy, r = P.discs(l)
        S = {}
        for kind in ("strong", "weak"):
            off, idx = P.list(l, kind)
            pairs = set()
            for b in range(4 ** l):
                row = idx[off[b]:off[b + 1]].tolist()
                assert row == sorted(row)                        # ascending (DESIGN R13)
                assert len(set(row)) == len(row)
                pairs |= {(b, c) for c in row}
            assert pairs == {(c, b) for (b, c) in pairs}         # symmetric
            S[kind] = pairs
        assert not (S["strong"] & S["weak"])
        for b in range(4 ** l):
            assert (b, b) in S["strong"]                         # always strong to itself
        for (b, c) in S["weak"]:
            assert orc.well_separated(complex(cx[b], cy[b]), r[b], complex(cx[c], cy[c]), r[c], theta)
        for (b, c) in S["strong"]:
            if b != c:
                assert not orc.well_separated(complex(cx[b], cy[b]), r[b], complex(cx[c], cy[c]), r[c], theta)
        if l >= 1:      # candidate soundness: lists of b are children of strong(parent(b))
            offp, idxp = P.list(l - 1, "strong")
            for (b, c) in S["strong"] | S["weak"]:
                assert (c >> 2) in set(idxp[offp[b >> 2]:offp[(b >> 2) + 1]].tolist())


def test_lists_lattice_stencil_closed_form(orc):
    """theta = 0.5 on a lattice with K x K leaves: offset o is strong iff
    |o|^2 < 4.5 ((K-1)/K)^2 (from R + theta r <= theta d with r = (K-1)h/sqrt 2),
    giving an interior strong stencil of 9 and 4*9 - 9 = 27 weak for K = 4."""
    K, L = 4, 4
    z = W.lattice(K, L, h=1.0, shuffle_seed=1)
    P = orc.plan(z, 0.5, L)
    off_s, _ = P.list(L, "strong")
    off_w, _ = P.list(L, "weak")
    ns = np.diff(off_s)
    nw = np.diff(off_w)
    side = 1 << L
    for b in range(4 ** L):
        bx, by = _morton_xy(b, L)
        if 2 <= bx < side - 2 and 2 <= by < side - 2:
            assert ns[b] == 9 and nw[b] == 27
    assert ns.max() == 9 and nw.max() == 27


def test_build_rejects_bad_input(orc):
    z = np.array([0.0 + 0j, 1.0 + 1j, 2.0 + 0j])
    for theta in (0.0, 1.0, -0.5, 1.5):
        with pytest.raises(ValueError):
            orc.plan(z, theta, 0)
    with pytest.raises(ValueError):
        orc.plan(z, 0.5, 1)           # N < 4^L (DESIGN R12)
    with pytest.raises(ValueError):
        orc.plan(np.array([0.0 + 0j, complex(np.nan, 0)]), 0.5, 0)
