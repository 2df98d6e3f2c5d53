"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle.

Bar (BASELINE north_star):
  - permutation, box offsets, discs (centre, radius) and the strong / weak CSR
    lists of every level: bit-exact;
  - Phi and Phi' (complex, FMM branch R2): normwise max-abs error / max-abs
    <= 1e-12 against the oracle FMM on the same inputs;
  - Re Phi (real m) and Phi' against the direct sum within BJ's 1e-6 gate.
Sizes span several tiles and ragged leaves; full-size configurations are
checked on sampled outputs (tests/test_gpu_fullsize.py).
"""
import numpy as np
import pytest
import torch

import workloads as W
from fullparity import errors as _errors

pytestmark = pytest.mark.gpu

TOL = 1e-12


def _nerr(a, b):
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-300))


def _gpu_plan(z, theta, p, L, real=False):
    from paper_1006_2269_b200 import Fmm2d
    zt = torch.from_numpy(z).cuda()
    return Fmm2d(zt, theta=theta, p=p, nlevels=L, real_strengths=real)


def _gpu_eval(plan, m):
    phi, dphi = plan.eval(torch.from_numpy(m).cuda())
    torch.cuda.synchronize()
    return phi.cpu().numpy(), dphi.cpu().numpy()


def _check_structure(gp, op, L):
    assert gp.L == op.L == L
    np.testing.assert_array_equal(gp.perm(), op.perm())
    for l in range(L + 1):
        np.testing.assert_array_equal(gp.offsets(l), op.offsets(l))
        gcx, gcy, gr = gp.discs(l)
        ocx, ocy, orr = op.discs(l)
        np.testing.assert_array_equal(gcx, ocx)
        np.testing.assert_array_equal(gcy, ocy)
        np.testing.assert_array_equal(gr, orr)
        for kind in ("strong", "weak"):
            go, gi = gp.list(l, kind)
            oo, oi = op.list(l, kind)
            np.testing.assert_array_equal(go, oo, err_msg=f"{kind} offsets level {l}")
            np.testing.assert_array_equal(gi, oi, err_msg=f"{kind} idx level {l}")


STRUCT_CASES = [
    ("C1", lambda: W.make_config("C1"), 0.5, None),
    ("C2", lambda: W.make_config("C2"), 0.5, None),
    ("C2-theta.3", lambda: W.make_config("C2"), 0.3, None),
    ("C2-theta.7", lambda: W.make_config("C2"), 0.7, None),
    ("C3-200k", lambda: W.make_config("C3", n=200_000), 0.5, None),
    ("C4-200k", lambda: W.make_config("C4", n=200_000), 0.5, None),
    ("lattice-ties", lambda: (W.lattice(6, 4, h=0.5, shuffle_seed=2), None), 0.5, 4),
    ("ragged-7777", lambda: W.make("uniform", 7777, seed=3), 0.5, 3),
    # level-1 weak pairs (DESIGN R15): four tight clusters, one per level-1 box
    ("corners-t.5", lambda: W.make("corners", 2000, seed=31), 0.5, 2),
    ("corners-t.3", lambda: W.make("corners", 40_000, seed=32), 0.3, 4),
]


@pytest.mark.parametrize("name,mk,theta,L", STRUCT_CASES, ids=[c[0] for c in STRUCT_CASES])
def test_tree_and_lists_bit_exact(orc, name, mk, theta, L):
    z, _ = mk()
    if L is None:
        L = orc.nlevels(len(z), 35)
    gp = _gpu_plan(z, theta, 17, L)
    op = orc.plan(z, theta, L)
    _check_structure(gp, op, L)


def test_tree_adversarial_ties_dups_negzero(orc):
    rng = np.random.default_rng(9)
    n = 5000
    x = np.round(rng.random(n) * 20) / 20          # heavy ties in x and y
    y = np.round(rng.random(n) * 20) / 20
    x[:50] = -0.0                                  # -0 mixed with +0
    y[50:100] = 0.0
    x[100:400] = 0.25                              # 300 duplicates
    y[100:400] = 0.75
    z = x + 1j * y
    for L in (2, 4):
        gp = _gpu_plan(z, 0.5, 8, L)
        op = orc.plan(z, 0.5, L)
        _check_structure(gp, op, L)


def test_tree_tiny_and_forced_levels(orc):
    for n, L in ((1, 0), (3, 0), (4, 1), (17, 2), (64, 3)):
        z, _ = W.make("uniform", n, seed=n)
        gp = _gpu_plan(z, 0.5, 4, L)
        op = orc.plan(z, 0.5, L)
        _check_structure(gp, op, L)


def test_tree_presort_paths(orc):
    """The 32-bit-key presort with equal-key runs fixed in place (DESIGN 6.1) and the
    64-bit-key fallback build the same tree as the oracle.  Near-ties: distinct x that
    share a 32-bit key bucket (runs of 2..32, fixed in place); heavy ties: runs longer
    than 32 (the axis falls back to 64-bit keys)."""
    from paper_1006_2269_b200 import Fmm2d
    rng = np.random.default_rng(17)
    n = 10_000
    x = np.round(rng.random(n) * 1000) / 1000 + rng.random(n) * 1e-13     # ~10 per bucket
    y = rng.random(n)
    near = x + 1j * y
    heavy = np.round(rng.random(n) * 100) / 100 + 1j * y                     # ~100 per value
    for z, key64_expected in ((near, 0), (heavy, 1)):
        L = 4
        op = orc.plan(z, 0.5, L)
        gp = _gpu_plan(z, 0.5, 8, L)
        assert int(gp.stats()["tree_key64"]) == key64_expected
        _check_structure(gp, op, L)
        g64 = Fmm2d(torch.from_numpy(z).cuda(), theta=0.5, p=8, nlevels=L, tree_key64=True)
        assert int(g64.stats()["tree_key64"]) == 3
        _check_structure(g64, op, L)


@pytest.mark.parametrize("cfg,n", [("C1", None), ("C2", None), ("C3", 200_000)])
def test_tree_global_only_equals_on_chip_finish(orc, cfg, n):
    """The deepest levels split on chip (k_tree_local) and every step in global memory
    (k_partition only) give the same tree as the oracle (DESIGN 6.1)."""
    from paper_1006_2269_b200 import Fmm2d
    z, _ = W.make_config(cfg, n=n)
    L = orc.nlevels(len(z), 35)
    op = orc.plan(z, 0.5, L)
    g = Fmm2d(torch.from_numpy(z).cuda(), theta=0.5, p=8, nlevels=L, tree_global_only=True)
    _check_structure(g, op, L)


EVAL_CASES = [
    ("C1", "C1", None, 0.5, 17),
    ("C2-t.5-p17", "C2", None, 0.5, 17),
    ("C2-t.3-p8", "C2", None, 0.3, 8),
    ("C2-t.7-p30", "C2", None, 0.7, 30),
    ("C3-100k", "C3", 100_000, 0.5, 17),
    ("C4-100k", "C4", 100_000, 0.5, 17),
]


@pytest.mark.parametrize("name,cfg,n,theta,p", EVAL_CASES, ids=[c[0] for c in EVAL_CASES])
def test_eval_matches_oracle(orc, name, cfg, n, theta, p):
    z, m = W.make_config(cfg, n=n)
    L = orc.nlevels(len(z), 35)
    gp = _gpu_plan(z, theta, p, L)
    op = orc.plan(z, theta, L)
    phi_o, dphi_o = op.eval(m, p)
    phi_g, dphi_g = _gpu_eval(gp, m)
    assert np.isfinite(phi_g).all() and np.isfinite(dphi_g).all()
    e1, e2 = _nerr(phi_g, phi_o), _nerr(dphi_g, dphi_o)
    assert e1 <= TOL and e2 <= TOL, (e1, e2)
    # pointwise, with the floor 1e-3 max|ref| (tests/fullparity.py)
    p1, p2 = _errors(phi_g, phi_o), _errors(dphi_g, dphi_o)
    assert p1["point"] <= TOL and p2["point"] <= TOL, (p1, p2)


@pytest.mark.parametrize("threads", [64, 96, 128])
@pytest.mark.parametrize("cfg,n", [("C2", None), ("C3", 60_000)])
def test_near_block_sizes(orc, monkeypatch, threads, cfg, n):
    """k_near picks its block size per plan (64 / 96 / 128 threads: the fewest idle lanes for the
    plan's target tuples); every choice gives the oracle's result within the parity bar
    (FMM2D_NEAR_THREADS forces one; the group partial sums are added in a different order)."""
    monkeypatch.setenv("FMM2D_NEAR_THREADS", str(threads))
    z, m = W.make_config(cfg, n=n)
    L = orc.nlevels(len(z), 35)
    gp = _gpu_plan(z, 0.5, 17, L)
    phi_o, dphi_o = orc.plan(z, 0.5, L).eval(m, 17)
    phi_g, dphi_g = _gpu_eval(gp, m)
    e1, e2 = _nerr(phi_g, phi_o), _nerr(dphi_g, dphi_o)
    assert e1 <= TOL and e2 <= TOL, (threads, e1, e2)
    p1, p2 = _errors(phi_g, phi_o), _errors(dphi_g, dphi_o)
    assert p1["point"] <= TOL and p2["point"] <= TOL, (threads, p1, p2)


@pytest.mark.parametrize("n,theta,L", [(2000, 0.5, 2), (40_000, 0.3, 4), (40_000, 0.5, 4)])
def test_eval_level1_weak_pairs(orc, n, theta, L):
    """Level-1 M2L carries the whole inter-cluster field (corners input, DESIGN R15): the GPU
    lists hold the 12 level-1 weak pairs, the outputs match the oracle within 1e-12 and the
    direct sum within BJ's gate."""
    z, m = W.make("corners", n, "real", seed=33)
    gp = _gpu_plan(z, theta, 17, L, real=True)
    op = orc.plan(z, theta, L)
    _check_structure(gp, op, L)
    assert len(gp.list(1, "weak")[1]) == 12
    phi_o, dphi_o = op.eval(m, 17)
    phi_g, dphi_g = _gpu_eval(gp, m)
    assert _nerr(phi_g, phi_o) <= TOL and _nerr(dphi_g, dphi_o) <= TOL
    lo = gp.expansions(1, "local")
    assert np.abs(lo - op.expansions(1, "local")).max() <= 1e-12 * np.abs(op.expansions(1, "local")).max()
    t = W.sample_targets(n, 200, seed=34)
    phi_d, dphi_d = orc.direct(z, m, targets=t)
    assert _nerr(phi_g[t].real, phi_d.real) <= 1e-6
    assert _nerr(dphi_g[t], dphi_d) <= orc.error_bound(theta, 17)


def test_eval_real_strength_flag_matches(orc):
    z, m = W.make_config("C1")
    L = 2
    a = _gpu_eval(_gpu_plan(z, 0.5, 17, L, real=True), m)
    b = _gpu_eval(_gpu_plan(z, 0.5, 17, L, real=False), m)
    op = orc.plan(z, 0.5, L)
    phi_o, dphi_o = op.eval(m, 17)
    assert _nerr(a[0], phi_o) <= TOL and _nerr(a[1], dphi_o) <= TOL
    assert _nerr(a[0], b[0]) <= TOL


def test_expansions_per_level_match_oracle(orc):
    """Diagnostic parity of every multipole and local expansion (locate any error)."""
    z, m = W.make_config("C2", n=20_000)
    L = orc.nlevels(len(z), 35)
    gp = _gpu_plan(z, 0.5, 17, L)
    op = orc.plan(z, 0.5, L)
    op.eval(m, 17)
    _gpu_eval(gp, m)
    for l in range(L + 1):
        for kind in ("mpole", "local"):
            g = gp.expansions(l, kind)
            o = op.expansions(l, kind)
            if l == 0 and kind == "local":
                assert np.all(g == 0) and np.all(o == 0)
                continue
            # coefficient-wise normwise error, scaled per coefficient index
            for k in range(18):
                den = np.abs(o[:, k]).max()
                if den > 0:
                    assert np.abs(g[:, k] - o[:, k]).max() <= 1e-12 * den, (l, kind, k)


def test_eval_vs_direct_sum_gate(orc):
    z, m = W.make_config("C1")
    gp = _gpu_plan(z, 0.5, 17, 2)
    phi_g, dphi_g = _gpu_eval(gp, m)
    phi_d, dphi_d = orc.direct(z, m)
    assert _nerr(phi_g.real, phi_d.real) <= 1e-6
    assert _nerr(dphi_g, dphi_d) <= orc.error_bound(0.5, 17)


def test_eval_root_only_equals_direct(orc):
    z, m = W.make("uniform", 300, "phase", seed=31)       # L = 0: pure P2P, > 128 targets
    phi_g, dphi_g = _gpu_eval(_gpu_plan(z, 0.5, 5, 0), m)
    phi_d, dphi_d = orc.direct(z, m)
    assert _nerr(phi_g, phi_d) <= 1e-13 and _nerr(dphi_g, dphi_d) <= 1e-13


@pytest.mark.parametrize("n,L", [(1, 0), (2, 0), (3, 0), (4, 1), (5, 1), (16, 2)])
def test_eval_tiny_inputs_match_direct(orc, n, L):
    """Degenerate sizes: one point (empty sum: Phi = Phi' = 0), a pair, one point per leaf
    (every leaf-level box is its own near list), forced levels on tiny inputs.  Against the
    oracle: Phi and Phi'; against the direct sum: Re Phi and Phi' (real strengths: the FMM
    branch of Im Phi is not the principal-branch sum's, DESIGN R2)."""
    z, m = W.make("uniform", n, "real", seed=100 + n)
    phi_g, dphi_g = _gpu_eval(_gpu_plan(z, 0.5, 17, L), m)
    if n == 1:
        assert np.all(phi_g == 0) and np.all(dphi_g == 0)
        return
    phi_o, dphi_o = orc.plan(z, 0.5, L).eval(m, 17)
    assert _nerr(phi_g, phi_o) <= TOL and _nerr(dphi_g, dphi_o) <= TOL
    phi_d, dphi_d = orc.direct(z, m)
    assert _nerr(phi_g.real, phi_d.real) <= 1e-6 and _nerr(dphi_g, dphi_d) <= 1e-6


def test_host_pointer_path_equals_device_path():
    from paper_1006_2269_b200 import Fmm2d
    z, m = W.make_config("C1")
    dev = _gpu_eval(_gpu_plan(z, 0.5, 17, 2), m)
    hp = Fmm2d(z, theta=0.5, p=17, nlevels=2)           # numpy -> FMM2D_HOST_PTRS
    phi, dphi = hp.eval(m)
    np.testing.assert_array_equal(phi.numpy(), dev[0])
    np.testing.assert_array_equal(dphi.numpy(), dev[1])


@pytest.mark.parametrize("host", [True, False])
def test_build_eval_equals_build_then_eval(host):
    """fmm2d_build_eval (the strengths' copy overlapping the build for host buffers) gives
    the result of fmm2d_build + fmm2d_eval bit for bit, and its plan is reusable."""
    import torch
    from paper_1006_2269_b200 import Fmm2d
    z, m = W.make_config("C2", n=40_000)
    ref = _gpu_plan(z, 0.5, 17, 5)
    a = _gpu_eval(ref, m)
    m2 = np.ascontiguousarray(m[::-1])
    a2 = _gpu_eval(ref, m2)
    if host:
        plan, phi, dphi = Fmm2d.build_eval(z, m, theta=0.5, p=17, nlevels=5)
        got = (phi.numpy(), dphi.numpy())
        phi2, dphi2 = plan.eval(m2)
        got2 = (phi2.numpy(), dphi2.numpy())
    else:
        zd, md, m2d = (torch.from_numpy(v).cuda() for v in (z, m, m2))
        plan, phi, dphi = Fmm2d.build_eval(zd, md, theta=0.5, p=17, nlevels=5)
        got = (phi.cpu().numpy(), dphi.cpu().numpy())
        phi2, dphi2 = plan.eval(m2d)
        got2 = (phi2.cpu().numpy(), dphi2.cpu().numpy())
    for x, y in zip(got + got2, a + a2):
        np.testing.assert_array_equal(x, y)
    plan.close()


def test_async_host_two_problems_in_flight():
    """FMM2D_ASYNC_HOST: two host-buffer problems in flight on two streams (the bench's e2e
    pattern) give the synchronous results bit for bit once each stream is synchronised."""
    import torch
    from paper_1006_2269_b200 import Fmm2d
    z1, m1 = W.make_config("C2", n=40_000)
    z2, m2 = W.make_config("C3", n=60_000)
    ref1 = Fmm2d.build_eval(z1, m1, theta=0.5, p=17)[1:]
    ref2 = Fmm2d.build_eval(z2, m2, theta=0.5, p=17)[1:]
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    out = []
    plans = []
    for z, m, st in ((z1, m1, s1), (z2, m2, s2), (z1, m1, s2)):
        ph = torch.empty(z.shape[0], dtype=torch.complex128).pin_memory()
        dh = torch.empty(z.shape[0], dtype=torch.complex128).pin_memory()
        plans.append(Fmm2d.build_eval(z, m, ph, dh, theta=0.5, p=17, stream=st, async_host=True)[0])
        out.append((ph, dh))
    s1.synchronize()
    s2.synchronize()
    for (ph, dh), ref in zip(out, (ref1, ref2, ref1)):
        np.testing.assert_array_equal(ph.numpy(), ref[0].numpy())
        np.testing.assert_array_equal(dh.numpy(), ref[1].numpy())
    # FMM2D_ASYNC_HOST covered build_eval's own evaluation only: a later eval on the host
    # plan is synchronous (results valid on return, no stream synchronisation)
    ph2, dh2 = plans[1].eval(m2)
    np.testing.assert_array_equal(np.asarray(ph2), ref2[0].numpy())
    np.testing.assert_array_equal(np.asarray(dh2), ref2[1].numpy())
    for p_ in plans:
        p_.close()


def test_reserve_pool_then_build():
    """fmm2d_reserve grows the memory pool once; builds afterwards work as before."""
    import torch
    from paper_1006_2269_b200 import Fmm2d, reserve_pool
    reserve_pool(1 << 30)
    reserve_pool(1 << 20)                               # already large enough: no-op
    z, m = W.make_config("C2", n=20_000)
    a = Fmm2d.build_eval(z, m, theta=0.5, p=17, nlevels=5)[1:]
    b = _gpu_eval(_gpu_plan(z, 0.5, 17, 5), m)
    np.testing.assert_array_equal(a[0].numpy(), b[0])
    np.testing.assert_array_equal(a[1].numpy(), b[1])


def test_eval_deterministic_and_reusable():
    z, m = W.make_config("C2", n=30_000)
    gp = _gpu_plan(z, 0.5, 17, 5)
    a = _gpu_eval(gp, m)
    b = _gpu_eval(gp, m)
    np.testing.assert_array_equal(a[0], b[0])
    np.testing.assert_array_equal(a[1], b[1])
    m2 = np.ascontiguousarray(m[::-1])
    c = _gpu_eval(gp, m2)                                  # new strengths, same plan
    assert not np.array_equal(c[0], a[0])


def test_coincident_distinct_points_are_nonfinite():
    """Coincident DISTINCT points are not an error (DESIGN R21): their pair has dz = 0,
    so Phi and Phi' of both points are non-finite; every other point stays finite."""
    z, m = W.make("uniform", 3000, seed=5)
    z[1234] = z[77]
    phi, dphi = _gpu_eval(_gpu_plan(z, 0.5, 17, 3), m)
    bad = np.zeros(len(z), bool)
    bad[[77, 1234]] = True
    assert not np.isfinite(phi[bad]).all() and not np.isfinite(dphi[bad]).all()
    assert np.isfinite(phi[~bad]).all() and np.isfinite(dphi[~bad]).all()


def test_nonfinite_rejected():
    from paper_1006_2269_b200 import Fmm2d, FmmError
    z = np.zeros(100, np.complex128) + np.arange(100)
    z[7] = complex(np.inf, 0)
    with pytest.raises(FmmError) as e:
        Fmm2d(torch.from_numpy(z).cuda(), nlevels=1)
    assert e.value.code == -2


@pytest.mark.parametrize("cfg,n", [("C2", 50_000), ("C3", 100_000), ("C4", 100_000), ("C1", None)])
def test_symmetric_near_field_equals_one_sided(orc, cfg, n):
    """FMM2D_SYMMETRIC_P2P evaluates each unordered leaf pair once (both directions); the
    default evaluates every ordered pair.  Same sums up to rounding, and both match the
    oracle within the 1e-12 bar."""
    from paper_1006_2269_b200 import Fmm2d
    z, m = W.make_config(cfg, n=n)
    L = orc.nlevels(len(z), 35)
    zt, mt = torch.from_numpy(z).cuda(), torch.from_numpy(m).cuda()
    real = W.CONFIGS[cfg].strengths == "real"
    out = {}
    for one_sided in (False, True):
        plan = Fmm2d(zt, theta=0.5, p=17, nlevels=L, real_strengths=real, symmetric_p2p=not one_sided)
        phi, dphi = plan.eval(mt)
        torch.cuda.synchronize()
        out[one_sided] = (phi.cpu().numpy(), dphi.cpu().numpy())
    assert _nerr(out[False][0], out[True][0]) <= 1e-13 and _nerr(out[False][1], out[True][1]) <= 1e-13
    phi_o, dphi_o = orc.plan(z, 0.5, L).eval(m, 17)
    assert _nerr(out[False][0], phi_o) <= TOL and _nerr(out[False][1], dphi_o) <= TOL


RR_CASES = [("C3-100k", "C3", 100_000), ("C4-100k", "C4", 100_000), ("C3-30k-p8", "C3", 30_000)]


@pytest.mark.parametrize("name,cfg,n", RR_CASES, ids=[c[0] for c in RR_CASES])
def test_rr_exchange_lists_and_eval_match_oracle(orc, name, cfg, n):
    """FMM2D_RR_EXCHANGE (DESIGN R23): the near / P2L / M2P split of the leaf
    strong lists bit-exact, Phi and Phi' within 1e-12 of the oracle pass with the same
    conversions, and the conversions actually remove direct pairs."""
    from paper_1006_2269_b200 import Fmm2d
    z, m = W.make_config(cfg, n=n)
    L = orc.nlevels(len(z), 35)
    p = 8 if name.endswith("p8") else 17
    op = orc.plan(z, 0.5, L, rr_exchange=True)
    gp = Fmm2d(torch.from_numpy(z).cuda(), theta=0.5, p=p, nlevels=L, rr_exchange=True)
    for kind in ("strong", "near", "p2l", "m2p"):
        go, gi = gp.list(L, kind)
        oo, oi = op.list(L, kind)
        np.testing.assert_array_equal(go, oo, err_msg=kind)
        np.testing.assert_array_equal(gi, oi, err_msg=kind)
    assert op.list(L, "p2l")[1].size > 0
    phi_o, dphi_o = op.eval(m, p)
    phi_g, dphi_g = _gpu_eval(gp, m)
    assert _nerr(phi_g, phi_o) <= TOL and _nerr(dphi_g, dphi_o) <= TOL
    off = Fmm2d(torch.from_numpy(z).cuda(), theta=0.5, p=p, nlevels=L)
    assert gp.stats()["p2p_pairs"] < off.stats()["p2p_pairs"]


def test_near_split_long_lists(orc):
    """Leaves whose near lists exceed FMM2D_NEAR_SPLIT source rows are evaluated in
    segments by several CTAs and combined in segment order: same results as the oracle
    (clustered input: leaves strongly coupled to thousands of leaves)."""
    z, m = W.make_config("C3", n=200_000)
    L = orc.nlevels(len(z), 35)
    op = orc.plan(z, 0.5, L)
    so, si = op.list(L, "strong")
    offL = op.offsets(L)
    sizes = np.diff(offL)
    rows = np.array([sizes[si[so[t]:so[t + 1]]].sum() for t in range(4 ** L)])
    assert (rows > 4096).sum() > 0
    phi_o, dphi_o = op.eval(m, 17)
    phi_g, dphi_g = _gpu_eval(_gpu_plan(z, 0.5, 17, L), m)
    assert _nerr(phi_g, phi_o) <= TOL and _nerr(dphi_g, dphi_o) <= TOL


PM_CASES = [("C2", None, 0.5, 17), ("C3-100k", 100_000, 0.5, 17), ("C2-t.3-p8", None, 0.3, 8)]


@pytest.mark.parametrize("name,n,theta,p", PM_CASES, ids=[c[0] for c in PM_CASES])
def test_parent_merge_lists_and_eval_match_oracle(orc, name, n, theta, p):
    """FMM2D_PARENT_MERGE (DESIGN R25): weak, strong and cross-level lists of
    every level bit-exact, Phi and Phi' within 1e-12 of the oracle pass with the merge."""
    from paper_1006_2269_b200 import Fmm2d
    cfg = name.split("-")[0]
    z, m = W.make_config(cfg, n=n)
    L = orc.nlevels(len(z), 35)
    op = orc.plan(z, theta, L, parent_merge=True)
    gp = Fmm2d(torch.from_numpy(z).cuda(), theta=theta, p=p, nlevels=L, parent_merge=True)
    nx = 0
    for l in range(L + 1):
        for kind in ("strong", "weak", "xweak"):
            go, gi = gp.list(l, kind)
            oo, oi = op.list(l, kind)
            np.testing.assert_array_equal(go, oo, err_msg=f"{kind} {l}")
            np.testing.assert_array_equal(gi, oi, err_msg=f"{kind} {l}")
        nx += op.list(l, "xweak")[1].size
    assert nx > 0
    phi_o, dphi_o = op.eval(m, p)
    phi_g, dphi_g = _gpu_eval(gp, m)
    assert _nerr(phi_g, phi_o) <= TOL and _nerr(dphi_g, dphi_o) <= TOL


@pytest.mark.parametrize("cfg,n,rr", [("C2", None, False), ("C3", 100_000, True), ("C3", 200_000, False)])
def test_overlapped_eval_bit_identical(cfg, n, rr):
    """FMM2D_OVERLAP runs the expansion chain on a side stream concurrently with the P2P
    sums (DESIGN 6.4); the default runs them one after the other.  Same summation order:
    bit-identical results (also with r/R exchange and split near lists)."""
    from paper_1006_2269_b200 import Fmm2d
    z, m = W.make_config(cfg, n=n)
    zt, mt = torch.from_numpy(z).cuda(), torch.from_numpy(m).cuda()
    out = []
    for ov in (True, False):
        plan = Fmm2d(zt, theta=0.5, p=17, leaf_target=35, overlap=ov, rr_exchange=rr)
        phi, dphi = plan.eval(mt)
        torch.cuda.synchronize()
        out.append((phi, dphi))
    assert torch.equal(out[0][0], out[1][0]) and torch.equal(out[0][1], out[1][1])


MID_CASES = [("C2", None, 0.5, 17), ("C3-100k", 100_000, 0.5, 17), ("C4-100k", 100_000, 0.5, 17),
             ("C1-t.3-p8", None, 0.3, 8)]


@pytest.mark.parametrize("name,n,theta,p", MID_CASES, ids=[c[0] for c in MID_CASES])
def test_midpoint_tree_matches_oracle(orc, name, n, theta, p):
    """FMM2D_MIDPOINT (Fig. 2 / Fig. 4 uniform baseline, DESIGN R26): permutation, offsets,
    discs (empty boxes r = -1) and lists of every level bit-exact, Phi and Phi' within
    1e-12 of the oracle pass on the same midpoint tree."""
    from paper_1006_2269_b200 import Fmm2d
    cfg = name.split("-")[0]
    z, m = W.make_config(cfg, n=n)
    L = orc.nlevels(len(z), 35)
    op = orc.plan(z, theta, L, midpoint=True)
    gp = Fmm2d(torch.from_numpy(z).cuda(), theta=theta, p=p, nlevels=L, midpoint=True)
    _check_structure(gp, op, L)
    phi_o, dphi_o = op.eval(m, p)
    phi_g, dphi_g = _gpu_eval(gp, m)
    assert _nerr(phi_g, phi_o) <= TOL and _nerr(dphi_g, dphi_o) <= TOL
