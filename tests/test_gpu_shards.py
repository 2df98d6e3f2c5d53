"""The partitioned (multi-GPU) pass, run as loopback shards on one GPU.

DESIGN.md section 8: rank r of P owns the level-k subtrees [r 4^k/P, (r+1) 4^k/P);
levels <= k are replicated, halo leaves and multipoles are imported.  Each own box
sees the same lists, multipoles and locals as in the one-GPU plan, in the same
order, so the union of the ranks' outputs must equal the one-GPU result BIT FOR BIT,
and every own box's lists must equal the one-GPU plan's rows.  Loopback transfers are
device copies between plans on one device; no kernel waits on another rank's.
"""
import numpy as np
import pytest
import torch

import workloads as W

pytestmark = pytest.mark.gpu


def _single(z, theta, p, L, real):
    from paper_1006_2269_b200 import Fmm2d
    return Fmm2d(z, theta=theta, p=p, nlevels=L, real_strengths=real)


CASES = [
    ("C2-P2", "C2", 50_000, 2, 0.5, 17),
    ("C2-P4", "C2", 50_000, 4, 0.5, 17),
    ("C2-P8", "C2", 50_000, 8, 0.5, 17),
    ("C3-P8", "C3", 200_000, 8, 0.5, 17),
    ("C4-P4", "C4", 200_000, 4, 0.5, 17),
    ("C1-P2-p8", "C1", None, 2, 0.3, 8),
    ("ragged-P8-t.7", "C2", 33_333, 8, 0.7, 30),
]


@pytest.mark.parametrize("name,cfg,n,P,theta,p", CASES, ids=[c[0] for c in CASES])
def test_loopback_shards_equal_single_gpu(orc, name, cfg, n, P, theta, p):
    from paper_1006_2269_b200 import LoopbackShards, partition_info
    z_np, m_np = W.make_config(cfg, n=n)
    N = len(z_np)
    L = orc.nlevels(N, 35)
    z = torch.from_numpy(z_np).cuda()
    m = torch.from_numpy(m_np).cuda()
    real = W.CONFIGS[cfg].strengths == "real"
    ref = _single(z, theta, p, L, real)
    phi_r, dphi_r = ref.eval(m)
    sh = LoopbackShards(z, P, theta=theta, p=p, nlevels=L, real_strengths=real)
    phi_s, dphi_s = sh.eval(m)
    torch.cuda.synchronize()
    assert torch.equal(phi_s, phi_r) and torch.equal(dphi_s, dphi_r)
    # a second evaluation with new strengths through the same shards
    m2 = torch.flip(m, [0]).contiguous()
    a = ref.eval(m2)
    b = sh.eval(m2)
    torch.cuda.synchronize()
    assert torch.equal(a[0], b[0]) and torch.equal(a[1], b[1])
    # structure: own boxes' lists and discs equal the one-GPU plan's
    perm_r = ref.perm()
    for r, s in enumerate(sh.shards):
        info = partition_info(N, P, r, theta=theta, p=p, nlevels=L)
        k = info["k"]
        h = s.halo_info()
        assert (h["nranks"], h["rank"], h["k"]) == (P, r, k)
        k0, k1 = info["positions"]
        assert h["positions"] == (k0, k1)
        np.testing.assert_array_equal(s.perm()[k0:k1], perm_r[k0:k1])
        for l in range(L + 1):
            for a_, b_ in zip(s.discs(l), ref.discs(l)):
                np.testing.assert_array_equal(a_, b_)
            nb = 4 ** l
            lo, hi = (0, nb) if l <= k else (nb // P * r, nb // P * (r + 1))
            for kind in ("strong", "weak"):
                so, si = s.list(l, kind)
                ro, ri = ref.list(l, kind)
                for b in range(lo, hi, max(1, (hi - lo) // 257)):
                    np.testing.assert_array_equal(si[so[b]:so[b + 1]], ri[ro[b]:ro[b + 1]])
                assert so[hi] - so[lo] == ro[hi] - ro[lo]
    sh.close()


def test_shard_partition_facts():
    from paper_1006_2269_b200 import partition_info, FmmError
    n = 1_000_003
    for P in (2, 4, 8, 16):
        parts = [partition_info(n, P, r) for r in range(P)]
        assert parts[0]["positions"][0] == 0 and parts[-1]["positions"][1] == n
        for a, b in zip(parts, parts[1:]):
            assert a["positions"][1] == b["positions"][0]
    with pytest.raises(FmmError):
        partition_info(n, 3, 0)                     # not a power of two


def test_shards_reject_unpartitionable():
    from paper_1006_2269_b200 import LoopbackShards, FmmError
    z_np, _ = W.make_config("C2", n=2000)
    z = torch.from_numpy(z_np).cuda()
    with pytest.raises(FmmError):
        LoopbackShards(z, 3, nlevels=3)             # P = 3: no level with 3 | 4^k
    with pytest.raises(FmmError):
        LoopbackShards(z, 8, nlevels=2)             # k = 2 needs L > 2


def test_loopback_shards_with_parent_merge(orc):
    """Cross-level halo multipoles (parent merge) through the partition: bit-identical."""
    from paper_1006_2269_b200 import Fmm2d, LoopbackShards
    z_np, m_np = W.make_config("C2", n=60_000)
    L = orc.nlevels(len(z_np), 35)
    z, m = torch.from_numpy(z_np).cuda(), torch.from_numpy(m_np).cuda()
    ref = Fmm2d(z, theta=0.5, p=17, nlevels=L, parent_merge=True)
    a = ref.eval(m)
    for P in (2, 8):
        sh = LoopbackShards(z, P, theta=0.5, p=17, nlevels=L, parent_merge=True)
        b = sh.eval(m)
        torch.cuda.synchronize()
        assert torch.equal(a[0], b[0]) and torch.equal(a[1], b[1])
        sh.close()


@pytest.mark.parametrize("name", ["lattice-ties", "dups-negzero"])
def test_loopback_shards_ties_and_duplicates(name):
    """Split records found by selection with heavy ties (lattice, duplicates, -0) and the
    per-box presort's 64-bit fallback: shards still equal the one-GPU result bit for bit."""
    from paper_1006_2269_b200 import Fmm2d, LoopbackShards
    if name == "lattice-ties":
        z_np = W.lattice(8, 3, h=0.5, shuffle_seed=4)
        L = 4
    else:
        rng = np.random.default_rng(12)
        n = 20_000
        # heavy ties in each coordinate (never two coincident points): x on a grid of 51
        # values (-0.0 among them), a block of 600 with x = 0.5, then y = 0.25 on 300 of
        # them with x moved off the tie
        x = np.round(rng.random(n) * 50) / 50
        y = rng.random(n)
        x[:40] = -0.0
        x[100:700] = 0.5
        y[100:400] = 0.25
        x[100:400] = np.arange(300) * 1e-6 + 0.5
        z_np = x + 1j * y
        L = 4
    m_np = np.random.default_rng(1).uniform(-1, 1, z_np.shape[0]) + 0j
    z, m = torch.from_numpy(z_np).cuda(), torch.from_numpy(m_np).cuda()
    ref = Fmm2d(z, theta=0.5, p=12, nlevels=L)
    a = ref.eval(m)
    for P in (2, 8):
        sh = LoopbackShards(z, P, theta=0.5, p=12, nlevels=L)
        b = sh.eval(m)
        torch.cuda.synchronize()
        assert torch.equal(a[0], b[0]) and torch.equal(a[1], b[1])
        sh.close()


@pytest.mark.parametrize("case", ["uniform-300k", "C3-200k", "ties-200k"])
def test_loopback_shards_sliced_selection(monkeypatch, case):
    """FMM2D_SEL_SLICED=1: the top-level selection counted and collected slice by slice (the
    NCCL path's per-rank slices, summed / gathered as its all-reduce and all-gather would) --
    shards still equal the one-GPU result bit for bit."""
    from paper_1006_2269_b200 import Fmm2d, LoopbackShards
    monkeypatch.setenv("FMM2D_SEL_SLICED", "1")
    rng = np.random.default_rng(33)
    if case == "uniform-300k":
        z_np = rng.random(300_000) + 1j * rng.random(300_000)
    elif case == "C3-200k":
        z_np, _ = W.make_config("C3", n=200_000)
    else:
        n = 200_000
        z_np = np.round(rng.random(n) * 8) / 8 + 1j * rng.random(n)      # 9 distinct x values
    m_np = rng.uniform(-1, 1, z_np.shape[0]) + 0j
    z, m = torch.from_numpy(z_np).cuda(), torch.from_numpy(m_np).cuda()
    ref = Fmm2d(z, theta=0.5, p=12, leaf_target=40)
    a = ref.eval(m)
    for P in (2, 4, 8):
        sh = LoopbackShards(z, P, theta=0.5, p=12, leaf_target=40)
        b = sh.eval(m)
        torch.cuda.synchronize()
        assert torch.equal(a[0], b[0]) and torch.equal(a[1], b[1])
        sh.close()
    ref.close()
