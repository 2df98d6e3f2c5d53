"""Whole-problem parity of the CUDA path against the oracle (test infrastructure).

``compare(z, m, theta, p, L, ...)`` builds and evaluates the GPU plan through the C ABI,
builds and evaluates the oracle plan (oracle/, plain C++), and compares
  - perm, box offsets, discs and the strong / weak CSR lists of EVERY level bit for bit
    (median splits, discs of Criterion 1, the recursive connectivity rule),
  - Phi and Phi' over ALL N sources: normwise max|d|/max|ref| (DESIGN R3) and
    pointwise |d_i| / max(|ref_i|, floor * max|ref|) (the floor keeps points where Phi_i
    nearly cancels from dividing rounding noise by ~0; stated with the result).
It returns a dict of timings and errors; the callers assert the bars.  Used by
tests/test_gpu_fullsize.py and tools/full_parity.py (the one-off C5 log under profiles/).
"""
from __future__ import annotations

import time

import numpy as np

PT_FLOOR = 1e-3


def errors(g, o, floor=PT_FLOOR):
    d = np.abs(g - o)
    a = np.abs(o)
    amax = float(a.max()) if a.size else 0.0
    if amax == 0.0:
        return {"norm": float(d.max()) if d.size else 0.0, "point": 0.0, "point_q50": 0.0, "point_q99": 0.0}
    pw = d / np.maximum(a, floor * amax)
    return {"norm": float(d.max() / amax), "point": float(pw.max()),
            "point_q50": float(np.quantile(pw, 0.5)), "point_q99": float(np.quantile(pw, 0.99))}


def compare(z, m, theta, p, L, real=True, levels=None, evaluate=True, log=print, rr_exchange=False,
            parent_merge=False):
    """rr_exchange / parent_merge: the optional steps (R23, R25) on both
    sides; their lists (leaf near / P2L / M2P, cross-level weak) are compared bit for bit too."""
    import torch

    import oracle
    from paper_1006_2269_b200 import Fmm2d

    n = len(z)
    out = {"n": n, "theta": theta, "p": p, "L": L, "pt_floor": PT_FLOOR}
    t0 = time.time()
    gp = Fmm2d(torch.from_numpy(z).cuda(), theta=theta, p=p, nlevels=L, real_strengths=real,
               rr_exchange=rr_exchange, parent_merge=parent_merge)
    if evaluate:
        phi, dphi = gp.eval(torch.from_numpy(m).cuda())
        torch.cuda.synchronize()
        phi_g, dphi_g = phi.cpu().numpy(), dphi.cpu().numpy()
        del phi, dphi
    out["gpu_s"] = time.time() - t0
    log(f"gpu build+eval {out['gpu_s']:.1f} s")
    t0 = time.time()
    op = oracle.plan(z, theta, L, rr_exchange=rr_exchange, parent_merge=parent_merge)
    out["oracle_build_s"] = time.time() - t0
    log(f"oracle build {out['oracle_build_s']:.1f} s")
    t0 = time.time()
    if not np.array_equal(gp.perm(), op.perm()):
        raise AssertionError("perm differs")
    out["levels_compared"] = []
    out["entries_compared"] = {"strong": 0, "weak": 0}
    for l in (range(L + 1) if levels is None else levels):
        if not np.array_equal(gp.offsets(l), op.offsets(l)):
            raise AssertionError(f"offsets differ at level {l}")
        for name, a, b in zip(("cx", "cy", "r"), gp.discs(l), op.discs(l)):
            if not np.array_equal(a, b):
                raise AssertionError(f"disc {name} differs at level {l}")
        kinds = ["strong", "weak"]
        if parent_merge and l >= 2:
            kinds.append("xweak")
        if rr_exchange and l == L:
            kinds += ["near", "p2l", "m2p"]
        for kind in kinds:
            go, gi = gp.list(l, kind)
            oo, oi = op.list(l, kind)
            if not np.array_equal(go, oo):
                raise AssertionError(f"{kind} offsets differ at level {l}")
            if not np.array_equal(gi, oi):
                raise AssertionError(f"{kind} entries differ at level {l}")
            out["entries_compared"][kind] = out["entries_compared"].get(kind, 0) + int(len(oi))
            del go, gi, oo, oi
        out["levels_compared"].append(l)
    out["structure_s"] = time.time() - t0
    log(f"structure bit-exact on levels {out['levels_compared']} ({out['entries_compared']}) "
        f"{out['structure_s']:.1f} s")
    gp.close()
    del gp
    if evaluate:
        t0 = time.time()
        phi_o, dphi_o = op.eval(m, p)
        out["oracle_eval_s"] = time.time() - t0
        log(f"oracle eval {out['oracle_eval_s']:.1f} s")
        if not (np.isfinite(phi_g).all() and np.isfinite(dphi_g).all()):
            raise AssertionError("non-finite GPU output")
        out["phi"] = errors(phi_g, phi_o)
        out["dphi"] = errors(dphi_g, dphi_o)
        log(f"phi {out['phi']}  dphi {out['dphi']}")
    del op
    return out
