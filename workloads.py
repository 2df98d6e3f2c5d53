"""Seeded synthetic workloads (inputs only -- no FMM arithmetic lives here).

Shared by the oracle side (tests, bench cpu_baseline) and the CUDA side (tests,
bench, smoke).  The paper measures only on synthetic point sets (P:457-464,
P:486-491); the configurations are BASELINE.json ``configs[0..4]``
(C1..C5), with the recipes of SURVEY.md section 8(d) restated in DESIGN.md
"Input recipe".  Generators are numpy PCG64 streams seeded with
``SEED_BASE + config index`` (or an explicit seed).

Every generator returns ``(z, m)``: complex128 arrays of length N (positions
z_j = x_j + i y_j and strengths m_j).
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

SEED_BASE = 100622690


@dataclass(frozen=True)
class Config:
    name: str
    n: int
    dist: str            # uniform | clusters | curve
    strengths: str       # real | phase
    theta: float
    p: int
    leaf_target: int


CONFIGS = {
    # BASELINE.json configs[0]: N=1e3 uniform, real m in [-1,1], theta=.5, p=17, ~35/leaf (3 levels)
    "C1": Config("C1", 1_000, "uniform", "real", 0.5, 17, 35),
    # configs[1]: N=1e5 uniform, unit-modulus complex m; theta/p sweep around (0.5, 17)
    "C2": Config("C2", 100_000, "uniform", "phase", 0.5, 17, 35),
    # configs[2]: N=1e6, 10 Gaussian clusters (sigma=.01) + 10% uniform background
    "C3": Config("C3", 1_000_000, "clusters", "real", 0.5, 17, 35),
    # configs[3]: N=1e7 on the curve x=t, y=0.1 sin(8 pi t), 1e-4 jitter
    "C4": Config("C4", 10_000_000, "curve", "real", 0.5, 17, 35),
    # configs[4]: N=1e8 uniform, ~40/leaf (12 levels): the metric's workload
    "C5": Config("C5", 100_000_000, "uniform", "real", 0.5, 17, 40),
}


def _rng(seed: int) -> np.random.Generator:
    return np.random.Generator(np.random.PCG64(seed))


def positions(dist: str, n: int, rng: np.random.Generator) -> np.ndarray:
    if dist == "uniform":
        xy = rng.random((n, 2))
        return xy[:, 0] + 1j * xy[:, 1]
    if dist == "clusters":
        # floor(0.9 N) cluster points, point i in cluster (i mod 10); cluster centres
        # U[0,1)^2; isotropic N(0, 0.01^2) per coordinate, no clipping; rest U[0,1)^2
        nc = (9 * n) // 10
        centres = rng.random((10, 2))
        k = np.arange(nc) % 10
        pts = centres[k] + 0.01 * rng.standard_normal((nc, 2))
        bg = rng.random((n - nc, 2))
        xy = np.concatenate([pts, bg], axis=0)
        return xy[:, 0] + 1j * xy[:, 1]
    if dist == "curve":
        # t ~ U[0,1): x = t + e_x, y = 0.1 sin(8 pi t) + e_y, e ~ N(0, (1e-4)^2)
        t = rng.random(n)
        e = 1e-4 * rng.standard_normal((n, 2))
        return (t + e[:, 0]) + 1j * (0.1 * np.sin(8.0 * np.pi * t) + e[:, 1])
    if dist.startswith("corners"):
        # four tight Gaussian clusters (sigma = 1e-3, or "corners:<sigma>") at the corners
        # of the square [0.2, 0.8]^2, point i in cluster (i mod 4): with N divisible by 4
        # every level-1 box of the median tree is exactly one cluster, so the level-1 boxes
        # are weakly coupled and level-1 M2L carries the whole far field
        sig = float(dist.split(":")[1]) if ":" in dist else 1e-3
        centres = np.array([[0.2, 0.2], [0.2, 0.8], [0.8, 0.2], [0.8, 0.8]])
        xy = centres[np.arange(n) % 4] + sig * rng.standard_normal((n, 2))
        return xy[:, 0] + 1j * xy[:, 1]
    if dist == "disc":
        # Fig. 3 (i): uniform in the unit disc
        r = np.sqrt(rng.random(n))
        a = 2.0 * np.pi * rng.random(n)
        return r * np.cos(a) + 1j * (r * np.sin(a))
    if dist == "disc_r":
        # Fig. 3 (ii): "radial density proportional to 1/r" in the unit disc;
        # reading R24: the areal density is ~1/r, so the radius is uniform on [0, 1)
        r = rng.random(n)
        a = 2.0 * np.pi * rng.random(n)
        return r * np.cos(a) + 1j * (r * np.sin(a))
    if dist == "disc_logr":
        # Fig. 3 (ii) under SPEC's reading (S:483 design decision): radial density ~ 1/r on the
        # truncated support [1e-8, 1], i.e. a log-uniform radius (the SURVEY f3 row's reading)
        r = np.exp(rng.uniform(np.log(1e-8), 0.0, n))
        a = 2.0 * np.pi * rng.random(n)
        return r * np.cos(a) + 1j * (r * np.sin(a))
    if dist.startswith("normal:") or dist.startswith("layer:"):
        # Fig. 4: "a normal distribution with variance sigma^2 or ... a 'layer'
        # distribution where the x-coordinate is uniformly distributed in [0,1], and the
        # y-coordinate again is N(0, sigma^2)-distributed ... forced by rejection to fit
        # exactly within the unit square" (clustering at the origin / the x-axis)
        kind, sig = dist.split(":")
        sig = float(sig)
        out = np.empty(0, np.complex128)
        while out.shape[0] < n:
            k = 2 * (n - out.shape[0]) + 64
            y = sig * rng.standard_normal(k)
            x = sig * rng.standard_normal(k) if kind == "normal" else rng.random(k)
            ok = (x >= 0) & (x <= 1) & (y >= 0) & (y <= 1)
            out = np.concatenate([out, (x + 1j * y)[ok]])
        return out[:n]
    raise ValueError(dist)


def strengths(kind: str, n: int, rng: np.random.Generator) -> np.ndarray:
    if kind == "real":
        return (2.0 * rng.random(n) - 1.0).astype(np.complex128)     # U[-1,1], Im m = 0
    if kind == "phase":
        return np.exp(1j * (2.0 * np.pi * rng.random(n)))               # e^{i phi}
    if kind == "mass":
        return np.full(n, 1.0 / n, np.complex128)                       # total mass 1 (Fig. 3)
    raise ValueError(kind)


def make(dist: str, n: int, strength_kind: str = "real", seed: int = SEED_BASE):
    rng = _rng(seed)
    z = positions(dist, n, rng)
    m = strengths(strength_kind, n, rng)
    return np.ascontiguousarray(z), np.ascontiguousarray(m)


def make_config(name: str, n: int | None = None, seed: int | None = None):
    """Inputs of BASELINE config ``name`` (optionally at a reduced N, same recipe)."""
    c = CONFIGS[name]
    idx = list(CONFIGS).index(name)
    return make(c.dist, c.n if n is None else n, c.strengths,
                SEED_BASE + idx if seed is None else seed)


def lattice(K: int, L: int, h: float = 1.0, shuffle_seed: int | None = None):
    """A (K 2^L) x (K 2^L) regular lattice with spacing h (tree special case: the
    median splits fall between columns, so leaves are K x K sub-blocks)."""
    s = K * (1 << L)
    ix, iy = np.meshgrid(np.arange(s), np.arange(s), indexing="ij")
    z = (h * ix.ravel()) + 1j * (h * iy.ravel())
    if shuffle_seed is not None:
        z = z[_rng(shuffle_seed).permutation(z.shape[0])]
    return np.ascontiguousarray(z.astype(np.complex128))


def sample_targets(n: int, M: int, seed: int = SEED_BASE + 99) -> np.ndarray:
    """Seeded random target sample (P:463-464 measure errors on M random points)."""
    M = min(M, n)
    return np.sort(_rng(seed).choice(n, size=M, replace=False)).astype(np.int64)
