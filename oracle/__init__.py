"""CPU oracle for the asymmetric adaptive 2D FMM (arXiv 1006.2269).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` may import this
package.  The product path (``paper_1006_2269_b200``) never imports it and
shares no code with it.

This module is a ctypes wrapper (argument marshalling only) over
``oracle/liboracle_fmm2d.so``, built from ``oracle/oracle_fmm2d.cpp`` with
``-O2 -ffp-contract=off -fopenmp``.  Every numeric step is in that C++ file,
which cites the paper passage it follows.

Parity status of each oracle function (what pins it, see tests/test_oracle_*.py):
  direct        pinned: closed forms (two-body), mpmath brute force
  nlevels       pinned: BASELINE.json level counts (C1: 3 levels, C5: 12 levels)
  tree          pinned: rank-count brute force, box sizes as a function of N,
                lattice -> uniform quadtree closed form
  discs         pinned: tight-bbox identities, lattice radius closed form
  lists         pinned: exactly-once pair coverage audit, symmetry, lattice stencil
                closed form, criterion examples + geometric meaning
  p2m/m2m/m2l/l2l/l2p pinned: closed forms (single charge, log 5, M2L series of a
                unit charge about 4, [1,1]->[2,1]), translation identities
  eval          pinned: error vs direct sum within the paper's a-priori law
                (P:281-285), decay slope ~ log10(theta), ordering in theta
  parent merge  pinned (O8): list audit (each cross pair replaces exactly four
                weak children and is itself well separated), exactly-once pair coverage,
                the pass against the direct sum within the gate, fewer M2L pairs
  midpoint tree pinned (O9, Fig. 2/4 baseline): equals the median tree on an aligned lattice
                (both are the uniform quadtree), containment of every point in its
                geometric cell, box counts = brute-force cell counts, exactly-once
                coverage with empty boxes, the pass against the direct sum
  rr exchange   pinned (O7): predicate worked examples + the exchanged
                geometric meaning, P2L closed form and P2L = M2L o P2M identity, M2P of a
                single charge, conversion-list audit (exchanged holds, original fails,
                symmetric bookkeeping), exactly-once pair coverage, the whole pass vs
                the direct sum within the gate
No function is "parity unpinned".
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle_fmm2d.cpp")
_LIB = os.environ.get("FMM2D_ORACLE_LIB") or os.path.join(_HERE, "liboracle_fmm2d.so")

_CFLAGS = ["-O2", "-ffp-contract=off", "-fno-fast-math", "-fopenmp", "-fPIC", "-shared", "-Wall"]


def build(force: bool = False) -> str:
    """Compile the oracle shared library in-tree (g++)."""
    if os.environ.get("FMM2D_ORACLE_LIB"):
        return _LIB
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(["g++", *_CFLAGS, "-o", _LIB, _SRC])
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB)
        dp = ctypes.POINTER(ctypes.c_double)
        i64p = ctypes.POINTER(ctypes.c_int64)
        u32p = ctypes.POINTER(ctypes.c_uint32)
        vp = ctypes.c_void_p
        L.oracle_direct.argtypes = [dp, dp, ctypes.c_int64, i64p, ctypes.c_int64, dp, dp]
        L.oracle_well_separated.argtypes = [ctypes.c_double] * 7
        L.oracle_nlevels.argtypes = [ctypes.c_int64, ctypes.c_int]
        L.oracle_build.argtypes = [dp, ctypes.c_int64, ctypes.c_double, ctypes.c_int, ctypes.POINTER(vp)]
        L.oracle_build_ex.argtypes = [dp, ctypes.c_int64, ctypes.c_double, ctypes.c_int, ctypes.c_int,
                                      ctypes.POINTER(vp)]
        L.oracle_rr_exchange.argtypes = [ctypes.c_double] * 7
        L.oracle_p2l.argtypes = [dp, dp, ctypes.c_int64, ctypes.c_double, ctypes.c_double, ctypes.c_int, dp]
        L.oracle_free.argtypes = [vp]
        L.oracle_free.restype = None
        L.oracle_levels.argtypes = [vp]
        L.oracle_get_perm.argtypes = [vp, u32p]
        L.oracle_get_offsets.argtypes = [vp, ctypes.c_int, i64p]
        L.oracle_get_discs.argtypes = [vp, ctypes.c_int, dp, dp, dp]
        L.oracle_list_total.argtypes = [vp, ctypes.c_int, ctypes.c_int]
        L.oracle_list_total.restype = ctypes.c_int64
        L.oracle_get_list.argtypes = [vp, ctypes.c_int, ctypes.c_int, i64p, u32p]
        L.oracle_eval.argtypes = [vp, dp, ctypes.c_int, dp, dp]
        L.oracle_get_expansions.argtypes = [vp, ctypes.c_int, ctypes.c_int, dp]
        L.oracle_p2m.argtypes = [dp, dp, ctypes.c_int64, ctypes.c_double, ctypes.c_double, ctypes.c_int, dp]
        L.oracle_m2m.argtypes = [dp, ctypes.c_double, ctypes.c_double, ctypes.c_double, ctypes.c_double, ctypes.c_int, dp]
        L.oracle_m2l.argtypes = [dp, ctypes.c_double, ctypes.c_double, ctypes.c_double, ctypes.c_double, ctypes.c_int, dp]
        L.oracle_l2l.argtypes = [dp, ctypes.c_double, ctypes.c_double, ctypes.c_double, ctypes.c_double, ctypes.c_int, dp]
        L.oracle_l2p.argtypes = [dp, ctypes.c_double, ctypes.c_double, ctypes.c_int, dp, ctypes.c_int64, dp, dp]
        L.oracle_m2p.argtypes = [dp, ctypes.c_double, ctypes.c_double, ctypes.c_int, dp, ctypes.c_int64, dp, dp]
        L.oracle_error_bound.argtypes = [ctypes.c_double, ctypes.c_int]
        L.oracle_error_bound.restype = ctypes.c_double
        _lib = L
    return _lib


def _dp(a):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def _c128(a) -> np.ndarray:
    """complex array -> contiguous complex128 (interleaved re, im)."""
    return np.ascontiguousarray(np.asarray(a, dtype=np.complex128))


def _as_f64(a: np.ndarray):
    return a.view(np.float64)


def direct(z, m, targets=None):
    """O0: Phi_i = sum_{j!=i} m_j Log(z_i - z_j), dPhi_i = sum_{j!=i} m_j/(z_i - z_j)
    (P:57-60), in long double.  Returns (phi, dphi) complex128 at ``targets``."""
    z = _c128(z)
    m = _c128(m)
    n = z.shape[0]
    if targets is None:
        nt, tp = n, None
    else:
        targets = np.ascontiguousarray(targets, dtype=np.int64)
        nt = targets.shape[0]
        tp = targets.ctypes.data_as(ctypes.POINTER(ctypes.c_int64))
    phi = np.zeros(nt, np.complex128)
    dphi = np.zeros(nt, np.complex128)
    rc = lib().oracle_direct(_dp(_as_f64(z)), _dp(_as_f64(m)), n, tp, nt if targets is not None else 0,
                             _dp(_as_f64(phi)), _dp(_as_f64(dphi)))
    if rc:
        raise ValueError(f"oracle_direct: {rc}")
    return phi, dphi


def well_separated(cb, rb, cc, rc, theta) -> bool:
    """Criterion 1 with the d > 0 guard (DESIGN R9)."""
    cb = complex(cb)
    cc = complex(cc)
    return bool(lib().oracle_well_separated(cb.real, cb.imag, rb, cc.real, cc.imag, rc, theta))


def nlevels(n: int, leaf_target: int) -> int:
    return int(lib().oracle_nlevels(n, leaf_target))


def error_bound(theta: float, p: int) -> float:
    """theta^{p+1}/(1-theta)^2, P:281-285 with the constant set to 1."""
    return float(lib().oracle_error_bound(theta, p))


class Plan:
    """Oracle tree + discs + lists for fixed (z, theta, L); ``eval(m, p)`` runs the
    evaluation pass.  Arrays are returned as numpy copies."""

    def __init__(self, z, theta: float, L: int, rr_exchange: bool = False, parent_merge: bool = False,
                 midpoint: bool = False):
        z = _c128(z)
        self.n = int(z.shape[0])
        self.theta = float(theta)
        self.L = int(L)
        self.rr_exchange = bool(rr_exchange)
        self.parent_merge = bool(parent_merge)
        h = ctypes.c_void_p()
        rc = lib().oracle_build_ex(_dp(_as_f64(z)), self.n, self.theta, self.L,
                                   (1 if rr_exchange else 0) | (2 if parent_merge else 0) | (4 if midpoint else 0),
                                   ctypes.byref(h))
        if rc:
            raise ValueError(f"oracle_build: {rc}")
        self._h = h

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            lib().oracle_free(h)
            self._h = None

    def perm(self) -> np.ndarray:
        out = np.empty(self.n, np.uint32)
        lib().oracle_get_perm(self._h, out.ctypes.data_as(ctypes.POINTER(ctypes.c_uint32)))
        return out

    def offsets(self, level: int) -> np.ndarray:
        out = np.empty(4 ** level + 1, np.int64)
        lib().oracle_get_offsets(self._h, level, out.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)))
        return out

    def discs(self, level: int):
        nb = 4 ** level
        cx, cy, r = (np.empty(nb, np.float64) for _ in range(3))
        lib().oracle_get_discs(self._h, level, _dp(cx), _dp(cy), _dp(r))
        return cx, cy, r

    def list(self, level: int, kind: str):
        """kind 'strong' or 'weak' (any level), 'near' / 'p2l' / 'm2p' (leaf level, the
        r/R exchange split of the strong list, O7) -> CSR (off int64[4^l+1], idx uint32[])."""
        k = {"strong": 0, "weak": 1, "near": 2, "p2l": 3, "m2p": 4, "xweak": 5}[kind]
        tot = lib().oracle_list_total(self._h, level, k)
        off = np.empty(4 ** level + 1, np.int64)
        idx = np.empty(max(tot, 1), np.uint32)
        lib().oracle_get_list(self._h, level, k, off.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)),
                              idx.ctypes.data_as(ctypes.POINTER(ctypes.c_uint32)))
        return off, idx[:tot]

    def eval(self, m, p: int):
        m = _c128(m)
        assert m.shape[0] == self.n
        phi = np.zeros(self.n, np.complex128)
        dphi = np.zeros(self.n, np.complex128)
        rc = lib().oracle_eval(self._h, _dp(_as_f64(m)), int(p), _dp(_as_f64(phi)), _dp(_as_f64(dphi)))
        if rc:
            raise ValueError(f"oracle_eval: {rc}")
        self.p = int(p)
        return phi, dphi

    def expansions(self, level: int, kind: str) -> np.ndarray:
        """Multipole ('mpole') or local ('local') coefficients of the last eval,
        shape (4^level, p+1) complex128."""
        out = np.empty((4 ** level, self.p + 1), np.complex128)
        lib().oracle_get_expansions(self._h, level, 1 if kind == "local" else 0, _dp(_as_f64(out)))
        return out


def plan(z, theta: float, L: int, rr_exchange: bool = False, parent_merge: bool = False,
         midpoint: bool = False) -> Plan:
    return Plan(z, theta, L, rr_exchange, parent_merge, midpoint)


def rr_exchange(cb, rb, cc, rc, theta) -> bool:
    """O7: Criterion 1 with the roles of r and R exchanged, r + theta R <= theta d,
    for r < R strictly."""
    cb = complex(cb)
    cc = complex(cc)
    return bool(lib().oracle_rr_exchange(cb.real, cb.imag, rb, cc.real, cc.imag, rc, theta))


def p2l(z, m, c, p):
    """O7 P2L: local expansion about c of the sources (z, m)."""
    z, m = _c128(z), _c128(m)
    b = np.zeros(p + 1, np.complex128)
    c = complex(c)
    lib().oracle_p2l(_dp(_as_f64(z)), _dp(_as_f64(m)), z.shape[0], c.real, c.imag, p, _dp(_as_f64(b)))
    return b


# --- single operators (pins) -------------------------------------------------

def p2m(z, m, c, p):
    z, m = _c128(z), _c128(m)
    a = np.zeros(p + 1, np.complex128)
    c = complex(c)
    lib().oracle_p2m(_dp(_as_f64(z)), _dp(_as_f64(m)), z.shape[0], c.real, c.imag, p, _dp(_as_f64(a)))
    return a


def m2m(a, c, cparent, p):
    a = _c128(a)
    b = np.zeros(p + 1, np.complex128)
    c, cp = complex(c), complex(cparent)
    lib().oracle_m2m(_dp(_as_f64(a)), c.real, c.imag, cp.real, cp.imag, p, _dp(_as_f64(b)))
    return b


def m2l(a, cs, ct, p):
    a = _c128(a)
    b = np.zeros(p + 1, np.complex128)
    cs, ct = complex(cs), complex(ct)
    lib().oracle_m2l(_dp(_as_f64(a)), cs.real, cs.imag, ct.real, ct.imag, p, _dp(_as_f64(b)))
    return b


def l2l(b, c, cnew, p):
    b = _c128(b)
    d = np.zeros(p + 1, np.complex128)
    c, cn = complex(c), complex(cnew)
    lib().oracle_l2l(_dp(_as_f64(b)), c.real, c.imag, cn.real, cn.imag, p, _dp(_as_f64(d)))
    return d


def l2p(b, c, p, z):
    b, z = _c128(b), _c128(np.atleast_1d(z))
    phi = np.zeros(z.shape[0], np.complex128)
    dphi = np.zeros(z.shape[0], np.complex128)
    c = complex(c)
    lib().oracle_l2p(_dp(_as_f64(b)), c.real, c.imag, p, _dp(_as_f64(z)), z.shape[0],
                     _dp(_as_f64(phi)), _dp(_as_f64(dphi)))
    return phi, dphi


def m2p(a, c, p, z):
    a, z = _c128(a), _c128(np.atleast_1d(z))
    phi = np.zeros(z.shape[0], np.complex128)
    dphi = np.zeros(z.shape[0], np.complex128)
    c = complex(c)
    lib().oracle_m2p(_dp(_as_f64(a)), c.real, c.imag, p, _dp(_as_f64(z)), z.shape[0],
                     _dp(_as_f64(phi)), _dp(_as_f64(dphi)))
    return phi, dphi
