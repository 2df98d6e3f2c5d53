"""Thin Python binding of libfmm2d.so (include/fmm2d.h): argument marshalling only.

Every step of the evaluation pass runs in the library's CUDA kernels; there is no
CPU fallback.  If the library is missing or no CUDA device is present the calls
raise.  PyTorch supplies device memory and streams.

    from paper_1006_2269_b200 import Fmm2d
    plan = Fmm2d(z, theta=0.5, p=17, leaf_target=40)     # z: complex128 (cuda tensor or numpy)
    phi, dphi = plan.eval(m)                             # Phi(z_i), Phi'(z_i) in input order

Method: S. Engblom, arXiv 1006.2269 -- Phi(z_i) = sum_{j!=i} m_j Log(z_i - z_j)
 by the asymmetric adaptive FMM.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# FMM2D_LIB selects an alternative build of the same library (tuning experiments only)
LIB_PATH = os.environ.get("FMM2D_LIB") or os.path.join(_HERE, "libfmm2d.so")

PMAX = 32
HOST_PTRS = 0x1
REAL_STRENGTHS = 0x2
SYMMETRIC_P2P = 0x4
TREE_KEY64 = 0x8
TREE_GLOBAL_ONLY = 0x10
RR_EXCHANGE = 0x20
PARENT_MERGE = 0x40
OVERLAP = 0x80
GATHER_OUTPUT = 0x100
MIDPOINT = 0x200
ASYNC_HOST = 0x400

EXPORT_PERM, EXPORT_OFFSETS, EXPORT_DISCS, EXPORT_STRONG, EXPORT_WEAK, EXPORT_MPOLE, EXPORT_LOCAL, \
    EXPORT_STATS, EXPORT_NEAR, EXPORT_RR_P2L, EXPORT_RR_M2P, EXPORT_XWEAK = range(1, 13)

# every symbol include/fmm2d.h declares
SYMBOLS = ["fmm2d_default_options", "fmm2d_build", "fmm2d_eval", "fmm2d_eval_timed", "fmm2d_launch_count",
           "fmm2d_free", "fmm2d_strerror", "fmm2d_last_error_detail", "fmm2d_plan_info", "fmm2d_export",
           "fmm2d_nccl_unique_id", "fmm2d_partition_info", "fmm2d_build_shards", "fmm2d_eval_shards",
           "fmm2d_halo_info", "fmm2d_build_eval", "fmm2d_reserve", "fmm2d_pool_trim", "fmm2d_pool_usage"]


class Options(ctypes.Structure):
    _fields_ = [("theta", ctypes.c_double), ("p", ctypes.c_int), ("leaf_target", ctypes.c_int),
                ("nlevels", ctypes.c_int), ("flags", ctypes.c_int), ("device", ctypes.c_int),
                ("stream", ctypes.c_void_p), ("nranks", ctypes.c_int), ("rank", ctypes.c_int),
                ("nccl_id", ctypes.c_void_p)]


class FmmError(RuntimeError):
    def __init__(self, code: int, what: str):
        self.code = code
        L = _lib
        msg = L.fmm2d_strerror(code).decode() if L else str(code)
        detail = L.fmm2d_last_error_detail().decode() if L else ""
        super().__init__(f"{what}: {msg} ({code}) {detail}".strip())


_lib = None


def lib():
    """Load libfmm2d.so (raises if it has not been built: no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"{LIB_PATH} is missing: build it with `make` (or __graft_entry__.build())")
        L = ctypes.CDLL(LIB_PATH)
        vp = ctypes.c_void_p
        L.fmm2d_default_options.argtypes = [ctypes.POINTER(Options)]
        L.fmm2d_build.argtypes = [vp, ctypes.c_int64, ctypes.POINTER(Options), ctypes.POINTER(vp)]
        L.fmm2d_eval.argtypes = [vp, vp, vp, vp]
        L.fmm2d_eval_timed.argtypes = [vp, vp, vp, vp, ctypes.POINTER(ctypes.c_double)]
        L.fmm2d_launch_count.argtypes = []
        L.fmm2d_launch_count.restype = ctypes.c_int64
        L.fmm2d_free.argtypes = [vp]
        L.fmm2d_free.restype = None
        L.fmm2d_strerror.argtypes = [ctypes.c_int]
        L.fmm2d_strerror.restype = ctypes.c_char_p
        L.fmm2d_last_error_detail.argtypes = []
        L.fmm2d_last_error_detail.restype = ctypes.c_char_p
        L.fmm2d_plan_info.argtypes = [vp, ctypes.POINTER(ctypes.c_int64), ctypes.POINTER(ctypes.c_int),
                                      ctypes.POINTER(ctypes.c_int), ctypes.POINTER(ctypes.c_int64),
                                      ctypes.POINTER(ctypes.c_int64)]
        L.fmm2d_export.argtypes = [vp, ctypes.c_int, ctypes.c_int, vp, ctypes.POINTER(ctypes.c_size_t)]
        L.fmm2d_nccl_unique_id.argtypes = [vp]
        L.fmm2d_partition_info.argtypes = [ctypes.c_int64, ctypes.POINTER(Options), ctypes.c_int, ctypes.c_int,
                                           ctypes.POINTER(ctypes.c_int64)]
        L.fmm2d_build_shards.argtypes = [vp, ctypes.c_int64, ctypes.POINTER(Options), ctypes.c_int,
                                         ctypes.POINTER(vp)]
        L.fmm2d_eval_shards.argtypes = [ctypes.POINTER(vp), ctypes.c_int, vp, vp, vp]
        L.fmm2d_halo_info.argtypes = [vp, ctypes.POINTER(ctypes.c_int64)]
        L.fmm2d_build_eval.argtypes = [vp, vp, ctypes.c_int64, ctypes.POINTER(Options), vp, vp, ctypes.POINTER(vp)]
        L.fmm2d_reserve.argtypes = [ctypes.c_int, ctypes.c_size_t]
        L.fmm2d_pool_trim.argtypes = [ctypes.c_int, ctypes.c_size_t]
        L.fmm2d_pool_usage.argtypes = [ctypes.c_int, ctypes.POINTER(ctypes.c_int64), ctypes.POINTER(ctypes.c_int64),
                                       ctypes.c_int]
        _lib = L
    return _lib


def launch_count() -> int:
    """Kernels launched by libfmm2d.so since it was loaded (CUB internals excluded)."""
    return int(lib().fmm2d_launch_count())


def _check(rc: int, what: str):
    if rc != 0:
        raise FmmError(rc, what)


def _options(theta=0.5, p=17, leaf_target=40, nlevels=-1, flags=0, device=0, stream=None, nranks=1, rank=0):
    opt = Options()
    lib().fmm2d_default_options(ctypes.byref(opt))
    opt.theta = float(theta)
    opt.p = int(p)
    opt.leaf_target = int(leaf_target)
    opt.nlevels = int(nlevels)
    opt.flags = int(flags)
    opt.device = int(device)
    opt.stream = ctypes.c_void_p(stream)
    opt.nranks = int(nranks)
    opt.rank = int(rank)
    return opt


def partition_info(n: int, nranks: int, rank: int, theta: float = 0.5, p: int = 17, leaf_target: int = 40,
                   nlevels: int = -1) -> dict:
    """Partition of the tree across ranks (host arithmetic only, no GPU needed):
    depth L, partition level k, own leaves, own leaf-order positions, own level-k subtrees."""
    info = (ctypes.c_int64 * 8)()
    opt = _options(theta, p, leaf_target, nlevels)
    _check(lib().fmm2d_partition_info(int(n), ctypes.byref(opt), int(nranks), int(rank), info),
           "fmm2d_partition_info")
    return {"L": info[0], "k": info[1], "leaves": (info[2], info[3]), "positions": (info[4], info[5]),
            "subtrees": (info[6], info[7])}


def nccl_unique_id() -> bytes:
    """A fresh 128-byte ncclUniqueId (make it on one rank, broadcast it to the others)."""
    buf = (ctypes.c_char * 128)()
    _check(lib().fmm2d_nccl_unique_id(buf), "fmm2d_nccl_unique_id")
    return bytes(buf)


def _ptr_of(a, host: bool, out: bool = False):
    """(pointer, keepalive) of a complex128 array: torch tensor (cuda or pinned cpu) or numpy.
    The caller keeps the keepalive bound until the C call (and, for asynchronous host plans,
    the stream) is done with the pointer.  Outputs (out=True) must already be contiguous
    complex128: a converted temporary would receive the results instead of the caller's array."""
    try:
        import torch
        if isinstance(a, torch.Tensor):
            if a.dtype != torch.complex128 or not a.is_contiguous():
                raise TypeError("expected a contiguous complex128 tensor")
            if host == a.is_cuda:
                raise TypeError("device/host pointer kind does not match the plan's flags")
            return a.data_ptr(), a
    except ImportError:
        pass
    if not host:
        raise TypeError("device plans need CUDA tensors")
    arr = np.ascontiguousarray(a, dtype=np.complex128)
    if out and not (isinstance(a, np.ndarray) and np.shares_memory(arr, a)):
        raise TypeError("outputs must be contiguous complex128 arrays (no conversion copy)")
    return arr.ctypes.data, arr


def reserve_pool(nbytes: int, device: int | None = None) -> None:
    """fmm2d_reserve: grow the device's stream-ordered memory pool (which the library's plans
    allocate from and keep) to at least nbytes, once, outside any timed section."""
    import torch
    if device is None:
        device = torch.cuda.current_device()
    _check(lib().fmm2d_reserve(int(device), int(nbytes)), "fmm2d_reserve")


def pool_trim(keep_bytes: int = 0, device: int | None = None) -> None:
    """fmm2d_pool_trim: return the library pool's unused memory to the device."""
    import torch
    if device is None:
        device = torch.cuda.current_device()
    _check(lib().fmm2d_pool_trim(int(device), int(keep_bytes)), "fmm2d_pool_trim")


def pool_usage(reset: bool = False, device: int | None = None) -> tuple:
    """fmm2d_pool_usage: (bytes in use, high-water bytes) of the library pool on `device`."""
    import torch
    if device is None:
        device = torch.cuda.current_device()
    u, h = ctypes.c_int64(), ctypes.c_int64()
    _check(lib().fmm2d_pool_usage(int(device), ctypes.byref(u), ctypes.byref(h), int(reset)), "fmm2d_pool_usage")
    return u.value, h.value


class Fmm2d:
    """A built plan (tree, discs, theta-criterion lists, expansion storage) for fixed
    positions z; ``eval(m)`` runs one evaluation pass.

    z: complex128 CUDA tensor (device plan) or host array (numpy / CPU tensor; the
    plan then uses FMM2D_HOST_PTRS and host inputs/outputs)."""

    def __init__(self, z, theta: float = 0.5, p: int = 17, leaf_target: int = 40, nlevels: int = -1,
                 real_strengths: bool = False, device: int | None = None, stream=None,
                 symmetric_p2p: bool = False, tree_key64: bool = False, tree_global_only: bool = False,
                 rr_exchange: bool = False, parent_merge: bool = False, overlap: bool = False,
                 gather_output: bool = False, midpoint: bool = False, async_host: bool = False,
                 nranks: int = 1, rank: int = 0,
                 nccl_id: bytes | None = None, _first=None):
        L = lib()
        import torch
        host = not (isinstance(z, torch.Tensor) and z.is_cuda)
        if device is None:
            device = z.device.index if (not host and z.device.index is not None) else torch.cuda.current_device()
        if stream is None:
            stream = torch.cuda.current_stream(device)
        self.device = device
        self.stream = stream
        self.host = host
        opt = Options()
        L.fmm2d_default_options(ctypes.byref(opt))
        opt.theta = float(theta)
        opt.p = int(p)
        opt.leaf_target = int(leaf_target)
        opt.nlevels = int(nlevels)
        opt.flags = ((HOST_PTRS if host else 0) | (REAL_STRENGTHS if real_strengths else 0)
                     | (SYMMETRIC_P2P if symmetric_p2p else 0) | (TREE_KEY64 if tree_key64 else 0)
                     | (TREE_GLOBAL_ONLY if tree_global_only else 0) | (RR_EXCHANGE if rr_exchange else 0)
                     | (PARENT_MERGE if parent_merge else 0) | (OVERLAP if overlap else 0)
                     | (GATHER_OUTPUT if gather_output else 0) | (MIDPOINT if midpoint else 0)
                     | (ASYNC_HOST if async_host else 0))
        opt.device = int(device)
        opt.stream = ctypes.c_void_p(stream.cuda_stream)
        opt.nranks = int(nranks)
        opt.rank = int(rank)
        self._nccl_id = None
        if nranks > 1:
            if nccl_id is None or len(nccl_id) != 128:
                raise ValueError("nranks > 1 needs the 128-byte nccl_id shared by all ranks")
            self._nccl_id = ctypes.create_string_buffer(bytes(nccl_id), 128)
            opt.nccl_id = ctypes.cast(self._nccl_id, ctypes.c_void_p)
        self.nranks, self.rank = int(nranks), int(rank)
        self.async_host = bool(async_host)
        self._opt = opt
        zp, keep = _ptr_of(z, host)
        self.n = int(keep.shape[0])
        h = ctypes.c_void_p()
        if _first is None:
            _check(L.fmm2d_build(ctypes.c_void_p(zp), self.n, ctypes.byref(opt), ctypes.byref(h)), "fmm2d_build")
        else:                                   # (m, phi, dphi): fmm2d_build_eval
            mp, mkeep = _ptr_of(_first[0], host)
            pp, pkeep = _ptr_of(_first[1], host, out=True) if _first[1] is not None else (None, None)
            dp, dkeep = _ptr_of(_first[2], host, out=True) if _first[2] is not None else (None, None)
            if host and (opt.flags & ASYNC_HOST):
                self._inflight = (keep, mkeep, pkeep, dkeep)   # read by the streams after the call returns
            _check(L.fmm2d_build_eval(ctypes.c_void_p(zp), ctypes.c_void_p(mp), self.n, ctypes.byref(opt),
                                      ctypes.c_void_p(pp), ctypes.c_void_p(dp), ctypes.byref(h)),
                   "fmm2d_build_eval")
            self.async_host = False             # FMM2D_ASYNC_HOST covered that evaluation only
        self._h = h
        n = ctypes.c_int64()
        nl = ctypes.c_int()
        pp = ctypes.c_int()
        wp = ctypes.c_int64()
        sp = ctypes.c_int64()
        _check(L.fmm2d_plan_info(h, ctypes.byref(n), ctypes.byref(nl), ctypes.byref(pp), ctypes.byref(wp),
                                 ctypes.byref(sp)), "fmm2d_plan_info")
        self.L = nl.value
        self.p = pp.value
        self.theta = float(theta)
        self.weak_pairs = wp.value
        self.strong_leaf_pairs = sp.value

    @classmethod
    def build_eval(cls, z, m, phi=None, dphi=None, **kw):
        """Build the plan and evaluate once (fmm2d_build_eval): for host arrays the strengths'
        copy to the device overlaps the tree build.  Returns (plan, phi, dphi); phi / dphi
        are allocated like eval's when not given (pinned host, or on the device)."""
        import torch
        host = not (isinstance(z, torch.Tensor) and z.is_cuda)
        n = int(z.shape[0])
        if phi is None or dphi is None:
            if host:
                pin = torch.cuda.is_available()
                phi = torch.empty(n, dtype=torch.complex128, pin_memory=pin) if phi is None else phi
                dphi = torch.empty(n, dtype=torch.complex128, pin_memory=pin) if dphi is None else dphi
            else:
                phi = torch.empty(n, dtype=torch.complex128, device=z.device) if phi is None else phi
                dphi = torch.empty(n, dtype=torch.complex128, device=z.device) if dphi is None else dphi
        plan = cls(z, _first=(m, phi, dphi), **kw)
        return plan, phi, dphi

    # -- evaluation -------------------------------------------------------
    def eval(self, m, phi=None, dphi=None, want_phi: bool = True, want_dphi: bool = True):
        """Phi(z_i), Phi'(z_i) in input order.  Device plans: complex128 CUDA tensors,
        asynchronous on the plan's stream.  Host plans: numpy/pinned arrays, synchronous --
        except for a plan built with async_host=True (FMM2D_ASYNC_HOST), where the call
        returns once the copies are enqueued and the results are valid after
        ``plan.stream.synchronize()``.  A plan from build_eval(async_host=True) is async for
        that call's evaluation only; its later eval calls are synchronous."""
        import torch
        if self._h is None:
            raise RuntimeError("plan freed")
        mp, mkeep = _ptr_of(m, self.host)
        if self.host:
            if want_phi and phi is None:
                phi = torch.empty(self.n, dtype=torch.complex128, pin_memory=torch.cuda.is_available())
            if want_dphi and dphi is None:
                dphi = torch.empty(self.n, dtype=torch.complex128, pin_memory=torch.cuda.is_available())
        else:
            dev = torch.device("cuda", self.device)
            if want_phi and phi is None:
                phi = torch.empty(self.n, dtype=torch.complex128, device=dev)
            if want_dphi and dphi is None:
                dphi = torch.empty(self.n, dtype=torch.complex128, device=dev)
        pp, pkeep = _ptr_of(phi, self.host, out=True) if phi is not None else (None, None)
        dp, dkeep = _ptr_of(dphi, self.host, out=True) if dphi is not None else (None, None)
        _check(lib().fmm2d_eval(self._h, ctypes.c_void_p(mp), ctypes.c_void_p(pp), ctypes.c_void_p(dp)),
               "fmm2d_eval")
        if self.host and self.async_host:
            self._inflight = (mkeep, pkeep, dkeep)     # the stream still reads / writes them
        return phi, dphi

    def eval_timed(self, m, phi, dphi) -> dict:
        """eval into preallocated outputs, synchronise, return per-phase device ms."""
        t = (ctypes.c_double * 8)()
        mp, mkeep = _ptr_of(m, self.host)
        pp, pkeep = _ptr_of(phi, self.host, out=True) if phi is not None else (None, None)
        dp, dkeep = _ptr_of(dphi, self.host, out=True) if dphi is not None else (None, None)
        _check(lib().fmm2d_eval_timed(self._h, ctypes.c_void_p(mp), ctypes.c_void_p(pp), ctypes.c_void_p(dp), t),
               "fmm2d_eval_timed")
        del mkeep, pkeep, dkeep
        return {"gather_ms": t[0], "upward_ms": t[1], "m2l_ms": t[2], "downward_ms": t[3], "near_ms": t[4],
                "eval_ms": t[5]}

    # -- exports (tests / diagnostics) -------------------------------------
    def _export(self, what: int, level: int = 0) -> bytes:
        L = lib()
        nbytes = ctypes.c_size_t(0)
        _check(L.fmm2d_export(self._h, what, level, None, ctypes.byref(nbytes)), "fmm2d_export(size)")
        buf = (ctypes.c_char * max(nbytes.value, 1))()
        _check(L.fmm2d_export(self._h, what, level, buf, ctypes.byref(nbytes)), "fmm2d_export")
        return bytes(buf)[: nbytes.value]

    def perm(self) -> np.ndarray:
        return np.frombuffer(self._export(EXPORT_PERM), np.uint32).copy()

    def offsets(self, level: int) -> np.ndarray:
        return np.frombuffer(self._export(EXPORT_OFFSETS, level), np.int64).copy()

    def discs(self, level: int):
        a = np.frombuffer(self._export(EXPORT_DISCS, level), np.float64).reshape(3, -1)
        return a[0].copy(), a[1].copy(), a[2].copy()

    def list(self, level: int, kind: str):
        """kind 'strong' / 'weak' (any level); 'near' / 'p2l' / 'm2p' (leaf level: the direct
        pairs and the r/R exchange conversions) -> CSR (off int64[4^l+1], idx uint32[])."""
        what = {"strong": EXPORT_STRONG, "weak": EXPORT_WEAK, "near": EXPORT_NEAR, "p2l": EXPORT_RR_P2L,
                "m2p": EXPORT_RR_M2P, "xweak": EXPORT_XWEAK}[kind]
        raw = self._export(what, level)
        nb = 4 ** level
        off = np.frombuffer(raw[: 8 * (nb + 1)], np.int64).copy()
        idx = np.frombuffer(raw[8 * (nb + 1):], np.uint32).copy()
        return off, idx

    def expansions(self, level: int, kind: str) -> np.ndarray:
        raw = self._export(EXPORT_LOCAL if kind == "local" else EXPORT_MPOLE, level)
        return np.frombuffer(raw, np.complex128).reshape(4 ** level, self.p + 1).copy()

    def halo_info(self) -> dict:
        info = (ctypes.c_int64 * 9)()
        _check(lib().fmm2d_halo_info(self._h, info), "fmm2d_halo_info")
        return {"import_leaves": info[0], "import_mpoles": info[1], "export_leaves": info[2],
                "export_mpoles": info[3], "nranks": info[4], "rank": info[5], "k": info[6],
                "positions": (info[7], info[8])}

    def stats(self) -> dict:
        s = np.frombuffer(self._export(EXPORT_STATS), np.float64)
        keys = ["n", "L", "p", "theta", "weak_pairs", "strong_leaf_pairs", "min_leaf", "max_leaf",
                "t_build_ms", "t_tree_ms", "t_lists_ms", "nboxes", "launches", "p2p_pairs", "tree_key64", "dev_bytes"]
        return {k: float(v) for k, v in zip(keys, s)}

    def close(self):
        if getattr(self, "_h", None) is not None and self._h.value:
            lib().fmm2d_free(self._h)
        self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()


class _ShardHandle(Fmm2d):
    """One rank of a loopback build (exports only; evaluate through LoopbackShards)."""

    def __init__(self, h, n, p, theta, device, stream):      # noqa: D401 - no build here
        self._h = h
        self.n = n
        self.theta = theta
        self.device = device
        self.stream = stream
        self.host = False
        nl = ctypes.c_int()
        pp = ctypes.c_int()
        _check(lib().fmm2d_plan_info(h, None, ctypes.byref(nl), ctypes.byref(pp), None, None), "fmm2d_plan_info")
        self.L = nl.value
        self.p = pp.value


class LoopbackShards:
    """The partitioned (multi-GPU) pass with all ranks as plans on ONE device, every
    transfer between ranks a device copy.  ``eval`` returns the
    complete Phi, Phi' (each rank writes the entries of the sources it owns)."""

    def __init__(self, z, nshards: int, theta: float = 0.5, p: int = 17, leaf_target: int = 40,
                 nlevels: int = -1, real_strengths: bool = False, stream=None, parent_merge: bool = False):
        import torch
        if not (isinstance(z, torch.Tensor) and z.is_cuda):
            raise TypeError("loopback shards take a complex128 CUDA tensor")
        device = z.device.index if z.device.index is not None else torch.cuda.current_device()
        if stream is None:
            stream = torch.cuda.current_stream(device)
        self.n = int(z.shape[0])
        self.device = device
        self.stream = stream
        flags = (REAL_STRENGTHS if real_strengths else 0) | (PARENT_MERGE if parent_merge else 0)
        opt = _options(theta, p, leaf_target, nlevels, flags, device, stream.cuda_stream, nshards, 0)
        hs = (ctypes.c_void_p * nshards)()
        zp, _ = _ptr_of(z, False)
        _check(lib().fmm2d_build_shards(ctypes.c_void_p(zp), self.n, ctypes.byref(opt), int(nshards), hs),
               "fmm2d_build_shards")
        self._hs = hs
        self.shards = [_ShardHandle(ctypes.c_void_p(hs[i]), self.n, p, theta, device, stream) for i in range(nshards)]

    def eval(self, m, phi=None, dphi=None):
        import torch
        dev = torch.device("cuda", self.device)
        if phi is None:
            phi = torch.zeros(self.n, dtype=torch.complex128, device=dev)
        if dphi is None:
            dphi = torch.zeros(self.n, dtype=torch.complex128, device=dev)
        mp = _ptr_of(m, False)[0]
        _check(lib().fmm2d_eval_shards(self._hs, len(self.shards), ctypes.c_void_p(mp),
                                       ctypes.c_void_p(phi.data_ptr()), ctypes.c_void_p(dphi.data_ptr())),
               "fmm2d_eval_shards")
        return phi, dphi

    def close(self):
        for s in self.shards:
            s.close()
        self.shards = []
