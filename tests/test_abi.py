"""The C-ABI library loads and exports every symbol include/fmm2d.h declares; host-side
validation (no GPU needed) rejects bad arguments with the documented codes."""
import ctypes
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "fmm2d.h")).read()
    return sorted(set(re.findall(r"FMM2D_API\s+[\w\s\*]*?\b(fmm2d_\w+)\s*\(", src)))


def test_header_symbols_exported():
    import paper_1006_2269_b200 as F
    L = F.lib()
    names = _declared()
    assert len(names) >= 8
    assert sorted(F.SYMBOLS) == names
    for s in names:
        assert hasattr(L, s), s


def test_exports_are_only_the_abi():
    import subprocess
    import paper_1006_2269_b200 as F
    out = subprocess.run(["nm", "-D", "--defined-only", F.LIB_PATH], capture_output=True, text=True).stdout
    funcs = sorted(l.split()[-1] for l in out.splitlines() if " T " in l)
    assert funcs == _declared()


def test_default_options_and_strerror():
    import paper_1006_2269_b200 as F
    L = F.lib()
    o = F.fmm2d.Options()
    assert L.fmm2d_default_options(ctypes.byref(o)) == 0
    assert (o.theta, o.p, o.leaf_target, o.nlevels, o.nranks, o.rank) == (0.5, 17, 40, -1, 1, 0)
    assert L.fmm2d_strerror(-1) == b"invalid argument"
    assert L.fmm2d_strerror(-2) == b"non-finite coordinate"
    assert L.fmm2d_default_options(None) == -1


@pytest.mark.parametrize("field,value", [("theta", 0.0), ("theta", 1.0), ("theta", -0.1), ("theta", float("nan")),
                                         ("p", 0), ("p", 33), ("leaf_target", 0), ("nlevels", 3)])
def test_build_rejects_invalid_options_without_gpu(field, value):
    import paper_1006_2269_b200 as F
    L = F.lib()
    o = F.fmm2d.Options()
    L.fmm2d_default_options(ctypes.byref(o))
    setattr(o, field, value)
    z = np.zeros(10, np.complex128)        # n = 10 < 4^3 for the nlevels case
    h = ctypes.c_void_p()
    rc = L.fmm2d_build(ctypes.c_void_p(z.ctypes.data), 10, ctypes.byref(o), ctypes.byref(h))
    assert rc == -1 and not h.value


def test_build_rejects_bad_sizes_and_nulls():
    import paper_1006_2269_b200 as F
    L = F.lib()
    o = F.fmm2d.Options()
    L.fmm2d_default_options(ctypes.byref(o))
    z = np.zeros(4, np.complex128)
    h = ctypes.c_void_p()
    assert L.fmm2d_build(ctypes.c_void_p(z.ctypes.data), 0, ctypes.byref(o), ctypes.byref(h)) == -1
    assert L.fmm2d_build(ctypes.c_void_p(z.ctypes.data), 1 << 31, ctypes.byref(o), ctypes.byref(h)) == -1
    assert L.fmm2d_build(None, 4, ctypes.byref(o), ctypes.byref(h)) == -1
    assert L.fmm2d_build(ctypes.c_void_p(z.ctypes.data), 4, None, ctypes.byref(h)) == -1
    assert L.fmm2d_eval(None, None, None, None) == -1
    L.fmm2d_free(None)                     # NULL-safe
    o.nranks = 2                           # a multi-rank build needs the shared NCCL id
    assert L.fmm2d_build(ctypes.c_void_p(z.ctypes.data), 4, ctypes.byref(o), ctypes.byref(h)) == -1
    nid = ctypes.create_string_buffer(128)
    o.nccl_id = ctypes.cast(nid, ctypes.c_void_p)
    o.nranks = 3                           # not a power of two: no level with 3 | 4^k
    assert L.fmm2d_build(ctypes.c_void_p(z.ctypes.data), 4, ctypes.byref(o), ctypes.byref(h)) == -6
    o.nranks = 2                           # n = 4: a one-level tree has nothing below k = 1
    assert L.fmm2d_build(ctypes.c_void_p(z.ctypes.data), 4, ctypes.byref(o), ctypes.byref(h)) == -6
    assert not h.value


def test_option_combinations_rejected_without_gpu():
    """Partitioned builds: the r/R exchange and the midpoint tree are one-GPU options
    (ENOTSUP, -6) -- checked before any device work."""
    import paper_1006_2269_b200 as F
    L = F.lib()
    z = np.zeros(1000, np.complex128)
    nid = ctypes.create_string_buffer(128)
    for flag in (F.fmm2d.RR_EXCHANGE, F.fmm2d.MIDPOINT):
        o = F.fmm2d.Options()
        L.fmm2d_default_options(ctypes.byref(o))
        o.nranks, o.rank, o.flags = 2, 0, flag
        o.nccl_id = ctypes.cast(nid, ctypes.c_void_p)
        h = ctypes.c_void_p()
        assert L.fmm2d_build(ctypes.c_void_p(z.ctypes.data), 1000, ctypes.byref(o), ctypes.byref(h)) == -6
        assert not h.value


def test_flag_values_match_header():
    import re
    import paper_1006_2269_b200 as F
    src = open(os.path.join(ROOT, "include", "fmm2d.h")).read()
    flags = {k: int(v, 16) for k, v in re.findall(r"#define FMM2D_(\w+)\s+(0x[0-9a-fA-F]+)", src)}
    for name in ("HOST_PTRS", "REAL_STRENGTHS", "SYMMETRIC_P2P", "TREE_KEY64", "TREE_GLOBAL_ONLY", "RR_EXCHANGE",
                 "PARENT_MERGE", "OVERLAP", "GATHER_OUTPUT", "MIDPOINT", "ASYNC_HOST"):
        assert getattr(F.fmm2d, name) == flags[name], name
    exports = {k: int(v) for k, v in re.findall(r"#define FMM2D_EXPORT_(\w+)\s+(\d+)", src)}
    for name, v in exports.items():
        assert getattr(F.fmm2d, "EXPORT_" + name) == v, name
