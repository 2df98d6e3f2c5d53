"""Accuracy of the product's table-driven FP64 log|z|, Arg z and reciprocals (fastmath.cuh),
built for the host and compared with long double over 4e6 random arguments spanning
2^+-60 and the axes / diagonal.  (The device build differs only in the MUFU reciprocal
estimate, which one cubic Newton step makes irrelevant; GPU parity tests cover it.)"""
import json
import os
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(tmp_path, *flags):
    exe = tmp_path / "test_fastmath"
    subprocess.check_call(["g++", "-O2", "-ffp-contract=off", *flags, "-o", str(exe),
                           os.path.join(ROOT, "tools", "test_fastmath.cpp")])
    return json.loads(subprocess.check_output([str(exe)]).decode())


def test_fastmath_ulps(tmp_path):
    r = _run(tmp_path)
    assert r["n"] > 3_000_000
    assert r["log_max_ulp"] <= 2.0
    assert r["log_max_abs"] <= 1e-14          # |log|dz|| up to ~42 here: < 1 ulp
    assert r["arg_max_ulp"] <= 2.0
    assert r["argneg_max_ulp"] <= 2.0 and r["pair_mismatch"] == 0   # Arg(-dz) of arg_pair (symmetric P2P)
    assert r["log0_is_neg_inf"] == 1 and r["arg_pi"] == 1 and r["arg_zero"] == 1
    # near-field log (k_near): each term enters Phi with its ABSOLUTE error, so the bar is
    # in units of eps = 2^-52 of max(1, |value|)
    assert r["log5_max_abs_eps"] <= 1.0           # degree-5 log1p, |u| < 2^-9
    # near-field Arg (arg_n: coarse reciprocal + one correction, single-double atan table): absolute
    # error in the same units, and small angles keep a relative error far below the 1e-12 parity bar
    assert r["argn_max_abs_eps"] <= 2.0 and r["argn_max_rel"] <= 2e-13


def test_fastmath_near_field_worst_case_reciprocal(tmp_path):
    """The device's reciprocal estimate (MUFU.RCP64H) is only ~2^-22 accurate; the host stand-in
    is perturbed by +-2^-22 on top of its float rounding, and by the replicated-table layout."""
    for sign in ("(1.0)", "(-1.0)"):
        r = _run(tmp_path, f"-DFM_HOST_RCP_PERTURB={sign}", "-DFMM2D_NEAR_RL=2", "-DFMM2D_NEAR_RA=4")
        assert r["argn_max_abs_eps"] <= 2.0 and r["argn_max_rel"] <= 2e-13
        assert r["log5_max_abs_eps"] <= 1.0 and r["pair_mismatch"] == 0
        assert r["log_max_ulp"] <= 2.0 and r["arg_max_ulp"] <= 2.0
