"""Accuracy of the product's table-driven FP64 log|z|, Arg z and reciprocals (fastmath.cuh),
built for the host and compared with long double over 4e6 random arguments spanning
2^+-60 and the axes / diagonal.  (The device build differs only in the MUFU reciprocal
estimate, which one cubic Newton step makes irrelevant; GPU parity tests cover it.)"""
import json
import os
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_fastmath_ulps(tmp_path):
    exe = tmp_path / "test_fastmath"
    subprocess.check_call(["g++", "-O2", "-ffp-contract=off", "-o", str(exe),
                           os.path.join(ROOT, "tools", "test_fastmath.cpp")])
    r = json.loads(subprocess.check_output([str(exe)]).decode())
    assert r["n"] > 3_000_000
    assert r["log_max_ulp"] <= 2.0
    assert r["log_max_abs"] <= 1e-14          # |log|dz|| up to ~42 here: < 1 ulp
    assert r["arg_max_ulp"] <= 2.0
    assert r["argneg_max_ulp"] <= 2.0 and r["pair_mismatch"] == 0   # Arg(-dz) of arg_pair (symmetric P2P)
    assert r["log0_is_neg_inf"] == 1 and r["arg_pi"] == 1 and r["arg_zero"] == 1
    # near-field log (k_near): each term enters Phi with its ABSOLUTE error, so the bar is
    # in units of eps = 2^-52 of max(1, |value|)
    assert r["log5_max_abs_eps"] <= 1.0           # degree-5 log1p, |u| < 2^-9
