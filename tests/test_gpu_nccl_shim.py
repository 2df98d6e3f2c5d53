"""The NCCL transport of the partitioned pass (shard.cu) executed by
several PROCESSES, one rank each, as the multi-GPU bench runs it -- on the one GPU this
environment has.  Real NCCL refuses two ranks on one device, so libfmm2d.so loads the test
shim tests/ncclshim (NCCL's ten entry points over CUDA IPC staging buffers and host
barriers; FMM2D_NCCL_LIB) instead of libnccl.so.2.  The library code is unchanged: the
communicator set-up, the in-place all-gathers of discs and level-k multipoles, the max /
sum all-reduces of the top-level selection, the grouped send/recv of the halo id lists,
leaf rows and multipoles, and the output all-reduce of FMM2D_GATHER_OUTPUT all run.

Bar: the union of the ranks' outputs equals the one-GPU result BIT FOR BIT (each own box
sees the one-GPU lists, multipoles and locals in the same order), for every evaluation of
a reused plan and for a second plan on the same communicator.
"""
import os
import subprocess
import sys
import tempfile

import numpy as np
import pytest
import torch

import workloads as W

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SHIM = os.path.join(ROOT, "tests", "ncclshim", "libncclshim.so")

CHILD = r"""
import ctypes, sys
import numpy as np, torch
sys.path.insert(0, sys.argv[1])
import workloads as W
from paper_1006_2269_b200 import Fmm2d
root, cfg, n, P, r, idhex, out, gather, pm = sys.argv[1:10]
n, P, r, gather, pm = int(n), int(P), int(r), int(gather), int(pm)
c = W.CONFIGS[cfg]
z, m = W.make_config(cfg, n=n)
zt, mt = torch.from_numpy(z).cuda(), torch.from_numpy(m).cuda()
res = {}
for build in range(2):                      # the second plan reuses the cached communicator
    plan = Fmm2d(zt, theta=c.theta, p=c.p, leaf_target=35, real_strengths=(c.strengths == "real"),
                 nranks=P, rank=r, nccl_id=bytes.fromhex(idhex), gather_output=bool(gather),
                 parent_merge=bool(pm))
    for k in range(2):                      # plan reuse
        phi = torch.zeros(n, dtype=torch.complex128, device="cuda")
        dphi = torch.zeros(n, dtype=torch.complex128, device="cuda")
        plan.eval(mt, phi, dphi)
        torch.cuda.synchronize()
        res[f"phi{build}{k}"] = phi.cpu().numpy()
        res[f"dphi{build}{k}"] = dphi.cpu().numpy()
    h = plan.halo_info()
    res["halo"] = np.array([h["import_leaves"], h["import_mpoles"], h["export_leaves"], h["export_mpoles"],
                            h["positions"][0], h["positions"][1], h["k"]], np.int64)
    plan.close()
shim = ctypes.CDLL(__import__("os").environ["FMM2D_NCCL_LIB"])
shim.ncclShimCallCount.restype = ctypes.c_long
res["calls"] = np.array([shim.ncclShimCallCount()])
np.savez(out, **res)
"""


def _run_ranks(cfg, n, P, gather=False, pm=False):
    assert os.path.exists(SHIM), "build the shim with `make` (tests/ncclshim)"
    idhex = (os.urandom(8).hex().encode() + bytes(128 - 16)).hex()   # 16 hex characters, zero padded
    env = dict(os.environ, FMM2D_NCCL_LIB=SHIM, FMM2D_NCCLSHIM_MB="128")
    with tempfile.TemporaryDirectory() as td:
        procs, outs = [], []
        for r in range(P):
            out = os.path.join(td, f"r{r}.npz")
            outs.append(out)
            procs.append(subprocess.Popen([sys.executable, "-c", CHILD, ROOT, cfg, str(n), str(P), str(r), idhex, out,
                                           str(int(gather)), str(int(pm))], env=env, stdout=subprocess.PIPE,
                                          stderr=subprocess.STDOUT, text=True))
        logs = []
        for p in procs:
            try:
                logs.append(p.communicate(timeout=600)[0])
            except subprocess.TimeoutExpired:
                for q in procs:
                    q.kill()
                raise
        for p, log in zip(procs, logs):
            assert p.returncode == 0, log[-3000:]
        return [dict(np.load(o)) for o in outs]


def _one_gpu(cfg, n, pm=False):
    from paper_1006_2269_b200 import Fmm2d
    c = W.CONFIGS[cfg]
    z, m = W.make_config(cfg, n=n)
    plan = Fmm2d(torch.from_numpy(z).cuda(), theta=c.theta, p=c.p, leaf_target=35,
                 real_strengths=(c.strengths == "real"), parent_merge=pm)
    phi, dphi = plan.eval(torch.from_numpy(m).cuda())
    torch.cuda.synchronize()
    return plan.perm(), phi.cpu().numpy(), dphi.cpu().numpy()


@pytest.mark.parametrize("cfg,n,P,pm", [("C2", 100_000, 2, False), ("C3", 200_000, 4, False),
                                        ("C1", 1000, 2, False), ("C2", 60_000, 4, True)])
def test_nccl_transport_multiprocess_bit_identical(cfg, n, P, pm):
    perm, phi1, dphi1 = _one_gpu(cfg, n, pm)
    res = _run_ranks(cfg, n, P, pm=pm)
    covered = np.zeros(n, bool)
    for r, R in enumerate(res):
        pos0, pos1 = int(R["halo"][4]), int(R["halo"][5])
        own = perm[pos0:pos1]
        assert not covered[own].any()
        covered[own] = True
        for b in range(2):
            for k in range(2):
                np.testing.assert_array_equal(R[f"phi{b}{k}"][own], phi1[own])
                np.testing.assert_array_equal(R[f"dphi{b}{k}"][own], dphi1[own])
        assert R["calls"][0] > 0                        # the shim (NCCL entry points) was used
        if P > 1:
            assert R["halo"][0] > 0 and R["halo"][1] > 0   # halo leaves and multipoles imported
    assert covered.all()


def test_nccl_transport_gather_output():
    """FMM2D_GATHER_OUTPUT: the sum all-reduce completes Phi, Phi' on every rank."""
    perm, phi1, dphi1 = _one_gpu("C2", 50_000)
    for R in _run_ranks("C2", 50_000, 2, gather=True):
        np.testing.assert_array_equal(R["phi00"], phi1)
        np.testing.assert_array_equal(R["dphi11"], dphi1)
