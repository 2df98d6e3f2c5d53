"""Host logic of the partitioned pass (no GPU): partition facts against the oracle's
tree, and the torch.distributed plumbing with world_size 2 over gloo on CPU."""
import os

import numpy as np
import pytest

import workloads as W


@pytest.mark.parametrize("n,P", [(1000, 2), (100_000, 4), (100_000, 8), (7777, 16), (54_321, 8)])
def test_partition_matches_oracle_offsets(orc, n, P):
    """Own positions = the oracle tree's offsets of the own level-k subtrees; own leaves
    = [r 4^L/P, (r+1) 4^L/P); the ranks tile [0, n) and the leaves without overlap."""
    from paper_1006_2269_b200 import partition_info
    z, _ = W.make("uniform", n, seed=n)
    L = orc.nlevels(n, 35)
    op = orc.plan(z, 0.5, L)
    k = partition_info(n, P, 0, nlevels=L)["k"]
    assert 4 ** k % P == 0 and (k == 0 or 4 ** (k - 1) % P != 0)
    off_k = op.offsets(k)
    pos, lv = [], []
    for r in range(P):
        i = partition_info(n, P, r, nlevels=L)
        assert i["L"] == L and i["k"] == k
        s0, s1 = i["subtrees"]
        assert (s0, s1) == (4 ** k // P * r, 4 ** k // P * (r + 1))
        assert i["positions"] == (off_k[s0], off_k[s1])
        assert i["leaves"] == (4 ** L // P * r, 4 ** L // P * (r + 1))
        pos.append(i["positions"])
        lv.append(i["leaves"])
    assert pos[0][0] == 0 and pos[-1][1] == n and lv[-1][1] == 4 ** L
    assert all(a[1] == b[0] for a, b in zip(pos, pos[1:]))
    assert all(a[1] == b[0] for a, b in zip(lv, lv[1:]))
    sizes = [b - a for a, b in pos]
    assert max(sizes) - min(sizes) <= 4 ** k // P       # equal counts up to 1 per level-k box


def _worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1006_2269_b200.dist import my_partition, shared_nccl_id
        nid = shared_nccl_id()
        part = my_partition(1_000_000)
        out = [None] * world
        dist.all_gather_object(out, (nid, part))
        q.put((rank, out))
    finally:
        dist.destroy_process_group()


def test_dist_plumbing_gloo_world2():
    """Two CPU processes (gloo): both ranks get the same NCCL unique id from rank 0, and
    their partitions tile the problem."""
    import multiprocessing as mp
    import socket
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for r in (0, 1):
        (id0, p0), (id1, p1) = res[r]
        assert id0 == id1 and len(id0) == 128
        assert p0["positions"][0] == 0 and p0["positions"][1] == p1["positions"][0]
        assert p1["positions"][1] == 1_000_000
    assert res[0] == res[1]


def test_bench_gpus_without_devices_fails_loudly():
    """`bench.py --gpus N` spawns N ranks itself (torch.distributed.run) when no launcher
    did; with fewer than N devices it must fail with a message, never time one GPU."""
    import subprocess
    import sys
    import torch
    if torch.cuda.device_count() >= 2:
        pytest.skip("this host has >= 2 GPUs")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--gpus", "2", "--steps", "1"],
                       capture_output=True, text=True, timeout=300)
    assert r.returncode == 2 and "needs 2 CUDA devices" in r.stderr, (r.returncode, r.stderr[-500:])
    r = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--gpus", "2", "--steps", "1"],
                       capture_output=True, text=True, timeout=300, env=dict(os.environ, WORLD_SIZE="1"))
    assert r.returncode != 0 and "WORLD_SIZE=1" in r.stderr
