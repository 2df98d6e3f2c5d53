"""Probe: device-resident C5 problems, one at a time vs NF in flight on NF streams
(fmm2d_build_eval with device pointers; the build of problem k+1 runs while problem k is
evaluated).  Prints device ms per problem.  (Experiment only.)"""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import workloads as W  # noqa: E402
from paper_1006_2269_b200 import Fmm2d, reserve_pool  # noqa: E402

cfg = W.CONFIGS["C5"]
z_np, m_np = W.make_config("C5")
dev = torch.device("cuda", 0)
z = torch.from_numpy(z_np).to(dev)
m = torch.from_numpy(m_np).to(dev)
kw = dict(theta=cfg.theta, p=cfg.p, leaf_target=cfg.leaf_target, real_strengths=True)
free, _ = torch.cuda.mem_get_info()
reserve_pool(int(0.5 * free))
for NF in (1, 2, 3):
    streams = [torch.cuda.Stream() for _ in range(NF)]
    outs = [(torch.empty(cfg.n, dtype=torch.complex128, device=dev),
             torch.empty(cfg.n, dtype=torch.complex128, device=dev)) for _ in range(NF)]
    inflight = []

    def step(k):
        o = outs[k % NF]
        with torch.cuda.stream(streams[k % NF]):
            plan = Fmm2d.build_eval(z, m, o[0], o[1], stream=streams[k % NF], **kw)[0]
        inflight.append((plan, streams[k % NF]))
        if len(inflight) > NF - 1:
            p, s = inflight.pop(0)
            s.synchronize()
            p.close()

    for k in range(NF + 2):
        step(k)
    while inflight:
        p, s = inflight.pop(0)
        s.synchronize()
        p.close()
    torch.cuda.synchronize()
    steps = 10
    t0 = time.perf_counter()
    for k in range(steps):
        step(k)
    while inflight:
        p, s = inflight.pop(0)
        s.synchronize()
        p.close()
    torch.cuda.synchronize()
    ms = (time.perf_counter() - t0) * 1e3 / steps
    print(f"NF={NF}: {ms:.2f} ms per problem ({cfg.n / ms * 1e3:.3e} points/s)", flush=True)
