"""Device memory per rank of the partitioned pass: every rank of a
loopback build on ONE GPU, built one after the other; per rank the bytes its plan holds
after the build (stats dev_bytes: perm / rows / expansions of the OWN positions and boxes,
halo stores, lists, discs) and the library pool's high-water mark while that rank's build
ran alone (the transient tree scratch included), against the one-GPU plan of the same
instance.

    python tools/shard_memory.py [--config C5] > profiles/r02/shard_memory.json
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import workloads as W  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C5")
    args = ap.parse_args()
    import torch
    from paper_1006_2269_b200 import Fmm2d, LoopbackShards, pool_usage
    c = W.CONFIGS[args.config]
    z_np, m_np = W.make_config(args.config)
    z = torch.from_numpy(z_np).cuda()
    out = {"config": args.config, "n": c.n, "note": "input z (16 B/pt) and m (16 B/pt) are the caller's, not counted"}
    torch.cuda.synchronize()
    pool_usage(reset=True)
    one = Fmm2d(z, theta=c.theta, p=c.p, leaf_target=c.leaf_target, real_strengths=True)
    torch.cuda.synchronize()
    out["one_gpu"] = {"plan_bytes": one.stats()["dev_bytes"], "build_high_water_bytes": pool_usage()[1]}
    one.close()
    for P in (2, 4, 8):
        pool_usage(reset=True)
        sh = LoopbackShards(z, P, theta=c.theta, p=c.p, leaf_target=c.leaf_target, real_strengths=True)
        torch.cuda.synchronize()
        per = [s.stats()["dev_bytes"] for s in sh.shards]
        out[f"P{P}"] = {"plan_bytes_per_rank": per, "max_plan_bytes": max(per),
                        "all_ranks_high_water_bytes": pool_usage()[1],
                        "note": "high water covers ALL ranks' plans (loopback: every rank on this GPU)"}
        sh.close()
    print(json.dumps(out))


if __name__ == "__main__":
    main()
