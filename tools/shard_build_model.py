"""Per-rank build cost of the partitioned pass, measured rank by rank on ONE GPU with the
loopback transport (each rank's tree stage runs alone, CUDA events): the replicated part
(selection of the top split records, level-k boxes) plus the rank's own presort and levels.
Compared with the one-GPU build of the same instance.

    python tools/shard_build_model.py [--config C5] [--ranks 8]
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
    ap.add_argument("--ranks", type=int, default=8)
    args = ap.parse_args()
    import torch
    from paper_1006_2269_b200 import Fmm2d, LoopbackShards
    c = W.CONFIGS[args.config]
    z_np, m_np = W.make_config(args.config)
    z = torch.from_numpy(z_np).cuda()
    one = []
    for _ in range(3):
        p = Fmm2d(z, theta=c.theta, p=c.p, leaf_target=c.leaf_target, real_strengths=True)
        one.append(p.stats()["t_tree_ms"] + p.stats()["t_lists_ms"])
        p.close()
    # twice: the first build of the loopback set grows the memory pool (all ranks' plans
    # live at once); the second reuses it, as a rank's repeated builds do
    for _ in range(2):
        sh = LoopbackShards(z, args.ranks, theta=c.theta, p=c.p, leaf_target=c.leaf_target, real_strengths=True)
        per = [s.stats()["t_tree_ms"] for s in sh.shards]
        sh.close()
    out = {"config": args.config, "ranks": args.ranks, "one_gpu_build_ms": min(one),
           "per_rank_tree_stage_ms": per, "note": "tree stage only (lists + halo set-up of a rank are not in t_tree_ms)"}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
