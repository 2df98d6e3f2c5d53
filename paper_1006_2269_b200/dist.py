"""torch.distributed plumbing of the partitioned pass.

One process per GPU.  All ranks hold the same full inputs; the library partitions the
tree by the balanced level-k subtrees and moves halo data with NCCL itself.  This
module only agrees on the NCCL unique id (made by rank 0, broadcast through the
process group -- gloo or nccl) and reads rank / world size from the group.

    import torch.distributed as dist
    from paper_1006_2269_b200.dist import sharded_plan
    plan = sharded_plan(z, theta=0.5, p=17)      # collective; z: full complex128 CUDA tensor
    phi, dphi = plan.eval(m)                     # collective; own entries written
"""
from __future__ import annotations

from .fmm2d import Fmm2d, nccl_unique_id, partition_info


def shared_nccl_id(group=None) -> bytes:
    """Rank 0 of `group` creates a NCCL unique id; every rank returns the same 128 bytes."""
    import torch.distributed as dist
    obj = [nccl_unique_id() if dist.get_rank(group) == 0 else None]
    dist.broadcast_object_list(obj, src=dist.get_global_rank(group, 0) if group is not None else 0, group=group)
    return obj[0]


def my_partition(n: int, group=None, **kw) -> dict:
    """This rank's share of the tree (host arithmetic; no GPU needed)."""
    import torch.distributed as dist
    return partition_info(n, dist.get_world_size(group), dist.get_rank(group), **kw)


def sharded_plan(z, group=None, nccl_id: bytes | None = None, **kw) -> Fmm2d:
    """Collective build of this rank's part of the partitioned plan (one GPU per rank).
    The library keeps one NCCL communicator per id: pass the same `nccl_id` (from
    shared_nccl_id) to every build of a job to reuse it; None makes a new one."""
    import torch.distributed as dist
    world, rank = dist.get_world_size(group), dist.get_rank(group)
    if world == 1:
        return Fmm2d(z, **kw)
    if nccl_id is None:
        nccl_id = shared_nccl_id(group)
    return Fmm2d(z, nranks=world, rank=rank, nccl_id=nccl_id, **kw)
