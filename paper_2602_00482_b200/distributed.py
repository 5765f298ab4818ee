"""Multi-GPU plumbing of the DFS step: one process per GPU, whole prefix trees
sharded across ranks by the min-max contiguous partitioner (partition_contiguous),
and the single gradient all-reduce per step (the reference reduces worker GradientStores in group
order on the host; here it is one in-place NCCL all-reduce over NVLink).

torch.distributed is used only as plumbing (process group, NCCL collective on a zero-copy view of
the engine's fp32 GradientStore)."""
from __future__ import annotations

from typing import List, Sequence

from . import TokenSequence, partition_contiguous


def shard_for_rank(seqs: Sequence[TokenSequence], rank: int, world: int) -> List[TokenSequence]:
    """The sequences (whole prefix trees) rank `rank` of `world` trains on."""
    if world <= 1:
        return list(seqs)
    plan = partition_contiguous(list(seqs), world)
    mine = set(plan["groups"][rank])
    return [s for s in seqs if s.seq_id in mine]


def grads_view(engine):
    """Zero-copy torch view (cuda, fp32) of the engine's flat GradientStore."""
    import torch

    ptr, n = engine.grads_device_ptr(), engine.n_params

    class _A:
        __cuda_array_interface__ = {"shape": (n,), "typestr": "<f4", "data": (ptr, False), "version": 3}

    return torch.as_tensor(_A(), device="cuda")


def allreduce_gradients(tensor, group=None) -> None:
    """Sum the per-rank GradientStores (in place)."""
    import torch.distributed as dist

    if dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(tensor, op=dist.ReduceOp.SUM, group=group)
