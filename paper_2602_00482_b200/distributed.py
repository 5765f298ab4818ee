"""Multi-GPU DFS step: one process per GPU, whole prefix trees sharded across ranks by
the min-max contiguous partitioner (partition_contiguous), and ONE gradient
all-reduce per step. The reference reduces the workers' GradientStores in group order on the host
(SPEC.md:278); here each rank's engine runs its shard and the flat fp32 GradientStore is summed in
place by the engine's own NCCL communicator (tt_nccl_comm_init_rank / tt_grads_allreduce, on the
engine stream) — no torch tensor, no torch collective on the data path.

torch.distributed (any backend, gloo is enough) is only the rendezvous: it ships rank 0's 128-byte
ncclUniqueId to the other ranks. A C++ host does the same with its own launcher.
"""
from __future__ import annotations

from typing import List, Optional, Sequence

from . import Engine, NcclComm, SchedulerConfig, TokenSequence, build_prefix_tree, nccl_unique_id, partition_contiguous


def shard_for_rank(seqs: Sequence[TokenSequence], rank: int, world: int) -> List[TokenSequence]:
    """The sequences (whole prefix trees) rank `rank` of `world` trains on."""
    if world <= 1:
        return list(seqs)
    plan = partition_contiguous(list(seqs), world)
    mine = set(plan["groups"][rank])
    return [s for s in seqs if s.seq_id in mine]


def exchange_unique_id(rank: int, group=None) -> bytes:
    """Rank 0's ncclGetUniqueId, broadcast over the torch.distributed rendezvous."""
    import torch.distributed as dist

    box = [nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(box, src=0, group=group)
    uid = box[0]
    if not isinstance(uid, (bytes, bytearray)) or len(uid) != 128:
        raise RuntimeError("exchange_unique_id: malformed NCCL unique id")
    return bytes(uid)


class DataParallel:
    """One rank of the data-parallel DFS step: its tree shard, its engine, its NCCL communicator.

    step() = zero the GradientStore, run the rank's prepared plan (tree_train_step), then the single
    in-place NCCL sum all-reduce; every rank ends with the gradient of the whole batch, which equals
    the dense gradient over all sequences."""

    def __init__(self, engine: Engine, rank: int, world: int, device: int, group=None,
                 comm: Optional[NcclComm] = None):
        self.engine, self.rank, self.world = engine, rank, world
        self.comm = comm
        if self.comm is None and world > 1:
            self.comm = NcclComm(exchange_unique_id(rank, group), world, rank, device)
        self._plan = None

    def shard(self, seqs: Sequence[TokenSequence]) -> List[TokenSequence]:
        return shard_for_rank(seqs, self.rank, self.world)

    def prepare(self, seqs: Sequence[TokenSequence], sched: Optional[SchedulerConfig] = None):
        """Build + plan the rank's shard once (metadata resident in HBM); step() replays it."""
        self._plan = self.engine.plan(build_prefix_tree(self.shard(seqs)), sched or SchedulerConfig())
        return self._plan

    def allreduce(self) -> None:
        if self.comm is not None:
            self.engine.allreduce_gradients(self.comm)

    def step(self):
        if self._plan is None:
            raise RuntimeError("DataParallel.step: call prepare() first")
        self.engine.zero_gradients()
        r = self._plan.execute()
        self.allreduce()
        return r

    def close(self):
        if self.comm is not None:
            self.comm.close()
            self.comm = None
