"""World-size-2 gloo run of the multi-GPU host logic (no GPU): shard whole trees with the native
partition_contiguous, run each rank's tree step (CPU oracle as the stand-in worker), all-reduce the
GradientStores, and check the result equals the dense oracle over all sequences.
Also checks the NCCL unique-id rendezvous every rank's engine communicator is built from
(paper_2602_00482_b200.distributed.exchange_unique_id: rank 0's ncclGetUniqueId over gloo)."""
import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402

CFG = (64, 32, 4, 2, 64, 256)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_2602_00482_b200 as tt
    from paper_2602_00482_b200.distributed import exchange_unique_id, shard_for_rank
    from oracle import treetrain_oracle as O

    cfg = O.ModelConfig(*CFG)
    flat = O.random_params(cfg, 5)
    seqs = O.grouped_corpus(6, 4, 5, 8, cfg.vocab_size, 17, shared_response=2, weight_jitter=True)
    mine = shard_for_rank([tt.TokenSequence(s.seq_id, s.tokens, s.weights) for s in seqs], rank, world)
    ids = {s.seq_id for s in mine}
    local = [s for s in seqs if s.seq_id in ids]
    root = O.order_children(O.build_prefix_tree(local), "subtree_tokens_desc")
    r = O.tree_train_step(cfg, flat, root, local)
    uid = torch.frombuffer(bytearray(exchange_unique_id(rank)), dtype=torch.uint8).to(torch.int64)
    uid_max, uid_min = uid.clone(), uid.clone()
    dist.all_reduce(uid_max, op=dist.ReduceOp.MAX)
    dist.all_reduce(uid_min, op=dist.ReduceOp.MIN)
    g = torch.from_numpy(r.grads.copy())
    loss = torch.tensor([r.total_loss], dtype=torch.float64)
    dist.all_reduce(g)  # the CPU stand-in for the engine's ncclAllReduce of the GradientStore
    dist.all_reduce(loss)
    n_local = torch.tensor([len(local)])
    dist.all_reduce(n_local)
    if rank == 0:
        out["uid_same"] = bool(torch.equal(uid_max, uid_min)) and int(uid.abs().sum()) > 0
        d = O.dense_train_step(cfg, flat, seqs)
        out["rel"] = O.compare_grads(g.numpy(), d.grads)[1]
        out["loss"] = (loss.item(), d.total_loss)
        out["n"] = int(n_local.item())
        out["N"] = len(seqs)
    dist.destroy_process_group()


def test_two_rank_shard_and_allreduce_equals_dense():
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(2, _free_port(), out), nprocs=2, join=True)
    assert out["uid_same"]  # every rank holds rank 0's NCCL unique id
    assert out["n"] == out["N"]  # shards cover every sequence exactly once
    assert out["rel"] <= 1e-8
    a, b = out["loss"]
    assert abs(a - b) <= 1e-10 * abs(b)
