"""Multi-GPU data-parallel DFS step through the engine's own NCCL communicator (SURVEY §8(e),
SPEC.md:278): whole trees sharded by partition_contiguous, each rank's tree step, ONE in-place
ncclAllReduce of the GradientStore (tt_grads_allreduce). The summed gradient must equal the dense
oracle over all sequences within the engine tolerances.

The one-rank case runs on any GPU box; the two-rank case needs two GPUs and is skipped otherwise
(the host logic of N > 1 is covered on CPU by tests/test_distributed_cpu.py)."""
import os
import socket

import numpy as np
import pytest

import paper_2602_00482_b200 as tt
from oracle import treetrain_oracle as O

from test_engine_gpu import GRAD_TOL, LOSS_TOL, SMALL, check_grads

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu


def _corpus(cfg):
    return O.grouped_corpus(6, 4, 40, 30, cfg.vocab_size, 61, shared_response=3, weight_jitter=True)


def _tt(seqs):
    return [tt.TokenSequence(s.seq_id, s.tokens, s.weights) for s in seqs]


def test_data_parallel_single_rank_nccl():
    from paper_2602_00482_b200.distributed import DataParallel

    cfg = O.ModelConfig(*SMALL)
    flat = O.round_bf16(O.random_params(cfg, 3))
    seqs = _corpus(cfg)
    eng = tt.Engine(tt.ModelConfig(*SMALL))
    eng.upload_params(flat)
    dp = DataParallel(eng, 0, 1, 0, comm=tt.NcclComm(tt.nccl_unique_id(), 1, 0, 0))
    dp.prepare(_tt(seqs))
    r = dp.step()
    got = eng.gradients()
    d = O.dense_train_step(cfg, flat, seqs)
    assert abs(r.total_loss - d.total_loss) <= LOSS_TOL * abs(d.total_loss)
    check_grads(cfg, got, d.grads)
    # replaying the step gives the same result (plan resident, all-reduce identity at one rank)
    r2 = dp.step()
    assert abs(r2.total_loss - r.total_loss) <= 1e-9 * abs(r.total_loss)
    assert np.allclose(eng.gradients(), got, rtol=0, atol=1e-5 * np.abs(got).max())
    dp.close()
    eng.close()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out):
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2602_00482_b200.distributed import DataParallel

    cfg = O.ModelConfig(*SMALL)
    flat = O.round_bf16(O.random_params(cfg, 3))
    seqs = _corpus(cfg)
    eng = tt.Engine(tt.ModelConfig(*SMALL), device=rank)
    eng.upload_params(flat)
    dp = DataParallel(eng, rank, world, rank)
    dp.prepare(_tt(seqs))
    r = dp.step()
    loss = torch.tensor([r.total_loss], dtype=torch.float64)
    dist.all_reduce(loss)
    g = eng.gradients()
    if rank == 0:
        out["grads"] = g
        out["loss"] = float(loss.item())
    else:
        out["grads1"] = g
    dp.close()
    eng.close()
    dist.destroy_process_group()


@pytest.mark.skipif(not torch.cuda.is_available() or torch.cuda.device_count() < 2, reason="needs 2 GPUs")
def test_data_parallel_two_ranks_nccl_equals_dense():
    import torch.multiprocessing as mp

    out = mp.Manager().dict()
    mp.spawn(_worker, args=(2, _free_port(), out), nprocs=2, join=True)
    cfg = O.ModelConfig(*SMALL)
    flat = O.round_bf16(O.random_params(cfg, 3))
    d = O.dense_train_step(cfg, flat, _corpus(cfg))
    assert abs(out["loss"] - d.total_loss) <= LOSS_TOL * abs(d.total_loss)
    check_grads(cfg, out["grads"], d.grads, tol=GRAD_TOL)
    assert np.array_equal(out["grads"], out["grads1"])  # every rank holds the same summed gradient
