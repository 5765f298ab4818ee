"""The whole DFS step driven from C++ through the header-only wrapper (include/treetrain_b200.hpp)
on the GPU, without Python or PyTorch in the process (tests/cpp/engine_demo.cpp): a prepared plan
(execute, execute_async overlapped with the next plan's preparation), a one-rank NCCL all-reduce, a
segment-level DFS over a 3-segment chain with the loss on the device, and weighted_nll. Results are
compared with the f64 oracle under the engine tolerances (tests/test_engine_gpu.py)."""
import os
import subprocess

import numpy as np
import pytest

from oracle import treetrain_oracle as O
from paper_2602_00482_b200 import _native

from test_engine_gpu import LOSS_TOL, SMALL, check_grads

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_cpp_engine_step_chain_nccl_nll(tmp_path):
    exe = str(tmp_path / "engine_demo")
    libdir = os.path.dirname(_native.LIB_PATH)
    r = subprocess.run(["g++", "-std=c++17", "-O1", "-I", os.path.join(ROOT, "include"),
                        os.path.join(ROOT, "tests", "cpp", "engine_demo.cpp"), "-L", libdir, "-ltreetrain_b200",
                        f"-Wl,-rpath,{libdir}", "-o", exe], capture_output=True, text=True)
    if r.returncode != 0:
        pytest.fail(r.stderr)
    cfg = O.ModelConfig(*SMALL)
    flat = O.round_bf16(O.random_params(cfg, 71))
    seqs = O.grouped_corpus(2, 3, 40, 30, cfg.vocab_size, 72, weight_jitter=True)
    inp = str(tmp_path / "in.bin")
    with open(inp, "wb") as f:
        np.array([cfg.vocab_size, cfg.d_model, cfg.n_heads, cfg.n_layers, cfg.d_ff, cfg.max_position, flat.size,
                  len(seqs)], dtype=np.uint64).tofile(f)
        flat.astype(np.float64).tofile(f)
        for s in seqs:
            np.array([len(s.tokens)], dtype=np.uint64).tofile(f)
            np.asarray(s.tokens, dtype=np.int32).tofile(f)
            np.asarray(s.weights, dtype=np.float64).tofile(f)
    out = str(tmp_path / "out")
    res = subprocess.run([exe, inp, out], capture_output=True, text=True, timeout=600)
    assert res.returncode == 0, res.stderr
    lines = dict(ln.split(" ", 1) for ln in res.stdout.strip().splitlines())
    # 1. tree step through the plan (sync and async) + one-rank all-reduce
    ref = O.tree_train_step(cfg, flat, O.order_children(O.build_prefix_tree(seqs), "subtree_tokens_desc"), seqs)
    l1, l2 = (float(x) for x in lines["TREE"].split())
    assert abs(l1 - ref.total_loss) <= LOSS_TOL * abs(ref.total_loss)
    assert abs(l2 - l1) <= 1e-9 * abs(l1)
    check_grads(cfg, np.fromfile(out + ".grads1", dtype=np.float64), ref.grads)
    # 2. the first sequence as a 3-segment chain == its own tree step (chained == monolithic)
    s0 = seqs[0]
    ref0 = O.tree_train_step(cfg, flat, O.order_children(O.build_prefix_tree([s0]), "subtree_tokens_desc"), [s0])
    lc = float(lines["CHAIN"])
    assert abs(lc - ref0.total_loss) <= LOSS_TOL * abs(ref0.total_loss)
    check_grads(cfg, np.fromfile(out + ".grads2", dtype=np.float64), ref0.grads)
    # 3. weighted_nll (model.hpp:643-677) vs the oracle's
    V = cfg.vocab_size
    logits = (0.001 * (np.arange(2 * V) % 97)).astype(np.float32).reshape(2, V)
    lref, gref = O.weighted_nll(logits.astype(np.float64), [3, 5], [1.0, 0.5])
    ln_, g3 = (float(x) for x in lines["NLL"].split())
    assert abs(ln_ - lref) <= 1e-5 * abs(lref)
    assert abs(g3 - gref[0, 3]) <= 1e-5
    assert lines["INVALID_ARGUMENT"].strip()
