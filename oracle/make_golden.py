"""ORACLE — TEST INFRASTRUCTURE ONLY. Generates tests/golden/*.npz from the reference itself
(oracle/_ref/libttref.so, compiled from /root/reference by oracle/Makefile).

    python -m oracle.make_golden

Fixtures (all f64, the reference's T=double arithmetic):
  ref_small.npz : init_params(cfg, seed=7) (model.hpp:121-142); chained forward_segment logits and
                  KV (model.hpp:328); backward_segment grads + grad_prefix for a random upstream
                  (model.hpp:474); weighted_nll on uniform and random logits (model.hpp:643);
                  a DFS tree step over a grouped corpus executed with the reference arithmetic
                   — loss and gradients.
"""
from __future__ import annotations

import os

import numpy as np

from . import refimpl as R
from . import treetrain_oracle as O

OUT = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden")
CFG = O.ModelConfig(vocab_size=64, d_model=32, n_heads=4, n_layers=2, d_ff=64, max_position=256)


def corpus():
    return O.grouped_corpus(3, 4, 6, 9, CFG.vocab_size, 21, shared_response=2, weight_jitter=True)


def main():
    R.build()
    os.makedirs(OUT, exist_ok=True)
    flat = R.init_params(CFG, 7)
    rng = np.random.default_rng(1234)
    toks = rng.integers(0, CFG.vocab_size, 12).astype(np.int32)
    empty = np.zeros((CFG.n_layers, 0, CFG.d_model))
    la, ka, va = R.forward_segment(CFG, flat, empty, empty, toks[:5], 0)
    lb, kb, vb = R.forward_segment(CFG, flat, ka, va, toks[5:], 5)
    lfull, _, _ = R.forward_segment(CFG, flat, empty, empty, toks, 0)
    gl = rng.normal(size=lb.shape)
    gnk = rng.normal(size=kb.shape) * 0.1
    gnv = rng.normal(size=vb.shape) * 0.1
    g_b, gpk, gpv = R.backward_segment(CFG, flat, ka, va, toks[5:], 5, gl, gnk, gnv)
    uni_loss, _ = R.weighted_nll(np.zeros((4, CFG.vocab_size)), [1, 2, 3, 4], [1.0] * 4)
    rl = rng.normal(size=(6, CFG.vocab_size))
    rt = rng.integers(0, CFG.vocab_size, 6)
    rw = np.array([1.0, 0.0, 2.5, 1.0, 0.3, 0.0])
    nll_loss, nll_grad = R.weighted_nll(rl, rt, rw)
    seqs = corpus()
    root = O.order_children(O.build_prefix_tree(seqs), "subtree_tokens_desc")
    tree_loss, tree_grads = R.run_events(CFG, flat, R.EventList(root, seqs))
    np.savez_compressed(
        os.path.join(OUT, "ref_small.npz"),
        cfg=np.array([CFG.vocab_size, CFG.d_model, CFG.n_heads, CFG.n_layers, CFG.d_ff, CFG.max_position]),
        params=flat, tokens=toks, logits_a=la, logits_b=lb, logits_full=lfull, k_a=ka, v_a=va, k_b=kb, v_b=vb,
        grad_logits_b=gl, grad_new_k=gnk, grad_new_v=gnv, grads_b=g_b, grad_prefix_k=gpk, grad_prefix_v=gpv,
        uniform_loss=uni_loss, nll_logits=rl, nll_targets=rt, nll_weights=rw, nll_loss=nll_loss, nll_grad=nll_grad,
        tree_serialized=np.frombuffer(O.serialize_tree(root).encode(), dtype=np.uint8),
        tree_trace=np.frombuffer(O.dfs_trace(root).encode(), dtype=np.uint8),
        tree_loss=tree_loss, tree_grads=tree_grads)
    print("wrote", os.path.join(OUT, "ref_small.npz"))


if __name__ == "__main__":
    main()
