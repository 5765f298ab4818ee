"""Pins the numpy oracle to golden vectors produced by the reference itself (oracle/make_golden.py
runs the reference's forward_segment / backward_segment / weighted_nll / init_params compiled
from /root/reference). Needs no compiled code, so it runs anywhere."""
import os

import numpy as np
import pytest

from oracle import treetrain_oracle as O

GOLD = os.path.join(os.path.dirname(__file__), "golden", "ref_small.npz")


@pytest.fixture(scope="module")
def g():
    return np.load(GOLD)


def cfg_of(g):
    return O.ModelConfig(*[int(x) for x in g["cfg"]])


def test_forward_chain_matches_reference(g):
    cfg = cfg_of(g)
    P = O.unflatten(cfg, g["params"])
    toks = g["tokens"]
    empty = np.zeros((cfg.n_layers, 0, cfg.d_model))
    la, (ka, va), _ = O.forward_segment(cfg, P, empty, empty, toks[:5], 0)
    lb, (kb, vb), _ = O.forward_segment(cfg, P, ka, va, toks[5:], 5)
    for a, b in ((la, g["logits_a"]), (lb, g["logits_b"]), (ka, g["k_a"]), (vb, g["v_b"])):
        np.testing.assert_allclose(a, b, rtol=1e-12, atol=1e-14)
    # the reference's own KV-consistency property, as recorded: chained == monolithic
    np.testing.assert_array_equal(g["logits_b"], g["logits_full"][5:])


def test_backward_matches_reference(g):
    cfg = cfg_of(g)
    P = O.unflatten(cfg, g["params"])
    toks = g["tokens"]
    empty = np.zeros((cfg.n_layers, 0, cfg.d_model))
    _, (ka, va), _ = O.forward_segment(cfg, P, empty, empty, toks[:5], 0)
    _, _, acts = O.forward_segment(cfg, P, ka, va, toks[5:], 5)
    G = O.zero_like_params(cfg)
    gpk, gpv = O.backward_segment(cfg, P, acts, ka, va, G, g["grad_logits_b"], g["grad_new_k"], g["grad_new_v"])
    ref = g["grads_b"]
    got = O.flatten(cfg, G)
    assert np.abs(got - ref).max() <= 1e-12 * np.abs(ref).max()
    np.testing.assert_allclose(gpk, g["grad_prefix_k"], rtol=1e-10, atol=1e-14)
    np.testing.assert_allclose(gpv, g["grad_prefix_v"], rtol=1e-10, atol=1e-14)


def test_weighted_nll_matches_reference(g):
    V = int(g["cfg"][0])
    assert float(g["uniform_loss"]) == pytest.approx(4 * np.log(V), rel=1e-15)
    loss, grad = O.weighted_nll(g["nll_logits"], g["nll_targets"], g["nll_weights"])
    assert loss == pytest.approx(float(g["nll_loss"]), rel=1e-13)
    np.testing.assert_allclose(grad, g["nll_grad"], rtol=1e-12, atol=1e-15)


def test_tree_step_matches_reference(g):
    from oracle.make_golden import corpus

    cfg = cfg_of(g)
    seqs = corpus()
    root = O.order_children(O.build_prefix_tree(seqs), "subtree_tokens_desc")
    assert O.serialize_tree(root) == bytes(g["tree_serialized"]).decode()
    assert O.dfs_trace(root) == bytes(g["tree_trace"]).decode()
    r = O.tree_train_step(cfg, g["params"], root, seqs)
    assert r.total_loss == pytest.approx(float(g["tree_loss"]), rel=1e-12)
    assert O.compare_grads(r.grads, g["tree_grads"])[1] <= 1e-9
