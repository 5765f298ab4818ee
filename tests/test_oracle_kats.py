"""Known-answer tests of the CPU oracle against the reference SPEC's own examples.

The oracle is test infrastructure; these pin it before it is used to judge the CUDA path.
"""
import math

import numpy as np
import pytest

from oracle import treetrain_oracle as O

CFG = O.ModelConfig(vocab_size=64, d_model=32, n_heads=4, n_layers=2, d_ff=64, max_position=256)


def seqs_of(token_lists, weights=None):
    return [O.TokenSequence(i, list(t), list(weights[i]) if weights else [1.0] * len(t)) for i, t in enumerate(token_lists)]


def test_build_examples():
    # SPEC.md:138
    root = O.build_prefix_tree(seqs_of([[1, 2, 3], [1, 2, 4]]))
    assert [c.tokens for c in root.children] == [[1, 2]]
    assert [c.tokens for c in root.children[0].children] == [[3], [4]]
    assert O.tree_token_count(root) == 4
    # SPEC.md:139
    root = O.build_prefix_tree(seqs_of([[1, 2], [1, 2, 9]]))
    n = root.children[0]
    assert n.tokens == [1, 2] and n.leaf_marks == [0] and [c.tokens for c in n.children] == [[9]]
    assert O.tree_token_count(root) == 3


def test_group_count_and_dup_factor():
    # SPEC.md:149 (P + G*R), :175-176
    P, R, G = 7, 5, 8
    rng = np.random.default_rng(0)
    prompt = rng.integers(0, 50, P).tolist()
    seqs = seqs_of([prompt + [50 + g] + rng.integers(0, 50, R - 1).tolist() for g in range(G)])
    assert O.tree_token_count(O.build_prefix_tree(seqs)) == P + G * R
    assert O.duplication_factor(seqs_of([[1, 2, 3], [1, 2, 4]])) == pytest.approx(1.5)
    P = R = 6
    seqs = seqs_of([prompt[:6] + [50 + g] + [1] * 5 for g in range(8)])
    assert O.duplication_factor(seqs) == pytest.approx(16 / 9)
    assert O.duplication_factor(seqs_of([[1], [2, 3], [4]])) == 1.0


def test_order_children_desc_and_ties():
    # subtree tokens {5, 9, 2} -> (9, 5, 2); ties by first token ascending
    seqs = seqs_of([[0, 10] + [1] * 4, [0, 11] + [1] * 8, [0, 12, 1]])
    root = O.order_children(O.build_prefix_tree(seqs), "subtree_tokens_desc")
    kids = root.children[0].children
    assert [O.subtree_tokens(c) for c in kids] == [9, 5, 2]
    seqs = seqs_of([[0, 13, 1], [0, 12, 1], [0, 11, 1]])
    root = O.order_children(O.build_prefix_tree(seqs), "subtree_tokens_desc")
    assert [c.tokens[0] for c in root.children[0].children] == [11, 12, 13]


def test_lexicographic_sort_example():
    # SPEC.md:165
    out = O.lexicographic_sort(seqs_of([[2], [1, 5], [1, 3]]))
    assert [s.tokens for s in out] == [[1, 3], [1, 5], [2]]


def test_round_trip_and_compression():
    rng = np.random.default_rng(3)
    for trial in range(20):
        seqs = O.grouped_corpus(3, 4, 3, 5, 6, trial, shared_response=1)
        root = O.build_prefix_tree(seqs)
        paths = {}

        def rec(n, pre):
            cur = pre + n.tokens
            for m in n.leaf_marks:
                paths[m] = cur
            if n.tokens:
                assert not (len(n.children) == 1 and not n.leaf_marks)
            for c in n.children:
                rec(c, cur)

        rec(root, [])
        assert all(paths[s.seq_id] == s.tokens for s in seqs)
        # uncompressed-trie oracle for the token count
        prefixes = {tuple(s.tokens[:k]) for s in seqs for k in range(1, len(s.tokens) + 1)}
        assert O.tree_token_count(root) == len(prefixes)
        assert O.max_path_tokens(root) == max(len(s.tokens) for s in seqs)


def test_weighted_nll_kats():
    V = CFG.vocab_size
    loss, g = O.weighted_nll(np.zeros((3, V)), [1, 2, 3], [1.0, 1.0, 1.0])
    assert loss == pytest.approx(3 * math.log(V), rel=1e-14)
    loss, g = O.weighted_nll(np.random.default_rng(0).normal(size=(3, V)), [1, 2, 3], [0.0, 0.0, 0.0])
    assert loss == 0.0 and not g.any()


def test_zero_upstream_zero_grads():
    flat = O.random_params(CFG, 1)
    P = O.unflatten(CFG, flat)
    empty = np.zeros((CFG.n_layers, 0, CFG.d_model))
    _, _, acts = O.forward_segment(CFG, P, empty, empty, [1, 2, 3, 4], 0)
    G = O.zero_like_params(CFG)
    gk, gv = O.backward_segment(CFG, P, acts, empty, empty, G)
    assert all(not v.any() for v in G.values())


def test_chained_segments_bitwise():
    # SPEC.md:69,91 on the oracle: forward [t1..t8] == forward [t1..t4] then [t5..t8]
    flat = O.random_params(CFG, 2)
    P = O.unflatten(CFG, flat)
    toks = [3, 1, 4, 1, 5, 9, 2, 6]
    empty = np.zeros((CFG.n_layers, 0, CFG.d_model))
    full, _, _ = O.forward_segment(CFG, P, empty, empty, toks, 0)
    a, (k, v), _ = O.forward_segment(CFG, P, empty, empty, toks[:4], 0)
    b, _, _ = O.forward_segment(CFG, P, k, v, toks[4:], 4)
    np.testing.assert_allclose(b, full[4:], rtol=1e-12, atol=1e-13)


def test_chunk_boundaries():
    assert O.chunk_boundaries(10, 4) == [(0, 4), (4, 8), (8, 10)]
    assert O.chunk_boundaries(4, 4) == [(0, 4)]
    assert O.chunk_boundaries(1, 1000) == [(0, 1)]


def test_tree_equals_dense_f64():
    # SPEC.md:232,548 (scaled): tree step == dense oracle within 1e-8, loss within 1e-10
    seqs = O.grouped_corpus(4, 8, 6, 10, CFG.vocab_size, 5, shared_response=2, weight_jitter=True)
    flat = O.random_params(CFG, 3)
    root = O.order_children(O.build_prefix_tree(seqs), "subtree_tokens_desc")
    t = O.tree_train_step(CFG, flat, root, seqs)
    d = O.dense_train_step(CFG, flat, seqs)
    assert abs(t.total_loss - d.total_loss) <= 1e-10 * abs(d.total_loss)
    assert O.compare_grads(t.grads, d.grads)[1] <= 1e-8
    assert t.forward_tokens == O.tree_token_count(root)
    assert t.peak_live_kv_tokens <= O.max_path_tokens(root)


def test_order_invariance():
    seqs = O.grouped_corpus(3, 5, 4, 8, CFG.vocab_size, 9, shared_response=3)
    flat = O.random_params(CFG, 4)
    ref = None
    for pol in O.POLICIES:
        root = O.order_children(O.build_prefix_tree(seqs), pol)
        r = O.tree_train_step(CFG, flat, root, seqs)
        if ref is None:
            ref = r
        assert O.compare_grads(r.grads, ref.grads)[1] <= 1e-8


def test_incremental_cost_example():
    assert O.incremental_group_cost(3, [1, 2, 3], [1, 2, 4]) == 4
    assert O.incremental_group_cost(3, [1, 2, 3], [1, 2, 3]) == 3


def test_partition_optimal_vs_dp():
    # SPEC.md:413,554 (sampled): contiguous binary search == DP optimum
    rng = np.random.default_rng(11)
    for trial in range(150):
        N = int(rng.integers(1, 13))
        K = int(rng.integers(2, 5))
        seqs = seqs_of([rng.integers(0, 3, int(rng.integers(1, 6))).tolist() for _ in range(N)])
        a = O.partition_contiguous(seqs, K)
        b = O.brute_force_optimal(seqs, K)
        assert a.max_cost == b.max_cost
        assert sorted(x for g in a.groups for x in g) == list(range(N))
        assert a.duplicated_tokens <= (K - 1) * max(len(s.tokens) for s in seqs)


def test_partition_trivial_cases():
    seqs = seqs_of([[1, 2, 3], [1, 2, 4]])
    assert O.partition_contiguous(seqs, 1).max_cost == 4
    p = O.partition_contiguous(seqs_of([[1], [2, 2], [3, 3, 3]]), 3)
    assert p.max_cost == 3
    g = O.greedy_least_loaded(seqs_of([[5, 5], [5, 5]]), 2, "raw_tokens")
    assert g.duplicated_tokens == 2
