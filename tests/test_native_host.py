"""Host-side logic of libtreetrain_b200.so (no GPU needed): tree build / order / serialisation /
DFS trace and the partitioner must be bit-exact with the oracle restatement of SPEC.md."""
import numpy as np
import pytest

import paper_2602_00482_b200 as tt
from oracle import treetrain_oracle as O


def to_native(seqs):
    return [tt.TokenSequence(s.seq_id, s.tokens, s.weights) for s in seqs]


def corpora():
    rng = np.random.default_rng(7)
    out = [O.grouped_corpus(4, 8, 5, 9, 32, s, shared_response=s % 4, weight_jitter=True) for s in range(6)]
    for s in range(10):
        N = int(rng.integers(1, 30))
        seqs = []
        for i in range(N):
            L = int(rng.integers(1, 9))
            seqs.append(O.TokenSequence(i, rng.integers(0, 3, L).tolist(), rng.uniform(0, 2, L).tolist()))
        out.append(seqs)
    out.append([O.TokenSequence(0, [1, 2, 3], [1.0] * 3), O.TokenSequence(1, [1, 2, 3], [1.0] * 3)])  # duplicates
    out.append([O.TokenSequence(0, [1, 2], [1.0] * 2), O.TokenSequence(1, [1, 2, 9], [1.0] * 3)])
    return out


@pytest.mark.parametrize("policy", list(O.POLICIES))
def test_tree_serialisation_and_trace_bit_exact(policy):
    for seqs in corpora():
        ref = O.order_children(O.build_prefix_tree(seqs), policy)
        nat = tt.build_prefix_tree(to_native(seqs), policy)
        assert nat.serialize() == O.serialize_tree(ref)
        assert nat.dfs_trace() == O.dfs_trace(ref)
        st = nat.stats()
        assert st["tree_tokens"] == O.tree_token_count(ref)
        assert st["max_path_tokens"] == O.max_path_tokens(ref)
        assert st["num_nodes"] == O.num_nodes(ref)


def test_build_errors():
    with pytest.raises(ValueError):
        tt.build_prefix_tree([])
    with pytest.raises(ValueError):
        tt.build_prefix_tree([tt.TokenSequence(0, [])])


def test_lexicographic_sort_matches():
    for seqs in corpora():
        a = [s.seq_id for s in tt.lexicographic_sort(to_native(seqs))]
        b = [s.seq_id for s in O.lexicographic_sort(seqs)]
        assert a == b


def test_partition_matches_oracle_and_dp():
    rng = np.random.default_rng(5)
    for trial in range(200):
        N = int(rng.integers(1, 13))
        K = int(rng.integers(1, 5))
        seqs = [O.TokenSequence(i, rng.integers(0, 3, int(rng.integers(1, 6))).tolist(), None) for i in range(N)]
        a = tt.partition_contiguous(to_native(seqs), K)
        b = O.partition_contiguous(seqs, K)
        dp = O.brute_force_optimal(seqs, K)
        assert a["max_cost"] == b.max_cost == dp.max_cost
        assert a["groups"] == [sorted(g) for g in b.groups] or sorted(map(sorted, a["groups"])) == sorted(map(sorted, b.groups))
        assert a["duplicated_tokens"] == b.duplicated_tokens
        assert a["duplicated_tokens"] <= (K - 1) * max(len(s.tokens) for s in seqs)


def test_greedy_matches_oracle():
    rng = np.random.default_rng(6)
    for trial in range(50):
        N, K = int(rng.integers(1, 15)), int(rng.integers(1, 5))
        seqs = [O.TokenSequence(i, rng.integers(0, 3, int(rng.integers(1, 6))).tolist(), None) for i in range(N)]
        for mode in ("raw_tokens", "tree_tokens"):
            a = tt.greedy_least_loaded(to_native(seqs), K, mode)
            b = O.greedy_least_loaded(seqs, K, mode)
            assert a["costs"] == b.costs and a["duplicated_tokens"] == b.duplicated_tokens


def test_balancing_direction():
    # SPEC.md:556 (sampled): contiguous DFS partitioning duplicates fewer tokens than greedy raw
    wins = 0
    for s in range(40):
        seqs = O.grouped_corpus(8, 8, 6, 12, 50, s, shared_response=4)
        a = tt.partition_contiguous(to_native(seqs), 4)
        b = tt.greedy_least_loaded(to_native(seqs), 4, "raw_tokens")
        wins += a["duplicated_tokens"] < b["duplicated_tokens"]
    assert wins >= 38
