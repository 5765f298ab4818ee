"""Corpus JSONL I/O and gen-corpus, through the C-ABI (host-only, no GPU)."""
import json

import numpy as np
import pytest

import paper_2602_00482_b200 as tt


def _dup(seqs):
    return sum(len(s.tokens) for s in seqs) / tt.build_prefix_tree(seqs).stats()["tree_tokens"]


def test_gen_corpus_deterministic_and_byte_identical(tmp_path):
    spec = tt.CorpusSpec(num_prompts=5, group_size=4, prompt_len=(3, 9), response_len=(2, 7), branch_prob=0.3,
                         vocab_size=50, seed=11)
    a, b = tt.gen_corpus(spec), tt.gen_corpus(spec)
    assert len(a) == 20
    for x, y in zip(a, b):
        assert x.seq_id == y.seq_id and np.array_equal(x.tokens, y.tokens) and np.array_equal(x.weights, y.weights)
    tt.save_corpus_jsonl(a, tmp_path / "a.jsonl")
    tt.save_corpus_jsonl(b, tmp_path / "b.jsonl")
    assert (tmp_path / "a.jsonl").read_bytes() == (tmp_path / "b.jsonl").read_bytes()
    c = tt.gen_corpus(tt.CorpusSpec(**{**spec.__dict__, "seed": 12}))
    assert any(not np.array_equal(x.tokens, y.tokens) for x, y in zip(a, c))


def test_gen_corpus_group_size_one_has_no_sharing():
    # group_size=1 -> duplication_factor = 1.0 (distinct prompts)
    seqs = tt.gen_corpus(tt.CorpusSpec(num_prompts=30, group_size=1, prompt_len=(4, 8), response_len=(1, 5),
                                       branch_prob=0.5, vocab_size=1000, seed=3))
    assert _dup(seqs) == 1.0


@pytest.mark.parametrize("G,P,R", [(8, 6, 5), (16, 32, 32), (3, 1, 10)])
def test_gen_corpus_branch_prob_one_duplication_formula(G, P, R):
    # branch_prob=1, constant P, R -> duplication = G(P+R)/(P+GR)
    seqs = tt.gen_corpus(tt.CorpusSpec(num_prompts=4, group_size=G, prompt_len=(P, P), response_len=(R, R),
                                       branch_prob=1.0, vocab_size=5000, seed=G))
    assert _dup(seqs) == pytest.approx(G * (P + R) / (P + G * R), rel=1e-12)
    for s in seqs:  # weights 0 on the prompt, 1 on the response
        assert np.all(s.weights[:P] == 0) and np.all(s.weights[P:] == 1)


def test_jsonl_round_trip_exact(tmp_path):
    rng = np.random.default_rng(0)
    seqs = [tt.TokenSequence(i, rng.integers(0, 99, rng.integers(1, 20)).astype(np.int32), None) for i in range(9)]
    for s in seqs:
        s.weights = rng.random(len(s.tokens)) * 3.0  # arbitrary doubles must round trip exactly
    tt.save_corpus_jsonl(seqs, tmp_path / "c.jsonl")
    back = tt.load_corpus_jsonl(tmp_path / "c.jsonl")
    assert len(back) == len(seqs)
    for x, y in zip(seqs, back):
        assert x.seq_id == y.seq_id and np.array_equal(x.tokens, y.tokens)
        assert np.array_equal(np.asarray(x.weights), y.weights)  # bit-exact (%.17g)
    for line in (tmp_path / "c.jsonl").read_text().splitlines():
        obj = json.loads(line)  # valid JSON per line
        assert set(obj) == {"seq_id", "tokens", "weights"}


def test_jsonl_default_weights_and_string_ids(tmp_path):
    p = tmp_path / "d.jsonl"
    p.write_text('{"seq_id": "rollout-a", "tokens": [1, 2, 3, 4], "prompt_len": 2, "meta": {"x": [1, 2]}}\n'
                 '\n'
                 '{"tokens": [5, 6], "seq_id": 7}\n')
    a, b = tt.load_corpus_jsonl(p)
    assert a.name == "rollout-a" and list(a.weights) == [0.0, 0.0, 1.0, 1.0]  # SPEC.md:192 default
    assert b.seq_id == 7 and list(b.weights) == [1.0, 1.0]


@pytest.mark.parametrize("line,msg", [('{"seq_id": "x", "tokens": []}', "tokens"),
                                      ('{"seq_id": "x", "tokens": [1, 2], "weights": [1]}', "weights"),
                                      ('{"tokens": [1]}', "seq_id"),
                                      ('{"seq_id": "x", "tokens": [1.5]}', "int32"),
                                      ('{"seq_id": "x", "tokens": [1]', "expected")])
def test_jsonl_malformed_lines_raise_value_error(tmp_path, line, msg):
    p = tmp_path / "bad.jsonl"
    p.write_text('{"seq_id": "ok", "tokens": [1]}\n' + line + "\n")
    with pytest.raises(ValueError, match="line 2"):
        tt.load_corpus_jsonl(p)


def test_jsonl_missing_file_raises_runtime_error(tmp_path):
    with pytest.raises(RuntimeError):
        tt.load_corpus_jsonl(tmp_path / "nope.jsonl")


def test_corpus_feeds_partitioner_and_tree():
    seqs = tt.gen_corpus(tt.CorpusSpec(num_prompts=6, group_size=8, prompt_len=(20, 40), response_len=(10, 30),
                                       branch_prob=0.2, vocab_size=32000, seed=5))
    plan = tt.partition_contiguous(seqs, 3)
    assert sorted(i for g in plan["groups"] for i in g) == sorted(s.seq_id for s in seqs)
    assert plan["duplicated_tokens"] <= 2 * max(len(s.tokens) for s in seqs)
