"""GPU parity at the headline configuration and through the extended C-ABI boundary.

  * the c2 model shape (BASELINE configs[1]: V 151936, d 896, 14 heads of 64, 24 layers, d_ff 4864)
    on a short tree against the f64 oracle — with the default LM-head chunking and with >= 3 forced
    head chunks (the multi-chunk CE + split-K dX path the c2 bench runs);
  * the multi-chunk LM head and budget-split sibling batches at C1 / SMALL;
  * TTPM interchange: a file written by the reference's own save_parameters (model_io.cpp:44-71,
    through oracle/_ref) loaded with tt_params_load_ttpm gives bit-identical logits to uploading the
    same values;
  * the segment-level DFS entirely through the C-ABI with the loss on the device (tt_segment_loss),
    want_kv / want_activations semantics, the standalone tt_weighted_nll, f64 gradient download and
    the NCCL all-reduce on a one-rank communicator.

Tolerances as tests/test_engine_gpu.py (loss |rel| <= 5e-3; per-tensor rel-Frobenius <= 3e-2 and
cosine >= 0.999; logits rel-Frobenius <= 1e-2).
"""
import math

import numpy as np
import pytest

import paper_2602_00482_b200 as tt
from oracle import treetrain_oracle as O

from test_engine_gpu import C1, GRAD_TOL, LOGIT_TOL, LOSS_TOL, SMALL, check_grads, make, rel, tree_case

pytestmark = pytest.mark.gpu

C2 = (151936, 896, 14, 24, 4864, 1024)  # SURVEY §8 c2 model, reference architecture


def lean_params(cfg: O.ModelConfig, seed: int) -> np.ndarray:
    """N(0, 0.02) weights rounded to bf16 (unit gains), built tensor by tensor in float32 so the 0.56B
    c2 parameter vector costs one float64 copy of host memory."""
    rng = np.random.default_rng(seed)
    out = np.empty(O.param_count(cfg), dtype=np.float64)
    o = 0
    for name, shape in O.tensor_specs(cfg):
        n = int(np.prod(shape))
        if name.endswith("norm_gain"):
            out[o:o + n] = 1.0
        else:
            x = rng.standard_normal(n, dtype=np.float32) * np.float32(0.02)
            u = x.view(np.uint32)
            u += np.uint32(0x7FFF) + ((u >> np.uint32(16)) & np.uint32(1))
            u &= np.uint32(0xFFFF0000)
            out[o:o + n] = x
        o += n
    return out


@pytest.fixture(scope="module")
def c2_case():
    cfg = O.ModelConfig(*C2)
    flat = lean_params(cfg, 2602)
    # one rollout group: 96-token prompt + 4 branches of 64 tokens (257 loss rows: every response
    # row plus the prompt's last row, which predicts each branch's first token)
    seqs = O.grouped_corpus(1, 4, 96, 64, cfg.vocab_size, 482, weight_jitter=True)
    root = O.order_children(O.build_prefix_tree(seqs), "subtree_tokens_desc")
    ref = O.tree_train_step(cfg, flat, root, seqs)
    return cfg, flat, seqs, ref


@pytest.mark.parametrize("head_chunk_mb", [0, 120], ids=["auto_chunks", "three_head_chunks"])
def test_c2_model_shape_tree_vs_oracle(c2_case, head_chunk_mb):
    cfg, flat, seqs, ref = c2_case
    eng = tt.Engine(tt.ModelConfig(*C2))
    eng.upload_params(flat)
    if head_chunk_mb:
        # 120 MB of fp32 logits + bf16 dlogits = 128 rows of V = 151936 per chunk: 257 loss rows -> 3
        # chunks, each a 128 x 151936 x 896 logits GEMM, CE, dW_head and a split-K dX GEMM
        eng.set_option("head_chunk_mb", head_chunk_mb)
    tree = tt.build_prefix_tree([tt.TokenSequence(s.seq_id, s.tokens, s.weights) for s in seqs])
    eng.zero_gradients()
    r = eng.tree_train_step(tree, tt.SchedulerConfig())
    got = eng.gradients()
    assert abs(r.total_loss - ref.total_loss) <= LOSS_TOL * abs(ref.total_loss), (r.total_loss, ref.total_loss)
    worst = check_grads(cfg, got, ref.grads)
    print("c2 worst tensor", worst, "loss", r.total_loss, ref.total_loss)
    eng.close()


def test_multichunk_lm_head_vs_oracle():
    # C1 with a 1 MB head budget: 128-row chunks (2048+ loss rows -> 16+ chunks), each with its own
    # CE, dW_head read-modify-write and (split-K) dX GEMM
    cfg, flat, eng = make(C1, 51)
    eng.set_option("head_chunk_mb", 1)
    seqs = O.grouped_corpus(1, 8, 512, 256, cfg.vocab_size, 52, weight_jitter=True)
    tree_case(cfg, seqs, flat, eng, tt.SchedulerConfig())


@pytest.mark.parametrize("budget", [64, 150])
def test_budget_split_sibling_batches_vs_oracle(budget):
    # batch_token_budget splits a run of sibling leaves into several varlen batches (as the automatic
    # memory budget does at c4); results must not change
    cfg, flat, eng = make(SMALL, 53)
    seqs = O.grouped_corpus(2, 6, 60, 50, cfg.vocab_size, 54, weight_jitter=True)
    r_all, _ = tree_case(cfg, seqs, flat, eng, tt.SchedulerConfig(batch_token_budget=0))
    r, _ = tree_case(cfg, seqs, flat, eng, tt.SchedulerConfig(batch_token_budget=budget))
    assert r.num_batches > r_all.num_batches
    assert r.num_segments == r_all.num_segments


def test_reference_ttpm_interchange(tmp_path):
    """load_parameters (model_io.cpp:73-105) of a file the REFERENCE wrote (save_parameters,
    model_io.cpp:44-71, via oracle/_ref) == uploading the same values, bit for bit."""
    from oracle import refimpl as R

    if not R.available():
        pytest.skip("oracle/_ref/libttref.so not built")
    cfg = O.ModelConfig(*SMALL)
    flat = R.init_params(cfg, 7)  # the reference's init_params(cfg, seed = 7) (model.hpp:121-142)
    toks = list(np.random.default_rng(5).integers(0, cfg.vocab_size, 77))
    for dtype in ("f32", "f64"):
        path = str(tmp_path / f"ref_{dtype}.ttpm")
        R.save_ttpm(cfg, flat, path, dtype)
        a = tt.Engine(tt.ModelConfig(*SMALL))
        a.load_parameters(path)
        b = tt.Engine(tt.ModelConfig(*SMALL))
        b.upload_params(flat.astype(np.float32))
        la, lb = a.forward_segment(toks), b.forward_segment(toks)
        assert np.array_equal(la, lb), dtype
        a.close()
        b.close()
    bad = O.ModelConfig(SMALL[0], SMALL[1], SMALL[2], SMALL[3] + 1, SMALL[4], SMALL[5])
    path = str(tmp_path / "other.ttpm")
    R.save_ttpm(bad, R.init_params(bad, 7), path, "f32")
    e = tt.Engine(tt.ModelConfig(*SMALL))
    with pytest.raises(ValueError):
        e.load_parameters(path)
    with pytest.raises(RuntimeError):
        e.load_parameters(str(tmp_path / "missing.ttpm"))


def _targets(rng, n, V, zero_frac=0.2):
    t = rng.integers(0, V, n)
    w = rng.uniform(0.5, 1.5, n)
    w[rng.random(n) < zero_frac] = 0.0
    return t, w


@pytest.mark.parametrize("cfgt", [SMALL, (512, 256, 2, 2, 512, 1024)], ids=["dh64", "dh128"])
def test_segment_dfs_three_node_chain_device_loss(cfgt):
    """PUSH A, PUSH B, PUSH C, VISIT+POP C, VISIT+POP B, VISIT+POP A entirely through the C-ABI,
    the losses computed on the device (tt_segment_loss, multi-target rows on B): losses, every
    grad_prefix and the final gradients against the oracle's forward/backward_segment chain."""
    cfg, flat, eng = make(cfgt, 61)
    P = O.unflatten(cfg, flat)
    rng = np.random.default_rng(62)
    la_, lb_, lc_ = 70, 45, 58
    A, B, C = (rng.integers(0, cfg.vocab_size, n).tolist() for n in (la_, lb_, lc_))
    empty = np.zeros((cfg.n_layers, 0, cfg.d_model))
    lgA, (kA, vA), actsA = O.forward_segment(cfg, P, empty, empty, A, 0)
    lgB, (kB, vB), actsB = O.forward_segment(cfg, P, kA, vA, B, la_)
    kAB, vAB = np.concatenate([kA, kB], 1), np.concatenate([vA, vB], 1)
    lgC, _, actsC = O.forward_segment(cfg, P, kAB, vAB, C, la_ + lb_)
    tA, wA = _targets(rng, la_, cfg.vocab_size)
    tC, wC = _targets(rng, lc_, cfg.vocab_size)
    # B: two (target, weight) pairs on every third row (a node-boundary row)
    rowsB, tB, wB, offB = [], [], [], [0]
    for r in range(lb_):
        k = 2 if r % 3 == 0 else 1
        for _ in range(k):
            rowsB.append(r)
            tB.append(int(rng.integers(0, cfg.vocab_size)))
            wB.append(float(rng.uniform(0.5, 1.5)))
        offB.append(len(tB))
    lossC, gC = O.weighted_nll(lgC, tC, wC)
    lossB, gB = O.weighted_nll_pairs(lgB, rowsB, tB, wB)
    lossA, gA = O.weighted_nll(lgA, tA, wA)
    G = O.zero_like_params(cfg)
    gpk_C, gpv_C = O.backward_segment(cfg, P, actsC, kAB, vAB, G, gC)
    gpk_B, gpv_B = O.backward_segment(cfg, P, actsB, kA, vA, G, gB, gpk_C[:, la_:], gpv_C[:, la_:])
    O.backward_segment(cfg, P, actsA, empty, empty, G, gA, gpk_C[:, :la_] + gpk_B, gpv_C[:, :la_] + gpv_B)

    eng.zero_gradients()
    for seg in (A, B, C):
        assert eng.forward_segment(seg, want_logits=False) is None
    assert abs(eng.segment_loss(tC, wC) - lossC) <= LOSS_TOL * abs(lossC)
    dk, dv = eng.backward_segment()
    assert rel(dk, gpk_C) <= GRAD_TOL and rel(dv, gpv_C) <= GRAD_TOL, (rel(dk, gpk_C), rel(dv, gpv_C))
    assert abs(eng.segment_loss(tB, wB, row_off=offB) - lossB) <= LOSS_TOL * abs(lossB)
    dk, dv = eng.backward_segment()
    assert rel(dk, gpk_B) <= GRAD_TOL and rel(dv, gpv_B) <= GRAD_TOL, (rel(dk, gpk_B), rel(dv, gpv_B))
    assert abs(eng.segment_loss(tA, wA) - lossA) <= LOSS_TOL * abs(lossA)
    eng.backward_segment()
    check_grads(cfg, eng.gradients(np.float64), O.flatten(cfg, G))
    assert eng.accum_count == 3 and eng.stack_depth() == (0, 0)


def test_segment_want_kv_and_want_activations():
    cfg, flat, eng = make(SMALL, 71)
    P = O.unflatten(cfg, flat)
    rng = np.random.default_rng(72)
    A = rng.integers(0, cfg.vocab_size, 40).tolist()
    B = rng.integers(0, cfg.vocab_size, 33).tolist()
    empty = np.zeros((cfg.n_layers, 0, cfg.d_model))
    lgA, (kA, vA), actsA = O.forward_segment(cfg, P, empty, empty, A, 0)
    lgB, _, actsB = O.forward_segment(cfg, P, kA, vA, B, len(A))
    # forward only (want_kv = want_activations = False): logits, nothing pushed
    la = eng.forward_segment(A, want_kv=False, want_activations=False)
    assert rel(la, lgA) <= LOGIT_TOL and eng.stack_depth() == (0, 0)
    # A without activations (its pop recomputes them), B without KV (a leaf: nothing may go on top)
    eng.forward_segment(A, want_logits=False, want_activations=False)
    lb = eng.forward_segment(B, want_kv=False)
    assert rel(lb, lgB) <= LOGIT_TOL and eng.stack_depth() == (len(A) + len(B), 2)
    with pytest.raises(ValueError):
        eng.forward_segment([1, 2, 3])
    tB, wB = _targets(rng, len(B), cfg.vocab_size)
    tA, wA = _targets(rng, len(A), cfg.vocab_size)
    _, gB = O.weighted_nll(lgB, tB, wB)
    _, gA = O.weighted_nll(lgA, tA, wA)
    G = O.zero_like_params(cfg)
    gpk, gpv = O.backward_segment(cfg, P, actsB, kA, vA, G, gB)
    O.backward_segment(cfg, P, actsA, empty, empty, G, gA, gpk, gpv)
    eng.zero_gradients()
    with pytest.raises(ValueError):  # both a device loss and host grad_logits
        eng.segment_loss(tB, wB)
        eng.backward_segment(gB)
    eng.stack_reset()
    eng.zero_gradients()
    eng.forward_segment(A, want_logits=False, want_activations=False)
    eng.forward_segment(B, want_logits=False, want_kv=False)
    eng.backward_segment(gB, want_grad_prefix=False)
    with pytest.raises(ValueError):  # weighted_nll needs the segment's activations
        eng.segment_loss(tA, wA)
    eng.backward_segment(gA)  # recompute + backward
    check_grads(cfg, eng.gradients(), O.flatten(cfg, G))
    with pytest.raises(ValueError):  # grad_logits shape is checked (model.hpp:488-490)
        eng.forward_segment(A, want_logits=False)
        eng.backward_segment(np.zeros((len(A) + 1, cfg.vocab_size), np.float32))


@pytest.mark.parametrize("V", [512, 151936])
def test_weighted_nll_device_vs_oracle(V):
    eng = tt.Engine(tt.ModelConfig(V, 128, 2, 1, 256, 64))
    rng = np.random.default_rng(81)
    n = 37
    logits = rng.normal(0, 3, (n, V)).astype(np.float32)
    t, w = _targets(rng, n, V)
    loss, grad = eng.weighted_nll(logits, t, w)
    rl, rg = O.weighted_nll(logits.astype(np.float64), t, w)
    assert abs(loss - rl) <= 1e-5 * abs(rl) and rel(grad, rg) <= 1e-5
    assert not grad[w == 0].any()  # weight-0 rows stay zero (model.hpp:658)
    # multi-target rows
    off = [0]
    tt_, ww = [], []
    rows = []
    for r in range(n):
        for _ in range(1 + r % 3):
            rows.append(r)
            tt_.append(int(rng.integers(0, V)))
            ww.append(float(rng.uniform(0.1, 2.0)))
        off.append(len(tt_))
    loss, grad = eng.weighted_nll(logits, tt_, ww, row_off=off)
    rl, rg = O.weighted_nll_pairs(logits.astype(np.float64), rows, tt_, ww)
    assert abs(loss - rl) <= 1e-5 * abs(rl) and rel(grad, rg) <= 1e-5
    with pytest.raises(ValueError):
        eng.weighted_nll(logits, [V] + list(t[1:]), w)
    with pytest.raises(ValueError):
        eng.weighted_nll(logits, t, [math.nan] + list(w[1:]))


def test_grads_f64_download_and_single_rank_nccl_allreduce():
    cfg, flat, eng = make(SMALL, 91)
    seqs = O.grouped_corpus(2, 3, 30, 40, cfg.vocab_size, 92)
    eng.zero_gradients()
    eng.tree_train_step(tt.build_prefix_tree([tt.TokenSequence(s.seq_id, s.tokens, s.weights) for s in seqs]))
    g32 = eng.gradients()
    g64 = eng.gradients(np.float64)
    assert g64.dtype == np.float64 and np.array_equal(g64, g32.astype(np.float64))
    comm = tt.NcclComm(tt.nccl_unique_id(), 1, 0, 0)  # one rank: the all-reduce is the identity
    eng.allreduce_gradients(comm)
    assert np.array_equal(eng.gradients(), g32)
    comm.close()


def test_token_out_of_range_rejected_before_upload():
    cfg, flat, eng = make(SMALL, 93)
    bad = [tt.TokenSequence(0, [1, 2, cfg.vocab_size], [1.0, 1.0, 1.0])]
    with pytest.raises(ValueError):
        eng.tree_train_step(tt.build_prefix_tree(bad))
    with pytest.raises(ValueError):
        eng.dense_train_step([tt.TokenSequence(0, [-1, 2, 3])])
    g = eng.gradients()
    assert not g.any()  # nothing ran


def test_plan_from_another_engine_rejected_and_option_change_recaptures():
    cfg, flat, a = make(SMALL, 94)
    b = tt.Engine(tt.ModelConfig(*SMALL))
    b.upload_params(flat)
    seqs = O.grouped_corpus(2, 3, 30, 40, cfg.vocab_size, 95)
    tree = tt.build_prefix_tree([tt.TokenSequence(s.seq_id, s.tokens, s.weights) for s in seqs])
    plan = a.plan(tree)
    with pytest.raises(ValueError):
        _exec_on(b, plan)
    r1 = plan.execute()
    r2 = plan.execute()  # captured
    a.set_option("gemm_2cta", 0)
    r3 = plan.execute()  # options changed: re-captured, same result
    assert abs(r3.total_loss - r1.total_loss) <= 1e-6 * abs(r1.total_loss)
    assert abs(r2.total_loss - r1.total_loss) <= 1e-9 * abs(r1.total_loss)


def _exec_on(eng, plan):
    import ctypes
    from paper_2602_00482_b200 import _native

    r = _native.StepResultC()
    tt._check(_native.lib().tt_plan_execute(eng._h, plan._h, ctypes.byref(r)))


def test_wide_model_d_above_4096_vs_oracle():
    # d = 5120 (a 14B-class width): RMSNorm forward / backward spread a row over several warps
    cfg, flat, eng = make((512, 5120, 40, 1, 512, 256), 96)
    seqs = O.grouped_corpus(1, 3, 40, 30, cfg.vocab_size, 97)
    tree_case(cfg, seqs, flat, eng, tt.SchedulerConfig())
