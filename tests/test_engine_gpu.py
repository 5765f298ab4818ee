"""GPU parity: the CUDA engine (through the C-ABI) against the CPU oracle on the same seeded
inputs and the same bf16-rounded weights.

Tolerances (bf16 operands, fp32 accumulation / residual / dK-dV stack / gradients, fp64 loss):
  loss                 |rel| <= 5e-3
  logits               rel-Frobenius <= 1e-2
  gradients (per tensor of for_each_tensor order, model.hpp:42-59)
                       rel-Frobenius <= 3e-2 and cosine >= 0.999; the attention query/key
                       projections (w_q, w_k) rel-Frobenius <= 5e-2 and cosine >= 0.999
The w_q / w_k gradients are contractions of dS = P*(dP - D), whose rows sum to zero (softmax shift
invariance) while the bf16 activations feeding it (normed x, q, k, v, O, dO) carry a large common
component (the sinusoidal PE dominates the random-init residual stream), so their relative error is
amplified: at the c2 shape they measure 1.7e-2 median / 3.0e-2 max against 3.5e-3-5.4e-3 for every
other tensor (tools/c2_grad_diag.py). The attention kernels themselves match an fp32
emulation of their own bf16 operand rounding to three digits (tools/attn_precision.py), and
tools/qk_grad_precision.py reproduces the amplification from activation rounding alone on the CPU.
Tree structure and traversal are checked bit-exactly in tests/test_native_host.py.
"""
import math

import numpy as np
import pytest

import paper_2602_00482_b200 as tt
from oracle import treetrain_oracle as O

pytestmark = pytest.mark.gpu

SMALL = (512, 128, 2, 2, 256, 1024)  # V, d, H, L, d_ff, max_position ; head_dim 64
DH128 = (512, 256, 2, 2, 512, 1024)  # head_dim 128
C1 = (1024, 256, 4, 2, 1024, 2048)   # BASELINE configs[0] model (V proposed in SURVEY §8(d))

LOSS_TOL, LOGIT_TOL, GRAD_TOL, QK_GRAD_TOL, COS_TOL = 5e-3, 1e-2, 3e-2, 5e-2, 0.999


def make(cfgt, seed=0):
    ocfg = O.ModelConfig(*cfgt)
    flat = O.round_bf16(O.random_params(ocfg, seed))
    eng = tt.Engine(tt.ModelConfig(*cfgt))
    eng.upload_params(flat)
    return ocfg, flat, eng


def rel(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30))


def check_grads(cfg, got, ref, tol=GRAD_TOL, cos_tol=COS_TOL, qk_tol=None):
    """Per-tensor gradient check vs the oracle. qk_tol (default: QK_GRAD_TOL under the oracle
    tolerance, else the same as tol) bounds w_q / w_k; engine-vs-engine checks stay uniform."""
    if qk_tol is None:
        qk_tol = QK_GRAD_TOL if tol == GRAD_TOL else tol
    o = 0
    worst = (0.0, "")
    scale = np.linalg.norm(ref)
    for name, shape in O.tensor_specs(cfg):
        n = int(np.prod(shape))
        g, r = got[o:o + n].astype(np.float64), ref[o:o + n]
        o += n
        rn = np.linalg.norm(r)
        if rn < 1e-6 * scale:  # tensor with (near) zero gradient: check absolute size only
            assert np.linalg.norm(g) <= 1e-4 * scale + 1e-12, name
            continue
        e = rel(g, r)
        cs = float(g @ r / (np.linalg.norm(g) * rn))
        worst = max(worst, (e, name))
        lim = qk_tol if name.endswith((".w_q", ".w_k")) else tol
        assert e <= lim and cs >= cos_tol, f"{name}: rel {e:.3e} cos {cs:.6f}"
    return worst


def tree_case(cfg, seqs, flat, eng, sched):
    root = O.order_children(O.build_prefix_tree(seqs), "subtree_tokens_desc")
    ref = O.tree_train_step(cfg, flat, root, seqs)
    tree = tt.build_prefix_tree([tt.TokenSequence(s.seq_id, s.tokens, s.weights) for s in seqs])
    eng.zero_gradients()
    r = eng.tree_train_step(tree, sched)
    got = eng.gradients()
    assert abs(r.total_loss - ref.total_loss) <= LOSS_TOL * abs(ref.total_loss), (r.total_loss, ref.total_loss)
    worst = check_grads(cfg, got, ref.grads)
    assert r.forward_tokens == O.tree_token_count(root)
    return r, worst


@pytest.mark.parametrize("cfgt", [SMALL, DH128])
def test_forward_segment_chain_logits(cfgt):
    cfg, flat, eng = make(cfgt, 1)
    P = O.unflatten(cfg, flat)
    rng = np.random.default_rng(0)
    a = rng.integers(0, cfg.vocab_size, 70).tolist()
    b = rng.integers(0, cfg.vocab_size, 45).tolist()
    empty = np.zeros((cfg.n_layers, 0, cfg.d_model))
    la, (ka, va), _ = O.forward_segment(cfg, P, empty, empty, a, 0)
    lb, _, _ = O.forward_segment(cfg, P, ka, va, b, len(a))
    ga = eng.forward_segment(a)
    gb = eng.forward_segment(b)
    assert rel(ga, la) <= LOGIT_TOL and rel(gb, lb) <= LOGIT_TOL, (rel(ga, la), rel(gb, lb))
    eng.stack_reset()


@pytest.mark.parametrize("cfgt", [SMALL, DH128])
def test_backward_segment_chain(cfgt):
    cfg, flat, eng = make(cfgt, 2)
    P = O.unflatten(cfg, flat)
    rng = np.random.default_rng(1)
    a = rng.integers(0, cfg.vocab_size, 90).tolist()
    b = rng.integers(0, cfg.vocab_size, 66).tolist()
    empty = np.zeros((cfg.n_layers, 0, cfg.d_model))
    la, (ka, va), acts_a = O.forward_segment(cfg, P, empty, empty, a, 0)
    lb, _, acts_b = O.forward_segment(cfg, P, ka, va, b, len(a))
    _, gla = O.weighted_nll(la, rng.integers(0, cfg.vocab_size, len(a)), rng.uniform(0.5, 1.5, len(a)))
    _, glb = O.weighted_nll(lb, rng.integers(0, cfg.vocab_size, len(b)), rng.uniform(0.5, 1.5, len(b)))
    G = O.zero_like_params(cfg)
    gpk, gpv = O.backward_segment(cfg, P, acts_b, ka, va, G, glb)
    O.backward_segment(cfg, P, acts_a, empty, empty, G, gla, gpk, gpv)
    eng.zero_gradients()
    eng.forward_segment(a, want_logits=False)
    eng.forward_segment(b, want_logits=False)
    dk, dv = eng.backward_segment(glb)
    assert rel(dk, gpk) <= GRAD_TOL and rel(dv, gpv) <= GRAD_TOL, (rel(dk, gpk), rel(dv, gpv))
    eng.backward_segment(gla)
    check_grads(cfg, eng.gradients(), O.flatten(cfg, G))
    assert eng.accum_count == 2


@pytest.mark.parametrize("sibling_batch", [False, True])
def test_tree_step_small(sibling_batch):
    cfg, flat, eng = make(SMALL, 3)
    seqs = O.grouped_corpus(3, 5, 40, 70, cfg.vocab_size, 4, shared_response=10, weight_jitter=True)
    r, worst = tree_case(cfg, seqs, flat, eng, tt.SchedulerConfig(sibling_batch=sibling_batch))
    assert r.num_segments == O.num_nodes(O.build_prefix_tree(seqs))


def test_tree_step_prefix_contained_and_deep():
    cfg, flat, eng = make(SMALL, 4)
    rng = np.random.default_rng(9)
    base = rng.integers(0, cfg.vocab_size, 100).tolist()
    seqs = [O.TokenSequence(0, base[:40], [0.0] * 10 + [1.0] * 30),           # prefix-contained (leaf_mark)
            O.TokenSequence(1, base, [0.0] * 10 + [1.0] * 90),
            O.TokenSequence(2, base[:60] + [7, 8, 9], [0.0] * 10 + [2.0] * 53),
            O.TokenSequence(3, base[:60] + [7, 8, 10, 11], [0.0] * 10 + [0.5] * 57),
            O.TokenSequence(4, base[:20] + rng.integers(0, 500, 130).tolist(), [1.0] * 150)]
    for sb in (False, True):
        tree_case(cfg, seqs, flat, eng, tt.SchedulerConfig(sibling_batch=sb))


@pytest.mark.parametrize("tmode", [0, 2], ids=["dw_plain", "dw_transposed"])
def test_tree_step_gemm_orientation_vs_oracle(tmode):
    """Every dW / LM-head dX accumulate as C += A B^T (mode 0) or as C^T += B A^T (mode 2, the
    transposed reduce-add epilogue) gives the oracle's loss and gradients."""
    from paper_2602_00482_b200 import _native

    cfg, flat, eng = make(C1, 11)
    seqs = O.grouped_corpus(2, 4, 200, 120, cfg.vocab_size, 12, shared_response=6, weight_jitter=True)
    _native.lib().tt_debug_gemm_set_transpose(tmode)
    try:
        tree_case(cfg, seqs, flat, eng, tt.SchedulerConfig())
    finally:
        _native.lib().tt_debug_gemm_set_transpose(1)


def test_tree_step_d448_224_wide_gemm_tiles_vs_oracle():
    """d = 448 (7 heads of 64): every d-wide dX GEMM with >= 256 rows runs the 224-wide CTA-pair
    tiles (N % 256 != 0, K-major B); the step must still match the oracle."""
    cfg, flat, eng = make((512, 448, 7, 2, 1024, 1024), 13)
    seqs = O.grouped_corpus(2, 4, 256, 128, cfg.vocab_size, 14, shared_response=4, weight_jitter=True)
    tree_case(cfg, seqs, flat, eng, tt.SchedulerConfig())


def test_tree_step_dh128():
    cfg, flat, eng = make(DH128, 5)
    seqs = O.grouped_corpus(2, 4, 130, 90, cfg.vocab_size, 6, shared_response=5)
    tree_case(cfg, seqs, flat, eng, tt.SchedulerConfig())


def test_dense_step_matches_oracle():
    cfg, flat, eng = make(SMALL, 6)
    seqs = O.grouped_corpus(2, 3, 30, 50, cfg.vocab_size, 8, weight_jitter=True)
    ref = O.dense_train_step(cfg, flat, seqs)
    eng.zero_gradients()
    r = eng.dense_train_step([tt.TokenSequence(s.seq_id, s.tokens, s.weights) for s in seqs])
    assert abs(r.total_loss - ref.total_loss) <= LOSS_TOL * abs(ref.total_loss)
    check_grads(cfg, eng.gradients(), ref.grads)
    assert r.forward_tokens == sum(len(s.tokens) for s in seqs)


def test_tree_equals_dense_on_device():
    # SPEC.md:263 on the engine itself: tree step == flat per-sequence step
    cfg, flat, eng = make(SMALL, 7)
    seqs = O.grouped_corpus(2, 6, 50, 60, cfg.vocab_size, 10, shared_response=8, weight_jitter=True)
    eng.zero_gradients()
    rt = eng.tree_train_step(tt.build_prefix_tree([tt.TokenSequence(s.seq_id, s.tokens, s.weights) for s in seqs]))
    gt = eng.gradients()
    eng.zero_gradients()
    rd = eng.dense_train_step([tt.TokenSequence(s.seq_id, s.tokens, s.weights) for s in seqs])
    gd = eng.gradients()
    assert abs(rt.total_loss - rd.total_loss) <= 1e-3 * abs(rd.total_loss)
    check_grads(cfg, gt, gd.astype(np.float64), tol=1e-2, cos_tol=0.9999)
    assert rd.forward_tokens / rt.forward_tokens == pytest.approx(O.duplication_factor(seqs))


def test_c1_tree_vs_oracle():
    # BASELINE configs[0]: tiny 2-layer d=256, one prefix tree (512-token prompt, 8 branches x 256)
    cfg, flat, eng = make(C1, 7)
    seqs = O.grouped_corpus(1, 8, 512, 256, cfg.vocab_size, 3)
    for sb in (True, False):
        r, worst = tree_case(cfg, seqs, flat, eng, tt.SchedulerConfig(sibling_batch=sb))
        print("c1 worst tensor", worst, "batches", r.num_batches)


def test_kat_zero_weights_and_uniform_logits():
    cfg, flat, eng = make(SMALL, 8)
    seqs = O.grouped_corpus(2, 3, 20, 30, cfg.vocab_size, 11, prompt_weight=0.0)
    zs = [tt.TokenSequence(s.seq_id, s.tokens, [0.0] * len(s.tokens)) for s in seqs]
    eng.zero_gradients()
    r = eng.tree_train_step(tt.build_prefix_tree(zs))
    assert r.total_loss == 0.0 and not eng.gradients().any()
    # zero output head -> uniform logits -> loss = ln V per weighted position
    P = O.unflatten(cfg, flat.copy())
    P["output_head"][:] = 0.0
    eng.upload_params(O.flatten(cfg, P))
    ones = [tt.TokenSequence(s.seq_id, s.tokens, [1.0] * len(s.tokens)) for s in seqs]
    eng.zero_gradients()
    r = eng.tree_train_step(tt.build_prefix_tree(ones))
    npos = sum(len(s.tokens) - 1 for s in seqs)
    assert r.total_loss == pytest.approx(npos * math.log(cfg.vocab_size), rel=1e-5)


def test_errors_surface_as_exceptions():
    cfg, flat, eng = make(SMALL, 9)
    with pytest.raises(ValueError):
        eng.forward_segment([cfg.vocab_size + 5])
    with pytest.raises(ValueError):
        eng.forward_segment([])
    long = [tt.TokenSequence(0, [1] * (cfg.max_position + 1))]
    with pytest.raises(ValueError):
        eng.tree_train_step(tt.build_prefix_tree(long))


@pytest.mark.parametrize("cfgt", [SMALL, DH128], ids=["dh64_fused_bwd", "dh128_split_bwd"])
def test_attention_long_segments_vs_oracle(cfgt):
    # segments longer than one 128-query block on both sides of every key block, plus a shared
    # response stem: the fused dh = 64 backward (dQ partials reduced across key blocks) and the dh = 128
    # query-/key-parallel pair
    cfg, flat, eng = make(cfgt, 12)
    seqs = O.grouped_corpus(2, 4, 150, 200, cfg.vocab_size, 13, shared_response=20, weight_jitter=True)
    tree_case(cfg, seqs, flat, eng, tt.SchedulerConfig())


@pytest.mark.parametrize("ce_stats,logits_bf16", [(0, 0), (1, 0), (1, 1)])
def test_lm_head_ce_variants_vs_oracle(ce_stats, logits_bf16):
    # weighted_nll (model.hpp:643-677): CE from the GEMM-epilogue softmax statistics (ce_stats 1) over
    # fp32 logits or bf16 logits relative to the 32-column group max (logits_bf16 1, the default), or
    # from its own two passes over fp32 logits (0) — same step against the oracle
    cfg, flat, eng = make(SMALL, 18)
    eng.set_option("ce_stats", ce_stats)
    eng.set_option("logits_bf16", logits_bf16)
    seqs = O.grouped_corpus(2, 4, 150, 200, cfg.vocab_size, 19, shared_response=20, weight_jitter=True)
    tree_case(cfg, seqs, flat, eng, tt.SchedulerConfig())


@pytest.mark.parametrize("chunk", [37, 64, 1000])
def test_chunked_backward_vs_oracle(chunk):
    # chunk_boundaries / chunked_backward: older chunks recomputed from the stack
    cfg, flat, eng = make(SMALL, 14)
    seqs = O.grouped_corpus(2, 3, 150, 130, cfg.vocab_size, 15, shared_response=40, weight_jitter=True)
    r, _ = tree_case(cfg, seqs, flat, eng, tt.SchedulerConfig(chunk_len=chunk))
    root = O.build_prefix_tree(seqs)
    longest = max(len(n.tokens) for n in O.preorder(root))
    if chunk < longest:
        assert r.recompute_tokens > 0 and r.num_chunks > r.num_segments
    else:
        assert r.recompute_tokens == 0
    assert r.recompute_tokens <= r.forward_tokens


def test_chunk_invariance_and_leaf_kv_skip_on_device():
    # gradients independent of chunk_len and leaf_kv_skip; skip never
    # increases peak live KV, which stays within the longest path
    cfg, flat, eng = make(SMALL, 16)
    seqs = O.grouped_corpus(2, 4, 90, 110, cfg.vocab_size, 17, shared_response=12)
    tree = tt.build_prefix_tree([tt.TokenSequence(s.seq_id, s.tokens, s.weights) for s in seqs])
    out = {}
    for key, sc in (("base", tt.SchedulerConfig(sibling_batch=False)),
                    ("chunk", tt.SchedulerConfig(sibling_batch=False, chunk_len=29)),
                    ("skip", tt.SchedulerConfig(sibling_batch=False, leaf_kv_skip=True))):
        eng.zero_gradients()
        out[key] = (eng.tree_train_step(tree, sc), eng.gradients().astype(np.float64))
    base_r, base_g = out["base"]
    for key in ("chunk", "skip"):
        r, g = out[key]
        assert abs(r.total_loss - base_r.total_loss) <= 1e-3 * abs(base_r.total_loss)
        check_grads(cfg, g, base_g, tol=1e-2, cos_tol=0.9999)
    assert out["skip"][0].peak_live_kv_tokens <= base_r.peak_live_kv_tokens
    assert out["skip"][0].peak_live_kv_tokens <= tree.stats()["max_path_tokens"]
    assert out["skip"][0].recompute_tokens <= base_r.recompute_tokens


def _shape_property(cfgt, seqs, chunk=0):
    """Full-size model: tree step == flat per-sequence step on the device."""
    eng = tt.Engine(tt.ModelConfig(*cfgt))
    eng.init_params_random(3)
    tseqs = [tt.TokenSequence(s.seq_id, s.tokens, s.weights) for s in seqs]
    eng.zero_gradients()
    rt = eng.tree_train_step(tt.build_prefix_tree(tseqs), tt.SchedulerConfig(chunk_len=chunk))
    gt = eng.gradients().astype(np.float64)
    eng.zero_gradients()
    rd = eng.dense_train_step(tseqs)
    gd = eng.gradients().astype(np.float64)
    assert np.isfinite(rt.total_loss) and abs(rt.total_loss - rd.total_loss) <= 2e-3 * abs(rd.total_loss)
    cos = float(gt @ gd / (np.linalg.norm(gt) * np.linalg.norm(gd)))
    rel = float(np.linalg.norm(gt - gd) / np.linalg.norm(gd))
    assert cos >= 0.9999 and rel <= 2e-2, (cos, rel)
    assert rd.forward_tokens == sum(len(s.tokens) for s in seqs)
    return rt, rd


def test_c3_shape_deep_tree_tree_equals_flat():
    # BASELINE configs[2]: 1.5B shape, deep multi-turn tree (4 levels, fan-out 4; 8K path); the
    # chunked backward bounds activation memory by chunk_len (DFS stack-memory stress)
    rng = np.random.default_rng(21)
    V = 151936
    seqs, sid = [], 0

    def rec(prefix, depth):
        nonlocal sid
        if depth == 4:
            w = [0.0] * 512 + [1.0] * (len(prefix) - 512)
            seqs.append(O.TokenSequence(sid, prefix, w))
            sid += 1
            return
        firsts = rng.choice(V, size=4 if depth else 1, replace=False)
        for f in firsts:
            rec(prefix + [int(f)] + rng.integers(0, V, 2047).tolist(), depth + 1)

    rec([], 0)  # 4 levels of 2048-token nodes -> 64 leaves, 8192-token paths
    rt, rd = _shape_property((V, 1536, 12, 28, 8960, 8200), seqs, chunk=512)
    assert rt.recompute_tokens > 0


def test_c4_shape_7b_tree_equals_flat():
    # BASELINE configs[3] model (7B shape) on one rollout group
    seqs = O.grouped_corpus(1, 4, 512, 768, 152064, 23)
    _shape_property((152064, 3584, 28, 28, 18944, 1300), seqs)


@pytest.mark.parametrize("root_tokens", [0, 300, 4096])
def test_multi_root_batching_vs_oracle(root_tokens):
    # several prompt trees (forest roots whose children are all leaves) pushed as one multi-root
    # batch; each root's leaves attend to that root's rows only (prefix row base != 0). 0 = off.
    cfg, flat, eng = make(SMALL, 31)
    eng.set_option("root_batch_tokens", root_tokens)
    seqs = O.grouped_corpus(5, 3, 90, 70, cfg.vocab_size, 32, weight_jitter=True)
    r, _ = tree_case(cfg, seqs, flat, eng, tt.SchedulerConfig())
    tree = tt.build_prefix_tree([tt.TokenSequence(s.seq_id, s.tokens, s.weights) for s in seqs])
    plan = eng.plan(tree, tt.SchedulerConfig())
    assert plan.trace() == tree.dfs_trace()  # the logical DFS trace is unchanged by batching
    if root_tokens >= 5 * 90:
        assert r.num_batches < 5 * 2  # prompts share pushes


def test_plan_cuda_graph_replay_matches_eager():
    # a prepared plan is captured as one CUDA graph on its second execute and replayed afterwards;
    # replays must give the eager step's loss and gradients (same kernels, same order)
    cfg, flat, eng = make(SMALL, 41)
    seqs = O.grouped_corpus(3, 4, 60, 50, cfg.vocab_size, 42, weight_jitter=True)
    tree = tt.build_prefix_tree([tt.TokenSequence(s.seq_id, s.tokens, s.weights) for s in seqs])
    plan = eng.plan(tree, tt.SchedulerConfig())
    outs = []
    for _ in range(4):  # eager, capture + launch, replay, replay
        eng.zero_gradients()
        r = plan.execute()
        outs.append((r.total_loss, eng.gradients().copy(), r.num_launches))
    # fp32 atomics (dK/dV stack, split-K reduce-add, gain gradients) make the summation order, hence
    # the last bits, run-to-run dependent — eager runs differ from each other the same way
    for loss, g, nl in outs[1:]:
        assert abs(loss - outs[0][0]) <= 1e-9 * abs(outs[0][0]) and nl == outs[0][2]
        assert rel(g, outs[0][1]) <= 1e-5
    eng.set_option("cuda_graph", 0)
    eng.zero_gradients()
    r = plan.execute()
    assert abs(r.total_loss - outs[0][0]) <= 1e-9 * abs(outs[0][0]) and rel(eng.gradients(), outs[0][1]) <= 1e-5


@pytest.mark.parametrize("spec", ["small", "dh128"])
def test_programmatic_dependent_launch_matches_stream_order(spec):
    # every kernel launched with PDL (option pdl=1: the successor's prologue overlaps the predecessor's
    # tail, griddepcontrol.wait before any global access) must give the plain stream-ordered step
    # (pdl=0) and the oracle, eager and graph-replayed
    cfg, flat, eng = make(SMALL if spec == "small" else DH128, 47)
    seqs = O.grouped_corpus(3, 4, 60, 50, cfg.vocab_size, 48, weight_jitter=True)
    tree = tt.build_prefix_tree([tt.TokenSequence(s.seq_id, s.tokens, s.weights) for s in seqs])
    plan = eng.plan(tree, tt.SchedulerConfig())
    outs = {}
    for mode in (0, 1, 2):
        eng.set_option("pdl", mode)
        for _ in range(3):  # eager, capture + launch, replay
            eng.zero_gradients()
            r = plan.execute()
            outs.setdefault(mode, []).append((r.total_loss, eng.gradients().copy()))
    l0, g0 = outs[0][0]
    for mode in (1, 2):
        for loss, g in outs[mode]:
            assert abs(loss - l0) <= 1e-9 * abs(l0) and rel(g, g0) <= 1e-5
    ref = O.tree_train_step(cfg, flat, O.order_children(O.build_prefix_tree(seqs), "subtree_tokens_desc"), seqs)
    assert abs(outs[1][-1][0] - ref.total_loss) <= 5e-3 * abs(ref.total_loss)
    assert rel(outs[1][-1][1], ref.grads) <= 2e-2
    with pytest.raises(ValueError):
        eng.set_option("pdl", 3)


def test_plan_execute_async_overlapping_next_plan():
    # tt_plan_execute_async + tt_plan_wait: while step k runs, the next tree is built and planned
    # (its metadata goes over the copy stream); every step matches the synchronous execute, and a
    # second async step cannot be enqueued while one is in flight
    cfg, flat, eng = make(SMALL, 43)
    corpora = [O.grouped_corpus(2, 4, 50 + 10 * k, 40, cfg.vocab_size, 44 + k, weight_jitter=True) for k in range(3)]
    trees = lambda k: tt.build_prefix_tree([tt.TokenSequence(s.seq_id, s.tokens, s.weights) for s in corpora[k]])
    ref = []
    for k in range(3):
        eng.zero_gradients()
        r = eng.plan(trees(k), tt.SchedulerConfig()).execute()
        ref.append((r.total_loss, eng.gradients().copy()))
    plan = eng.plan(trees(0), tt.SchedulerConfig())
    for k in range(3):
        eng.zero_gradients()
        plan.execute_async()
        with pytest.raises(RuntimeError):
            plan.execute_async()
        nxt = eng.plan(trees(k + 1), tt.SchedulerConfig()) if k + 1 < 3 else None
        r = plan.wait()
        assert abs(r.total_loss - ref[k][0]) <= 1e-9 * abs(ref[k][0])
        assert rel(eng.gradients(), ref[k][1]) <= 1e-5
        plan = nxt
    with pytest.raises(ValueError):  # nothing in flight
        eng.plan(trees(0), tt.SchedulerConfig()).wait()
