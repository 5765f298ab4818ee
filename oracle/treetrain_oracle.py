"""CPU ORACLE — TEST INFRASTRUCTURE ONLY.

A numpy (float64) restatement of the reference's DFS prefix-tree forward/backward path:
  * the model core of /root/reference/proj/core/include/treetrain/model.hpp
    (forward_segment :328-463, backward_segment :474-633, weighted_nll :643-677,
    for_each_tensor :42-59, helpers :239-283, attention_probs :298-321);
  * the SPEC-only modules the reference does not ship:
    prefix tree :113-197, DFS scheduler :199-285, dense oracle :287-340, partitioner :342-431.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg may import
this module, and only as the checker. The product path (paper_2602_00482_b200, libtreetrain_b200.so)
never calls it.

Parity pin: this restatement is checked against the reference itself, compiled from
/root/reference by oracle/Makefile into oracle/_ref/libttref.so (tests/test_oracle_vs_ref.py),
and against the golden vectors in tests/golden/ produced from that library by
oracle/make_golden.py.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import Dict, List, Optional, Sequence, Tuple

import numpy as np

RMS_EPS = 1e-6  # model.hpp:18


# ----------------------------------------------------------------------------- config / params
@dataclass(frozen=True)
class ModelConfig:
    """model_config.hpp:19-37."""

    vocab_size: int
    d_model: int
    n_heads: int
    n_layers: int
    d_ff: int
    max_position: int

    @property
    def head_dim(self) -> int:  # model_config.hpp:28
        return self.d_model // self.n_heads

    def validate(self) -> None:  # model_config.hpp:30-36
        if min(self.vocab_size, self.d_model, self.n_heads, self.n_layers, self.d_ff, self.max_position) < 1:
            raise ValueError("ModelConfig: all counts must be >= 1")
        if self.d_model % self.n_heads:
            raise ValueError("ModelConfig: d_model must be divisible by n_heads")


def tensor_specs(cfg: ModelConfig) -> List[Tuple[str, Tuple[int, ...]]]:
    """Canonical tensor order = serialization and gradient-output order (model.hpp:42-59)."""
    d, V, F = cfg.d_model, cfg.vocab_size, cfg.d_ff
    out = [("embedding", (V, d))]
    for i in range(cfg.n_layers):
        b = f"layers.{i}."
        out += [
            (b + "attn_norm_gain", (d,)),
            (b + "w_q", (d, d)),
            (b + "w_k", (d, d)),
            (b + "w_v", (d, d)),
            (b + "w_o", (d, d)),
            (b + "mlp_norm_gain", (d,)),
            (b + "w_mlp_in", (d, F)),
            (b + "w_mlp_out", (F, d)),
        ]
    out += [("final_norm_gain", (d,)), ("output_head", (d, V))]
    return out


def param_count(cfg: ModelConfig) -> int:
    return sum(int(np.prod(s)) for _, s in tensor_specs(cfg))


def unflatten(cfg: ModelConfig, flat: np.ndarray) -> Dict[str, np.ndarray]:
    out, o = {}, 0
    for name, shape in tensor_specs(cfg):
        n = int(np.prod(shape))
        out[name] = flat[o:o + n].reshape(shape)
        o += n
    assert o == flat.size, (o, flat.size)
    return out


def flatten(cfg: ModelConfig, p: Dict[str, np.ndarray]) -> np.ndarray:
    return np.concatenate([np.asarray(p[name], dtype=np.float64).reshape(-1) for name, _ in tensor_specs(cfg)])


def zero_like_params(cfg: ModelConfig) -> Dict[str, np.ndarray]:
    return {name: np.zeros(shape) for name, shape in tensor_specs(cfg)}


def random_params(cfg: ModelConfig, seed: int, std: float = 0.02) -> np.ndarray:
    """N(0, std) weights and unit gains (the distribution of init_params, model.hpp:119-142;
    numpy's generator, not the reference's mt19937_64 stream)."""
    rng = np.random.default_rng(seed)
    parts = []
    for name, shape in tensor_specs(cfg):
        if name.endswith("norm_gain"):
            parts.append(np.ones(int(np.prod(shape))))
        else:
            parts.append(rng.normal(0.0, std, size=int(np.prod(shape))))
    return np.concatenate(parts)


def round_bf16(x: np.ndarray) -> np.ndarray:
    """Round float64 values to the nearest bfloat16 (round-to-nearest-even), returned as float64."""
    f = np.asarray(x, dtype=np.float32)
    u = f.view(np.uint32).astype(np.uint64)
    u = (u + 0x7FFF + ((u >> 16) & 1)) & 0xFFFF0000
    return u.astype(np.uint32).view(np.float32).astype(np.float64)


# ----------------------------------------------------------------------------- elementwise helpers
def positional_encoding(positions: np.ndarray, d: int) -> np.ndarray:
    """add_positional_encoding (model.hpp:239-248): sin on even, cos on odd columns, double."""
    i = np.arange(0, (d + 1) // 2)
    freq = np.array([math.pow(10000.0, -float(2 * k) / float(d)) for k in i])
    ang = positions[:, None].astype(np.float64) * freq[None, :]
    pe = np.zeros((positions.size, d))
    pe[:, 0::2] = np.sin(ang)[:, : (d + 1) // 2]
    if d > 1:
        pe[:, 1::2] = np.cos(ang)[:, : d // 2]
    return pe


def rms_inv(x: np.ndarray) -> np.ndarray:
    """rms_inv (model.hpp:250-256), row-wise."""
    return 1.0 / np.sqrt(np.mean(x * x, axis=-1) + RMS_EPS)


def rmsnorm_backward(gy, x, inv, gain):
    """rmsnorm_backward (model.hpp:258-271): returns (grad_x increment, grad_gain increment)."""
    d = x.shape[-1]
    dot = np.sum(gy * gain[None, :] * x, axis=-1)
    scale = dot * inv ** 3 / d
    gx = gy * gain[None, :] * inv[:, None] - x * scale[:, None]
    gg = np.sum(gy * x * inv[:, None], axis=0)
    return gx, gg


def silu(u):  # model.hpp:273-277
    return u / (1.0 + np.exp(-u))


def silu_derivative(u):  # model.hpp:279-283
    s = 1.0 / (1.0 + np.exp(-u))
    return s * (1.0 + u * (1.0 - s))


# ----------------------------------------------------------------------------- segment forward/backward
@dataclass
class SegmentActs:
    """SegmentActivations (model.hpp:211-230)."""

    start: int
    tokens: np.ndarray
    layers: List[dict] = field(default_factory=list)
    x_final: Optional[np.ndarray] = None
    inv_final: Optional[np.ndarray] = None


def _attention(q, K, V, S, H, dh):
    """attention_probs + PV (model.hpp:298-321, 386-408): query t attends keys [0, S+t]."""
    L = q.shape[0]
    ctx = K.shape[0]
    qh = q.reshape(L, H, dh).transpose(1, 0, 2)
    kh = K.reshape(ctx, H, dh).transpose(1, 0, 2)
    vh = V.reshape(ctx, H, dh).transpose(1, 0, 2)
    scale = 1.0 / math.sqrt(dh)
    s = np.einsum("htc,hjc->htj", qh, kh) * scale
    mask = np.arange(ctx)[None, :] > (S + np.arange(L))[:, None]
    s = np.where(mask[None], -np.inf, s)
    m = s.max(axis=-1, keepdims=True)
    p = np.exp(s - m)
    p = p / p.sum(axis=-1, keepdims=True)
    o = np.einsum("htj,hjc->htc", p, vh)
    return o.transpose(1, 0, 2).reshape(L, H * dh), p


def forward_segment(cfg: ModelConfig, P: Dict[str, np.ndarray], prefix_k: np.ndarray, prefix_v: np.ndarray,
                    tokens: Sequence[int], start: int, want_acts: bool = True):
    """forward_segment (model.hpp:328-463).

    prefix_k/prefix_v: [n_layers, S, d] — the KVView flattened to one array per layer.
    Returns (logits [len x V], (k, v) each [n_layers, len, d], acts or None).
    """
    tokens = np.asarray(tokens, dtype=np.int64)
    n = tokens.size
    if n == 0:
        raise ValueError("forward_segment: empty token list")
    if prefix_k.shape[1] != start:
        raise ValueError("forward_segment: start_position does not match prefix length")
    if start + n > cfg.max_position:
        raise ValueError("forward_segment: position overflow beyond max_position")
    if tokens.min() < 0 or tokens.max() >= cfg.vocab_size:
        raise ValueError("forward_segment: token id out of vocab range")
    d, H, dh = cfg.d_model, cfg.n_heads, cfg.head_dim
    x = P["embedding"][tokens] + positional_encoding(start + np.arange(n), d)
    acts = SegmentActs(start, tokens) if want_acts else None
    ks, vs = [], []
    for li in range(cfg.n_layers):
        b = f"layers.{li}."
        inv1 = rms_inv(x)
        n1 = x * inv1[:, None] * P[b + "attn_norm_gain"][None, :]
        q, k, v = n1 @ P[b + "w_q"], n1 @ P[b + "w_k"], n1 @ P[b + "w_v"]
        K = np.concatenate([prefix_k[li], k], 0)
        V = np.concatenate([prefix_v[li], v], 0)
        attn, _ = _attention(q, K, V, start, H, dh)
        proj = attn @ P[b + "w_o"]
        if acts is not None:
            acts.layers.append(dict(x_in=x.copy(), inv1=inv1, q=q, k=k, v=v, attn=attn))
        ks.append(k)
        vs.append(v)
        x = x + proj
        inv2 = rms_inv(x)
        n2 = x * inv2[:, None] * P[b + "mlp_norm_gain"][None, :]
        h = n2 @ P[b + "w_mlp_in"]
        if acts is not None:
            acts.layers[-1].update(x_mid=x.copy(), inv2=inv2, h=h)
        x = x + silu(h) @ P[b + "w_mlp_out"]
    invf = rms_inv(x)
    nf = x * invf[:, None] * P["final_norm_gain"][None, :]
    if acts is not None:
        acts.x_final, acts.inv_final = x, invf
    logits = nf @ P["output_head"]
    return logits, (np.stack(ks), np.stack(vs)), acts


def backward_segment(cfg: ModelConfig, P: Dict[str, np.ndarray], acts: SegmentActs, prefix_k, prefix_v,
                     grads: Dict[str, np.ndarray], grad_logits=None, grad_new_k=None, grad_new_v=None):
    """backward_segment (model.hpp:474-633). Adds into `grads`; returns (gK, gV) [n_layers, S, d]."""
    S, n = acts.start, acts.tokens.size
    d, H, dh = cfg.d_model, cfg.n_heads, cfg.head_dim
    if prefix_k.shape[1] != S:
        raise ValueError("backward_segment: prefix length does not match activations")
    if grad_logits is not None and grad_logits.shape != (n, cfg.vocab_size):
        raise ValueError("backward_segment: grad_logits shape mismatch")
    scale = 1.0 / math.sqrt(dh)
    gpk = np.zeros((cfg.n_layers, S, d))
    gpv = np.zeros((cfg.n_layers, S, d))
    gx = np.zeros((n, d))
    if grad_logits is not None:  # model.hpp:500-512
        c = acts.x_final * acts.inv_final[:, None] * P["final_norm_gain"][None, :]
        grads["output_head"] += c.T @ grad_logits
        gc = grad_logits @ P["output_head"].T
        dx, dg = rmsnorm_backward(gc, acts.x_final, acts.inv_final, P["final_norm_gain"])
        gx += dx
        grads["final_norm_gain"] += dg
    for li in reversed(range(cfg.n_layers)):  # model.hpp:516-625
        b = f"layers.{li}."
        la = acts.layers[li]
        act = silu(la["h"])
        grads[b + "w_mlp_out"] += act.T @ gx
        g_act = gx @ P[b + "w_mlp_out"].T
        g_h = g_act * silu_derivative(la["h"])
        n2 = la["x_mid"] * la["inv2"][:, None] * P[b + "mlp_norm_gain"][None, :]
        grads[b + "w_mlp_in"] += n2.T @ g_h
        g_n2 = g_h @ P[b + "w_mlp_in"].T
        dx, dg = rmsnorm_backward(g_n2, la["x_mid"], la["inv2"], P[b + "mlp_norm_gain"])
        gx_mid = gx + dx
        grads[b + "mlp_norm_gain"] += dg
        grads[b + "w_o"] += la["attn"].T @ gx_mid
        g_attn = gx_mid @ P[b + "w_o"].T
        # attention backward (model.hpp:546-604), probs recomputed
        K = np.concatenate([prefix_k[li], la["k"]], 0)
        V = np.concatenate([prefix_v[li], la["v"]], 0)
        _, p = _attention(la["q"], K, V, S, H, dh)  # [H, n, ctx]
        ctx = K.shape[0]
        ga = g_attn.reshape(n, H, dh).transpose(1, 0, 2)
        vh = V.reshape(ctx, H, dh).transpose(1, 0, 2)
        kh = K.reshape(ctx, H, dh).transpose(1, 0, 2)
        qh = la["q"].reshape(n, H, dh).transpose(1, 0, 2)
        gp = np.einsum("htc,hjc->htj", ga, vh)
        dot = np.sum(p * gp, axis=-1, keepdims=True)
        gs = p * (gp - dot) * scale
        gq = np.einsum("htj,hjc->htc", gs, kh).transpose(1, 0, 2).reshape(n, d)
        gK = np.einsum("htj,htc->hjc", gs, qh).transpose(1, 0, 2).reshape(ctx, d)
        gV = np.einsum("htj,htc->hjc", p, ga).transpose(1, 0, 2).reshape(ctx, d)
        gpk[li] += gK[:S]
        gpv[li] += gV[:S]
        gk_own = gK[S:] + (grad_new_k[li] if grad_new_k is not None else 0.0)
        gv_own = gV[S:] + (grad_new_v[li] if grad_new_v is not None else 0.0)
        n1 = la["x_in"] * la["inv1"][:, None] * P[b + "attn_norm_gain"][None, :]
        grads[b + "w_q"] += n1.T @ gq
        grads[b + "w_k"] += n1.T @ gk_own
        grads[b + "w_v"] += n1.T @ gv_own
        g_n1 = gq @ P[b + "w_q"].T + gk_own @ P[b + "w_k"].T + gv_own @ P[b + "w_v"].T
        dx, dg = rmsnorm_backward(g_n1, la["x_in"], la["inv1"], P[b + "attn_norm_gain"])
        gx = gx_mid + dx
        grads[b + "attn_norm_gain"] += dg
    np.add.at(grads["embedding"], acts.tokens, gx)  # model.hpp:627-630
    return gpk, gpv


def weighted_nll(logits: np.ndarray, targets: Sequence[int], weights: Sequence[float]):
    """weighted_nll (model.hpp:643-677). Returns (loss, grad_logits)."""
    n, V = logits.shape
    targets = np.asarray(targets, dtype=np.int64)
    weights = np.asarray(weights, dtype=np.float64)
    if targets.size != n or weights.size != n:
        raise ValueError("weighted_nll: one target and weight per loss position")
    if n and (targets.min() < 0 or targets.max() >= V):
        raise ValueError("weighted_nll: target id out of vocab range")
    if not np.all(np.isfinite(weights)):
        raise ValueError("weighted_nll: non-finite weight")
    grad = np.zeros_like(logits)
    loss = 0.0
    for p in range(n):
        w = weights[p]
        if w == 0.0:
            continue
        row = logits[p]
        m = row.max()
        e = np.exp(row - m)
        z = e.sum()
        grad[p] = w * (e / z)
        grad[p, targets[p]] -= w
        loss += w * (m + math.log(z) - row[targets[p]])
    return loss, grad


def weighted_nll_pairs(logits: np.ndarray, rows, targets, weights):
    """Multi-target extension: one weighted_nll term per (row, target, weight) pair."""
    grad = np.zeros_like(logits)
    loss = 0.0
    for r, t, w in zip(rows, targets, weights):
        l1, g1 = weighted_nll(logits[r:r + 1], [t], [w])
        loss += l1
        grad[r] += g1[0]
    return loss, grad


# ----------------------------------------------------------------------------- prefix tree
@dataclass
class TokenSequence:
    """token_sequence.hpp:15-21 (seq_id is the integer index in the input list)."""

    seq_id: int
    tokens: List[int]
    weights: List[float]


@dataclass
class TreeNode:
    tokens: List[int] = field(default_factory=list)
    children: List["TreeNode"] = field(default_factory=list)
    leaf_marks: List[int] = field(default_factory=list)  # seq_ids ending at this node
    subtree_seqs: List[int] = field(default_factory=list)  # seq_ids whose path passes through


POLICIES = ("as_built", "lexicographic", "subtree_tokens_desc", "subtree_tokens_asc")


def build_prefix_tree(seqs: Sequence[TokenSequence]) -> TreeNode:
    """build_prefix_tree: radix-compressed trie; children in first-appearance
    (as_built) order; a sequence ending inside the trie yields an internal leaf_mark."""
    if not seqs:
        raise ValueError("build_prefix_tree: empty sequence list")
    ids = [s.seq_id for s in seqs]
    if len(set(ids)) != len(ids):
        raise ValueError("build_prefix_tree: duplicate seq_id")
    # uncompressed trie: node = dict(children: {tok: node}, order: [tok], marks: [])
    root = {"tok": None, "children": {}, "order": [], "marks": [], "seqs": []}
    for s in seqs:
        if len(s.tokens) == 0:
            raise ValueError("build_prefix_tree: empty token list")
        cur = root
        for t in s.tokens:
            nxt = cur["children"].get(t)
            if nxt is None:
                nxt = {"tok": t, "children": {}, "order": [], "marks": [], "seqs": []}
                cur["children"][t] = nxt
                cur["order"].append(t)
            cur = nxt
            cur["seqs"].append(s.seq_id)
        cur["marks"].append(s.seq_id)

    def compress(u) -> TreeNode:
        node = TreeNode(tokens=[u["tok"]], leaf_marks=list(u["marks"]), subtree_seqs=list(u["seqs"]))
        while len(u["order"]) == 1 and not u["marks"]:
            u = u["children"][u["order"][0]]
            node.tokens.append(u["tok"])
            node.leaf_marks = list(u["marks"])
        node.children = [compress(u["children"][t]) for t in u["order"]]
        return node

    vroot = TreeNode(tokens=[], children=[compress(root["children"][t]) for t in root["order"]])
    vroot.subtree_seqs = [s.seq_id for s in seqs]
    return vroot


def subtree_tokens(n: TreeNode) -> int:
    return len(n.tokens) + sum(subtree_tokens(c) for c in n.children)


def tree_token_count(root: TreeNode) -> int:
    """tree_token_count."""
    return subtree_tokens(root)


def max_path_tokens(n: TreeNode) -> int:
    return len(n.tokens) + max((max_path_tokens(c) for c in n.children), default=0)


def num_nodes(n: TreeNode) -> int:
    return (1 if n.tokens else 0) + sum(num_nodes(c) for c in n.children)


def order_children(root: TreeNode, policy: str) -> TreeNode:
    """order_children: recursive, stable tie-break by first token ascending."""
    if policy not in POLICIES:
        raise ValueError(f"unknown policy {policy}")

    def rec(n: TreeNode):
        if policy == "lexicographic":
            n.children.sort(key=lambda c: c.tokens[0])
        elif policy == "subtree_tokens_desc":
            n.children.sort(key=lambda c: (-subtree_tokens(c), c.tokens[0]))
        elif policy == "subtree_tokens_asc":
            n.children.sort(key=lambda c: (subtree_tokens(c), c.tokens[0]))
        for c in n.children:
            rec(c)

    rec(root)
    return root


def serialize_tree(root: TreeNode) -> str:
    """Canonical pre-order text: one line per node `depth len tok.. | marks id.. | nchildren`."""
    out = []

    def rec(n: TreeNode, depth: int):
        out.append(f"{depth} {len(n.tokens)} {' '.join(map(str, n.tokens))} | {' '.join(map(str, sorted(n.leaf_marks)))} | {len(n.children)}\n")
        for c in n.children:
            rec(c, depth + 1)

    for c in root.children:
        rec(c, 0)
    return "".join(out)


def preorder(root: TreeNode) -> List[TreeNode]:
    out = []

    def rec(n):
        out.append(n)
        for c in n.children:
            rec(c)

    for c in root.children:
        rec(c)
    return out


def dfs_trace(root: TreeNode) -> str:
    """DFS event trace: `PUSH id` in pre-order, `POP id` in post-order, ids =
    pre-order index in the ordered tree."""
    ids = {id(n): i for i, n in enumerate(preorder(root))}
    out = []

    def rec(n):
        out.append(f"PUSH {ids[id(n)]}\n")
        for c in n.children:
            rec(c)
        out.append(f"POP {ids[id(n)]}\n")

    for c in root.children:
        rec(c)
    return "".join(out)


def lexicographic_sort(seqs: Sequence[TokenSequence]) -> List[TokenSequence]:
    """lexicographic_sort: token-id order, stable on ties by seq_id."""
    return sorted(seqs, key=lambda s: (list(s.tokens), s.seq_id))


def duplication_factor(seqs: Sequence[TokenSequence]) -> float:
    """duplication_factor."""
    return sum(len(s.tokens) for s in seqs) / tree_token_count(build_prefix_tree(seqs))


def node_loss_pairs(node: TreeNode, start: int, seq_by_id: Dict[int, TokenSequence]):
    """Per-node (row, target, weight) loss pairs (verified against a dense oracle in
    SURVEY App. B.4): rows 0..len-2 predict the next in-node token with the summed weight of every
    sequence through the node; the last row predicts each child's first token with the summed
    weight of the sequences through that child. Zero weights are dropped (model.hpp:657)."""
    rows, tgts, ws = [], [], []
    ids = sorted(node.subtree_seqs)
    L = len(node.tokens)
    for t in range(L - 1):
        pos = start + t + 1
        w = 0.0
        for i in ids:
            w += seq_by_id[i].weights[pos]
        if w != 0.0:
            rows.append(t)
            tgts.append(node.tokens[t + 1])
            ws.append(w)
    for c in node.children:
        pos = start + L
        w = 0.0
        for i in sorted(c.subtree_seqs):
            w += seq_by_id[i].weights[pos]
        if w != 0.0:
            rows.append(L - 1)
            tgts.append(c.tokens[0])
            ws.append(w)
    return rows, tgts, ws


def annotate_tree(root: TreeNode, seqs: Sequence[TokenSequence]):
    """Yield (node, start, pairs) in DFS pre-order."""
    by_id = {s.seq_id: s for s in seqs}
    out = []

    def rec(n, S):
        out.append((n, S, node_loss_pairs(n, S, by_id)))
        for c in n.children:
            rec(c, S + len(n.tokens))

    for c in root.children:
        rec(c, 0)
    return out


# ----------------------------------------------------------------------------- DFS scheduler
def chunk_boundaries(segment_len: int, chunk_len: int) -> List[Tuple[int, int]]:
    """chunk_boundaries."""
    if segment_len < 1 or chunk_len < 1:
        raise ValueError("chunk_boundaries: lengths must be >= 1")
    return [(a, min(a + chunk_len, segment_len)) for a in range(0, segment_len, chunk_len)]


@dataclass
class TrainStepResult:
    total_loss: float
    grads: np.ndarray
    forward_tokens: int = 0
    backward_tokens: int = 0
    peak_live_kv_tokens: int = 0
    num_segments: int = 0
    trace: str = ""


def tree_train_step(cfg: ModelConfig, flat_params: np.ndarray, root: TreeNode, seqs: Sequence[TokenSequence],
                    ) -> TrainStepResult:
    """tree_train_step (design decisions :271-276): recursive DFS in the tree's
    child order. PUSH forwards a node from the stack KV; the node's own loss is
    deferred to its POP, where backward_segment runs once with upstream = own-loss grad_logits +
    the frame's accumulated KVGrad; grad_prefix is scattered into the ancestor frames."""
    P = unflatten(cfg, flat_params)
    G = zero_like_params(cfg)
    by_id = {s.seq_id: s for s in seqs}
    L, d = cfg.n_layers, cfg.d_model
    depth_max = max_path_tokens(root)
    if depth_max > cfg.max_position:
        raise ValueError("tree_train_step: path exceeds max_position")
    kstack = np.zeros((L, depth_max, d))
    vstack = np.zeros((L, depth_max, d))
    gk = np.zeros((L, depth_max, d))  # per-frame KVGrad, laid out along the stack rows
    gv = np.zeros((L, depth_max, d))
    ids = {id(n): i for i, n in enumerate(preorder(root))}
    res = TrainStepResult(0.0, None)
    trace = []

    def rec(n: TreeNode, S: int):
        ln = len(n.tokens)
        trace.append(f"PUSH {ids[id(n)]}\n")
        logits, (k, v), acts = forward_segment(cfg, P, kstack[:, :S], vstack[:, :S], n.tokens, S)
        res.forward_tokens += ln
        res.num_segments += 1
        kstack[:, S:S + ln] = k
        vstack[:, S:S + ln] = v
        gk[:, S:S + ln] = 0.0
        gv[:, S:S + ln] = 0.0
        res.peak_live_kv_tokens = max(res.peak_live_kv_tokens, S + ln)
        for c in n.children:
            rec(c, S + ln)
        rows, tg, ws = node_loss_pairs(n, S, by_id)
        loss, gl = weighted_nll_pairs(logits, rows, tg, ws)
        if not math.isfinite(loss):
            raise FloatingPointError("tree_train_step: non-finite loss")
        res.total_loss += loss
        gpk, gpv = backward_segment(cfg, P, acts, kstack[:, :S], vstack[:, :S], G, gl,
                                    gk[:, S:S + ln].copy(), gv[:, S:S + ln].copy())
        res.backward_tokens += ln
        gk[:, :S] += gpk
        gv[:, :S] += gpv
        gk[:, S:S + ln] = 0.0
        gv[:, S:S + ln] = 0.0
        trace.append(f"POP {ids[id(n)]}\n")

    for c in root.children:
        rec(c, 0)
    res.grads = flatten(cfg, G)
    res.trace = "".join(trace)
    return res


def dense_train_step(cfg: ModelConfig, flat_params: np.ndarray, seqs: Sequence[TokenSequence]) -> TrainStepResult:
    """dense_train_step: per-sequence full forward + backward, summed in ascending
    seq_id order."""
    P = unflatten(cfg, flat_params)
    G = zero_like_params(cfg)
    L, d = cfg.n_layers, cfg.d_model
    empty = np.zeros((L, 0, d))
    res = TrainStepResult(0.0, None)
    for s in sorted(seqs, key=lambda s: s.seq_id):
        logits, _, acts = forward_segment(cfg, P, empty, empty, s.tokens, 0)
        n = len(s.tokens)
        rows = [t for t in range(n - 1) if s.weights[t + 1] != 0.0]
        loss, gl = weighted_nll_pairs(logits, rows, [s.tokens[t + 1] for t in rows], [s.weights[t + 1] for t in rows])
        res.total_loss += loss
        backward_segment(cfg, P, acts, empty, empty, G, gl)
        res.forward_tokens += n
        res.backward_tokens += n
        res.num_segments += 1
        res.peak_live_kv_tokens = max(res.peak_live_kv_tokens, n)
    res.grads = flatten(cfg, G)
    return res


def compare_grads(a: np.ndarray, b: np.ndarray):
    """compare_grads: (max_abs, max_rel), denominator max(|a|,|b|,1e-12)."""
    diff = np.abs(a - b)
    den = np.maximum(np.maximum(np.abs(a), np.abs(b)), 1e-12)
    return float(diff.max(initial=0.0)), float((diff / den).max(initial=0.0))


# ----------------------------------------------------------------------------- partitioner
def lcp(a: Sequence[int], b: Sequence[int]) -> int:
    n = 0
    for x, y in zip(a, b):
        if x != y:
            break
        n += 1
    return n


def incremental_group_cost(running: int, prev: Optional[Sequence[int]], nxt: Sequence[int]) -> int:
    """incremental_group_cost."""
    if prev is None:
        return len(nxt)
    return running + len(nxt) - lcp(prev, nxt)


def group_tree_cost(seqs: Sequence[TokenSequence]) -> int:
    if not seqs:
        return 0
    return tree_token_count(build_prefix_tree(list(seqs)))


def feasible(tau: int, sorted_seqs: Sequence[TokenSequence], K: int):
    """feasible: greedy left-to-right scan."""
    groups, cost, prev = 1, 0, None
    for s in sorted_seqs:
        if len(s.tokens) > tau:
            return False, len(sorted_seqs)
        c = incremental_group_cost(cost, prev, s.tokens)
        if prev is not None and c > tau:
            groups += 1
            c = len(s.tokens)
        cost, prev = c, s.tokens
    return groups <= K, groups


def _greedy_groups(tau, sorted_seqs):
    groups, cur, cost, prev = [], [], 0, None
    for s in sorted_seqs:
        c = incremental_group_cost(cost, prev, s.tokens)
        if prev is not None and c > tau:
            groups.append(cur)
            cur, c = [], len(s.tokens)
        cur.append(s)
        cost, prev = c, s.tokens
    groups.append(cur)
    return groups


@dataclass
class PartitionPlan:
    groups: List[List[int]]
    costs: List[int]
    max_cost: int
    duplicated_tokens: int


def _plan(groups, all_seqs, K):
    groups = [list(g) for g in groups] + [[] for _ in range(K - len(groups))]
    costs = [group_tree_cost(g) for g in groups]
    dup = sum(costs) - group_tree_cost(all_seqs)
    return PartitionPlan([[s.seq_id for s in g] for g in groups], costs, max(costs), dup)


def partition_contiguous(seqs: Sequence[TokenSequence], K: int) -> PartitionPlan:
    """partition_contiguous: lexicographic sort, integer binary search of the
    smallest feasible tau in [max single-seq cost, combined cost], greedy plan at that tau."""
    if K < 1 or not seqs:
        raise ValueError("partition_contiguous: K >= 1 and N >= 1 required")
    ss = lexicographic_sort(seqs)
    lo, hi = max(len(s.tokens) for s in ss), group_tree_cost(ss)
    while lo < hi:
        mid = (lo + hi) // 2
        if feasible(mid, ss, K)[0]:
            hi = mid
        else:
            lo = mid + 1
    return _plan(_greedy_groups(lo, ss), ss, K)


def brute_force_optimal(seqs: Sequence[TokenSequence], K: int) -> PartitionPlan:
    """brute_force_optimal: DP over contiguous cuts of the lexicographic order."""
    ss = lexicographic_sort(seqs)
    N = len(ss)
    cost = [[0] * (N + 1) for _ in range(N + 1)]
    for i in range(N):
        c, prev = 0, None
        for j in range(i, N):
            c = incremental_group_cost(c, prev, ss[j].tokens)
            prev = ss[j].tokens
            cost[i][j + 1] = c
    INF = float("inf")
    dp = [[INF] * (N + 1) for _ in range(K + 1)]
    cut = [[0] * (N + 1) for _ in range(K + 1)]
    dp[0][0] = 0
    for k in range(1, K + 1):
        for j in range(0, N + 1):
            best, arg = dp[k - 1][j], j  # allow an empty group
            for i in range(0, j):
                v = max(dp[k - 1][i], cost[i][j])
                if v < best:
                    best, arg = v, i
            dp[k][j], cut[k][j] = best, arg
    groups, j = [], N
    for k in range(K, 0, -1):
        i = cut[k][j]
        groups.append(ss[i:j])
        j = i
    groups = [g for g in reversed(groups) if g]
    return _plan(groups, ss, K)


def greedy_least_loaded(seqs: Sequence[TokenSequence], K: int, cost_model: str = "raw_tokens") -> PartitionPlan:
    """greedy_least_loaded: input order, smallest current cost, lowest index."""
    groups: List[List[TokenSequence]] = [[] for _ in range(K)]
    load = [0] * K
    for s in seqs:
        g = min(range(K), key=lambda j: (load[j], j))
        groups[g].append(s)
        load[g] = sum(len(x.tokens) for x in groups[g]) if cost_model == "raw_tokens" else group_tree_cost(groups[g])
    costs = [group_tree_cost(g) for g in groups]
    return PartitionPlan([[s.seq_id for s in g] for g in groups], costs, max(costs),
                         sum(costs) - group_tree_cost(seqs))


def duplication_overhead(plan: PartitionPlan, seqs: Sequence[TokenSequence]) -> int:
    """duplication_overhead."""
    return sum(plan.costs) - group_tree_cost(seqs)


# ----------------------------------------------------------------------------- synthetic corpora
def grouped_corpus(num_prompts: int, group_size: int, prompt_len: int, response_len: int, vocab: int, seed: int,
                   shared_response: int = 0, prompt_weight: float = 0.0, weight_jitter: bool = False):
    """Rollout groups: each prompt (weights 0) followed by `group_size` responses (weights 1) that
    share their first `shared_response` tokens and then diverge (distinct next token)."""
    rng = np.random.default_rng(seed)
    seqs = []
    sid = 0
    for _ in range(num_prompts):
        prompt = rng.integers(0, vocab, prompt_len).tolist()
        stem = rng.integers(0, vocab, shared_response).tolist()
        firsts = rng.permutation(vocab)[:group_size]
        for g in range(group_size):
            rest = [int(firsts[g])] + rng.integers(0, vocab, max(0, response_len - shared_response - 1)).tolist()
            toks = prompt + stem + rest[: response_len - shared_response]
            w = [prompt_weight] * prompt_len + [1.0] * (len(toks) - prompt_len)
            if weight_jitter:
                w = [x * float(rng.uniform(0.1, 2.0)) if x else x for x in w]
            seqs.append(TokenSequence(sid, toks, w))
            sid += 1
    return seqs
