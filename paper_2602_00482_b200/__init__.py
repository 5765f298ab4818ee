"""paper_2602_00482_b200 — B200-native DFS prefix-tree forward/backward engine (AReaL-DTA).

Python host mirror of the reference's C++ API over the C-ABI of libtreetrain_b200.so
(include/treetrain_b200.h). Names follow the reference:

  ModelConfig                (model_config.hpp:19-37)
  TokenSequence              (token_sequence.hpp:15-21)
  PrefixTree / build_prefix_tree / order_children / tree_token_count
  SchedulerConfig / TrainStepResult / Engine.tree_train_step
  Engine.dense_train_step
  Engine.forward_segment / Engine.backward_segment  (model.hpp:328-463, :474-633) on the device stack
  lexicographic_sort / partition_contiguous / greedy_least_loaded

Errors: ValueError <-> std::invalid_argument, RuntimeError <-> std::runtime_error,
FloatingPointError <-> the SPEC's abort on a non-finite loss. There is no CPU fallback.
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass
from typing import List, Optional, Sequence, Tuple

import numpy as np

from . import _native

__all__ = [
    "ModelConfig", "TokenSequence", "SchedulerConfig", "TrainStepResult", "PrefixTree", "Engine",
    "build_prefix_tree", "lexicographic_sort", "partition_contiguous", "greedy_least_loaded", "POLICIES",
    "CorpusSpec", "gen_corpus", "load_corpus_jsonl", "save_corpus_jsonl", "NcclComm", "nccl_unique_id",
]

POLICIES = {"as_built": 0, "lexicographic": 1, "subtree_tokens_desc": 2, "subtree_tokens_asc": 3}

_P = ctypes.POINTER


def _check(rc: int) -> None:
    if rc == 0:
        return
    msg = _native.lib().tt_last_error().decode()
    if rc == 1:
        raise ValueError(msg)
    if rc == 3:
        raise MemoryError(msg)
    if rc == 4:
        raise FloatingPointError(msg)
    raise RuntimeError(msg)


def _ptr(a: Optional[np.ndarray], t):
    return None if a is None else a.ctypes.data_as(_P(t))


@dataclass(frozen=True)
class ModelConfig:
    vocab_size: int
    d_model: int
    n_heads: int
    n_layers: int
    d_ff: int
    max_position: int
    precision: str = "f32"

    @property
    def head_dim(self) -> int:
        return self.d_model // self.n_heads

    def _c(self) -> _native.ModelConfigC:
        return _native.ModelConfigC(self.vocab_size, self.d_model, self.n_heads, self.n_layers, self.d_ff,
                                    self.max_position, 0 if self.precision == "f32" else 1, 0)

    def param_count(self) -> int:
        n = ctypes.c_uint64()
        _check(_native.lib().tt_param_count(ctypes.byref(self._c()), ctypes.byref(n)))
        return n.value


@dataclass
class TokenSequence:
    seq_id: int
    tokens: Sequence[int]
    weights: Optional[Sequence[float]] = None


def _csr(seqs: Sequence[TokenSequence], with_weights=True):
    lens = [len(s.tokens) for s in seqs]
    off = np.zeros(len(seqs) + 1, dtype=np.uint64)
    off[1:] = np.cumsum(lens)
    tok = np.ascontiguousarray(np.concatenate([np.asarray(s.tokens, dtype=np.int32) for s in seqs])
                               if seqs else np.zeros(0, np.int32), dtype=np.int32)
    w = None
    if with_weights:
        w = np.concatenate([np.asarray(s.weights if s.weights is not None else np.ones(len(s.tokens)), dtype=np.float64)
                            for s in seqs]) if seqs else np.zeros(0)
        w = np.ascontiguousarray(w, dtype=np.float64)
    return tok, off, w


@dataclass
class SchedulerConfig:
    """SPEC.md:204-207 (+ sibling batching, a B200 execution choice)."""

    chunk_len: int = 0
    leaf_kv_skip: bool = False
    child_order_policy: str = "subtree_tokens_desc"
    sibling_batch: bool = True
    batch_token_budget: int = 0

    def _c(self):
        return _native.SchedConfigC(self.chunk_len, int(self.leaf_kv_skip), POLICIES[self.child_order_policy],
                                    int(self.sibling_batch), 0, self.batch_token_budget)


@dataclass
class TrainStepResult:
    total_loss: float
    forward_tokens: int
    recompute_tokens: int
    backward_tokens: int
    peak_live_kv_tokens: int
    peak_live_activation_tokens: int
    num_segments: int
    num_chunks: int
    rollout_tokens: int
    num_batches: int
    num_launches: int
    peak_hbm_bytes: int
    h2d_bytes: int
    d2h_bytes: int

    @classmethod
    def _from(cls, r: _native.StepResultC):
        return cls(*(getattr(r, n) for n, _ in _native.StepResultC._fields_))


class PrefixTree:
    """Compressed prefix tree built by the native library (build_prefix_tree)."""

    def __init__(self, seqs: Sequence[TokenSequence]):
        self._seqs = list(seqs)
        tok, off, w = _csr(self._seqs)
        h = ctypes.c_void_p()
        _check(_native.lib().tt_tree_build(_ptr(tok, ctypes.c_int32), _ptr(off, ctypes.c_uint64),
                                           _ptr(w, ctypes.c_double), len(self._seqs), ctypes.byref(h)))
        self._h = h

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            _native.lib().tt_tree_destroy(h)
            self._h = None

    def order_children(self, policy: str = "subtree_tokens_desc") -> "PrefixTree":
        _check(_native.lib().tt_tree_order_children(self._h, POLICIES[policy]))
        return self

    def stats(self):
        a, b, c_, d = (ctypes.c_uint64() for _ in range(4))
        _check(_native.lib().tt_tree_stats(self._h, ctypes.byref(a), ctypes.byref(b), ctypes.byref(c_), ctypes.byref(d)))
        return dict(tree_tokens=a.value, num_sequences=b.value, num_nodes=c_.value, max_path_tokens=d.value)

    def tree_token_count(self) -> int:
        return self.stats()["tree_tokens"]

    def _text(self, fn) -> str:
        n = ctypes.c_uint64()
        _check(fn(self._h, None, 0, ctypes.byref(n)))
        buf = ctypes.create_string_buffer(n.value + 1)
        _check(fn(self._h, buf, n.value + 1, ctypes.byref(n)))
        return buf.raw[: n.value].decode()

    def serialize(self) -> str:
        return self._text(_native.lib().tt_tree_serialize)

    def dfs_trace(self) -> str:
        return self._text(_native.lib().tt_tree_dfs_trace)

    @property
    def rollout_tokens(self) -> int:
        return sum(len(s.tokens) for s in self._seqs)


def build_prefix_tree(seqs: Sequence[TokenSequence], policy: Optional[str] = "subtree_tokens_desc") -> PrefixTree:
    t = PrefixTree(seqs)
    if policy:
        t.order_children(policy)
    return t


def lexicographic_sort(seqs: Sequence[TokenSequence]) -> List[TokenSequence]:
    tok, off, _ = _csr(seqs, with_weights=False)
    order = np.zeros(len(seqs), dtype=np.uint64)
    _check(_native.lib().tt_lexicographic_sort(_ptr(tok, ctypes.c_int32), _ptr(off, ctypes.c_uint64), len(seqs),
                                               _ptr(order, ctypes.c_uint64)))
    return [seqs[int(i)] for i in order]


def _plan(fn, seqs, K, *extra):
    tok, off, _ = _csr(seqs, with_weights=False)
    grp = np.zeros(len(seqs), dtype=np.int32)
    costs = np.zeros(K, dtype=np.uint64)
    mx, dup = ctypes.c_uint64(), ctypes.c_uint64()
    _check(fn(_ptr(tok, ctypes.c_int32), _ptr(off, ctypes.c_uint64), len(seqs), K, *extra, _ptr(grp, ctypes.c_int32),
              _ptr(costs, ctypes.c_uint64), ctypes.byref(mx), ctypes.byref(dup)))
    groups = [[] for _ in range(K)]
    for i, g in enumerate(grp):
        groups[int(g)].append(seqs[i].seq_id)
    return dict(groups=groups, costs=[int(x) for x in costs], max_cost=mx.value, duplicated_tokens=dup.value)


def partition_contiguous(seqs: Sequence[TokenSequence], K: int):
    """lexicographic order, binary-searched min-max contiguous groups."""
    return _plan(_native.lib().tt_partition_contiguous, seqs, K)


def greedy_least_loaded(seqs: Sequence[TokenSequence], K: int, cost_model: str = "raw_tokens"):
    """SPEC.md:393-401."""
    return _plan(_native.lib().tt_greedy_least_loaded, seqs, K, 1 if cost_model == "raw_tokens" else 0)


# ------------------------------------------------------------------ corpus
@dataclass
class CorpusSpec:
    """[TYPE] CorpusSpec; lengths uniform in [lo, hi]."""

    num_prompts: int = 1
    group_size: int = 1
    prompt_len: Tuple[int, int] = (1, 1)
    response_len: Tuple[int, int] = (1, 1)
    branch_prob: float = 1.0
    vocab_size: int = 2
    seed: int = 0


def _corpus_to_seqs(h) -> List[TokenSequence]:
    L = _native.lib()
    n, nt = ctypes.c_uint64(), ctypes.c_uint64()
    _check(L.tt_corpus_size(h, ctypes.byref(n), ctypes.byref(nt)))
    tok = np.zeros(nt.value, dtype=np.int32)
    off = np.zeros(n.value + 1, dtype=np.uint64)
    w = np.zeros(nt.value, dtype=np.float64)
    _check(L.tt_corpus_export(h, _ptr(tok, ctypes.c_int32), _ptr(off, ctypes.c_uint64), _ptr(w, ctypes.c_double)))
    out = []
    buf = ctypes.create_string_buffer(256)
    need = ctypes.c_uint64()
    for i in range(n.value):
        _check(L.tt_corpus_seq_id(h, i, buf, len(buf), ctypes.byref(need)))
        if need.value > len(buf):
            buf = ctypes.create_string_buffer(int(need.value))
            _check(L.tt_corpus_seq_id(h, i, buf, len(buf), ctypes.byref(need)))
        sid = buf.value.decode()
        a, b = int(off[i]), int(off[i + 1])
        # integer ids stay integers (the dense oracle sums in seq_id order); any other
        # string id maps to its line index and is kept as .name
        ts = TokenSequence(int(sid) if sid.lstrip("-").isdigit() else i, tok[a:b].copy(), w[a:b].copy())
        ts.name = sid
        out.append(ts)
    return out


def _with_corpus(fn):
    h = ctypes.c_void_p()
    _check(fn(ctypes.byref(h)))
    try:
        return _corpus_to_seqs(h)
    finally:
        _native.lib().tt_corpus_destroy(h)


def load_corpus_jsonl(path: str) -> List[TokenSequence]:
    """Corpus JSONL reader: {"seq_id", "tokens", "weights"} per line."""
    return _with_corpus(lambda out: _native.lib().tt_corpus_load_jsonl(str(path).encode(), out))


def gen_corpus(spec: CorpusSpec) -> List[TokenSequence]:
    """[OP] gen-corpus, deterministic per seed."""
    c = _native.CorpusSpecC(spec.num_prompts, spec.group_size, spec.prompt_len[0], spec.prompt_len[1],
                            spec.response_len[0], spec.response_len[1], spec.branch_prob, spec.vocab_size, spec.seed)
    return _with_corpus(lambda out: _native.lib().tt_corpus_generate(ctypes.byref(c), out))


def save_corpus_jsonl(seqs: Sequence[TokenSequence], path: str) -> None:
    """Corpus JSONL writer (exact double round trip of the weights)."""
    tok, off, w = _csr(seqs)
    ids = (ctypes.c_char_p * max(1, len(seqs)))(*[str(getattr(s, "name", s.seq_id)).encode() for s in seqs])
    h = ctypes.c_void_p()
    _check(_native.lib().tt_corpus_from_csr(_ptr(tok, ctypes.c_int32), _ptr(off, ctypes.c_uint64),
                                            _ptr(w, ctypes.c_double), len(seqs), ids, ctypes.byref(h)))
    try:
        _check(_native.lib().tt_corpus_save_jsonl(h, str(path).encode()))
    finally:
        _native.lib().tt_corpus_destroy(h)


class StepPlan:
    """tt_step_plan: a prepared tree step (tt_plan_create / tt_plan_execute)."""

    def __init__(self, eng: "Engine", tree: PrefixTree, sched: SchedulerConfig):
        self._eng = eng
        self._tree = tree
        h = ctypes.c_void_p()
        _check(_native.lib().tt_plan_create(eng._h, tree._h, ctypes.byref(sched._c()), ctypes.byref(h)))
        self._h = h

    def execute(self) -> TrainStepResult:
        r = _native.StepResultC()
        _check(_native.lib().tt_plan_execute(self._eng._h, self._h, ctypes.byref(r)))
        return TrainStepResult._from(r)

    def execute_async(self) -> "StepPlan":
        """Enqueue the step and return at once (tt_plan_execute_async); wait() gives its result. The
        next step's tree may be built and planned meanwhile."""
        _check(_native.lib().tt_plan_execute_async(self._eng._h, self._h))
        return self

    def wait(self) -> TrainStepResult:
        r = _native.StepResultC()
        _check(_native.lib().tt_plan_wait(self._eng._h, self._h, ctypes.byref(r)))
        return TrainStepResult._from(r)

    def trace(self) -> str:
        n = ctypes.c_uint64()
        _check(_native.lib().tt_plan_trace(self._h, None, 0, ctypes.byref(n)))
        buf = ctypes.create_string_buffer(n.value + 1)
        _check(_native.lib().tt_plan_trace(self._h, buf, n.value + 1, ctypes.byref(n)))
        return buf.raw[: n.value].decode()

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            _native.lib().tt_plan_destroy(h)
            self._h = None


def nccl_unique_id() -> bytes:
    """ncclGetUniqueId (rank 0 creates it, every rank passes it to NcclComm)."""
    buf = (ctypes.c_uint8 * 128)()
    _check(_native.lib().tt_nccl_unique_id(buf))
    return bytes(buf)


class NcclComm:
    """One NCCL communicator (ncclCommInitRank) for the engine on `device`."""

    def __init__(self, unique_id: bytes, nranks: int, rank: int, device: int = 0):
        if len(unique_id) != 128:
            raise ValueError("NcclComm: unique id must be 128 bytes")
        buf = (ctypes.c_uint8 * 128)(*unique_id)
        h = ctypes.c_void_p()
        _check(_native.lib().tt_nccl_comm_init_rank(buf, nranks, rank, device, ctypes.byref(h)))
        self.handle = h

    def close(self):
        if getattr(self, "handle", None):
            _native.lib().tt_nccl_comm_destroy(self.handle)
            self.handle = None

    def __del__(self):
        self.close()


class Engine:
    """One B200 engine (weights, GradientStore, KV/dKV stacks, activation arena, one stream)."""

    def __init__(self, cfg: ModelConfig, device: int = 0):
        self.cfg = cfg
        h = ctypes.c_void_p()
        _check(_native.lib().tt_engine_create(ctypes.byref(cfg._c()), device, ctypes.byref(h)))
        self._h = h
        self.n_params = cfg.param_count()
        self._lens: List[int] = []

    def close(self):
        if getattr(self, "_h", None):
            _native.lib().tt_engine_destroy(self._h)
            self._h = None

    def __del__(self):
        self.close()

    @property
    def stream_ptr(self) -> int:
        s = ctypes.c_void_p()
        _check(_native.lib().tt_engine_stream(self._h, ctypes.byref(s)))
        return s.value or 0

    # ---- parameters / gradients
    def upload_params(self, flat: np.ndarray) -> None:
        """Parameters in for_each_tensor order (model.hpp:42-59)."""
        a = np.ascontiguousarray(flat, dtype=np.float32)
        _check(_native.lib().tt_params_upload_f32(self._h, _ptr(a, ctypes.c_float), a.size))

    def init_params_random(self, seed: int) -> None:
        _check(_native.lib().tt_params_init_random(self._h, seed))

    def load_parameters(self, path: str) -> None:
        _check(_native.lib().tt_params_load_ttpm(self._h, path.encode()))

    def zero_gradients(self) -> None:
        _check(_native.lib().tt_grads_zero(self._h))

    def gradients(self, dtype=np.float32) -> np.ndarray:
        """GradientStore in for_each_tensor order (model.hpp:42-59, 76-81); float32 or float64."""
        if np.dtype(dtype) == np.float64:
            out = np.zeros(self.n_params, dtype=np.float64)
            _check(_native.lib().tt_grads_download_f64(self._h, _ptr(out, ctypes.c_double), out.size))
            return out
        out = np.zeros(self.n_params, dtype=np.float32)
        _check(_native.lib().tt_grads_download_f32(self._h, _ptr(out, ctypes.c_float), out.size))
        return out

    def allreduce_gradients(self, comm: "NcclComm") -> None:
        """One in-place NCCL sum all-reduce of the GradientStore."""
        _check(_native.lib().tt_grads_allreduce(self._h, comm.handle))

    def weighted_nll(self, logits: np.ndarray, targets: Sequence[int], weights: Sequence[float],
                     row_off: Optional[Sequence[int]] = None, want_grad: bool = True):
        """weighted_nll (model.hpp:643-677) on the device: returns (loss, grad_logits [n x V] fp32).
        row_off (n + 1 offsets into targets/weights) makes rows multi-target."""
        lg = np.ascontiguousarray(logits, dtype=np.float32)
        if lg.ndim != 2 or lg.shape[1] != self.cfg.vocab_size:
            raise ValueError("weighted_nll: logits must be [n x vocab_size]")
        n = lg.shape[0]
        tg = np.ascontiguousarray(targets, dtype=np.int32)
        w = np.ascontiguousarray(weights, dtype=np.float64)
        ro = None if row_off is None else np.ascontiguousarray(row_off, dtype=np.uint64)
        if ro is None and (tg.size != n or w.size != n):
            raise ValueError("weighted_nll: one target and weight per loss position")
        if ro is not None and (ro.size != n + 1 or int(ro[-1]) > min(tg.size, w.size)):
            raise ValueError("weighted_nll: row_off must have n + 1 entries within targets / weights")
        grad = np.zeros_like(lg) if want_grad else None
        loss = ctypes.c_double()
        _check(_native.lib().tt_weighted_nll(self._h, lg.ctypes.data, n, _ptr(ro, ctypes.c_uint64),
                                             _ptr(tg, ctypes.c_int32), _ptr(w, ctypes.c_double), ctypes.byref(loss),
                                             None if grad is None else grad.ctypes.data))
        return loss.value, grad

    def grads_device_ptr(self) -> int:
        p, n = ctypes.c_void_p(), ctypes.c_uint64()
        _check(_native.lib().tt_grads_device_ptr(self._h, ctypes.byref(p), ctypes.byref(n)))
        return p.value

    @property
    def accum_count(self) -> int:
        n = ctypes.c_uint64()
        _check(_native.lib().tt_grads_accum_count(self._h, ctypes.byref(n)))
        return n.value

    # ---- steps
    def tree_train_step(self, tree: PrefixTree, sched: Optional[SchedulerConfig] = None) -> TrainStepResult:
        sched = sched or SchedulerConfig()
        r = _native.StepResultC()
        _check(_native.lib().tt_tree_train_step(self._h, tree._h, ctypes.byref(sched._c()), ctypes.byref(r)))
        return TrainStepResult._from(r)

    def plan(self, tree: PrefixTree, sched: Optional[SchedulerConfig] = None) -> "StepPlan":
        """Prepare a tree step once (schedule + metadata resident in HBM); execute it many times."""
        return StepPlan(self, tree, sched or SchedulerConfig())

    KCLASSES = ("gemm", "attn_fwd", "attn_bwd", "elementwise", "ce")

    def set_profiling(self, on: bool) -> None:
        _check(_native.lib().tt_engine_set_profiling(self._h, int(on)))

    def set_option(self, key: str, value: int) -> None:
        _check(_native.lib().tt_engine_set_option(self._h, key.encode(), int(value)))

    def profile_gemm_text(self) -> str:
        n = ctypes.c_uint64()
        _check(_native.lib().tt_engine_profile_gemm_text(self._h, None, 0, ctypes.byref(n)))
        buf = ctypes.create_string_buffer(n.value + 1)
        _check(_native.lib().tt_engine_profile_gemm_text(self._h, buf, n.value + 1, ctypes.byref(n)))
        return buf.raw[: n.value].decode()

    def profile(self, reset: bool = True):
        n = len(self.KCLASSES)
        ms, fl, by = (np.zeros(n) for _ in range(3))
        la = np.zeros(n, dtype=np.uint64)
        _check(_native.lib().tt_engine_profile(self._h, _ptr(ms, ctypes.c_double), _ptr(fl, ctypes.c_double),
                                               _ptr(by, ctypes.c_double), _ptr(la, ctypes.c_uint64), int(reset)))
        return {k: dict(ms=float(ms[i]), flops=float(fl[i]), bytes=float(by[i]), launches=int(la[i]))
                for i, k in enumerate(self.KCLASSES)}

    def dense_train_step(self, seqs: Sequence[TokenSequence]) -> TrainStepResult:
        tok, off, w = _csr(seqs)
        r = _native.StepResultC()
        _check(_native.lib().tt_dense_train_step(self._h, _ptr(tok, ctypes.c_int32), _ptr(off, ctypes.c_uint64),
                                                 _ptr(w, ctypes.c_double), len(seqs), ctypes.byref(r)))
        return TrainStepResult._from(r)

    # ---- segment level (device KV stack)
    def forward_segment(self, tokens: Sequence[int], want_logits: bool = True, want_kv: bool = True,
                        want_activations: bool = True) -> Optional[np.ndarray]:
        """PUSH: forward_segment (model.hpp:328-331) continuing from the device stack; returns logits
        [len x V] (fp32) or None. want_kv / want_activations as the reference (tt_segment_push_ex)."""
        tok = np.ascontiguousarray(tokens, dtype=np.int32)
        out = np.zeros((tok.size, self.cfg.vocab_size), dtype=np.float32) if want_logits else None
        _check(_native.lib().tt_segment_push_ex(self._h, _ptr(tok, ctypes.c_int32), tok.size, int(want_kv),
                                                int(want_activations), None if out is None else out.ctypes.data))
        if want_kv or want_activations:
            self._lens.append(tok.size)
        return out

    def segment_loss(self, targets: Sequence[int], weights: Sequence[float],
                     row_off: Optional[Sequence[int]] = None) -> float:
        """VISIT: weighted_nll of the top segment on the device (tt_segment_loss); the pop then takes
        its grad_logits from these pairs."""
        if not self._lens:
            raise ValueError("weighted_nll: empty stack")
        n = self._lens[-1]
        tg = np.ascontiguousarray(targets, dtype=np.int32)
        w = np.ascontiguousarray(weights, dtype=np.float64)
        ro = None if row_off is None else np.ascontiguousarray(row_off, dtype=np.uint64)
        if ro is None and (tg.size != n or w.size != n):
            raise ValueError("weighted_nll: one target and weight per loss position")
        if ro is not None and (ro.size != n + 1 or int(ro[-1]) > min(tg.size, w.size)):
            raise ValueError("weighted_nll: row_off must have len + 1 entries within targets / weights")
        loss = ctypes.c_double()
        _check(_native.lib().tt_segment_loss(self._h, _ptr(ro, ctypes.c_uint64), _ptr(tg, ctypes.c_int32),
                                             _ptr(w, ctypes.c_double), ctypes.byref(loss)))
        return loss.value

    def backward_segment(self, grad_logits: Optional[np.ndarray] = None, want_grad_prefix: bool = True):
        """POP: backward_segment of the top segment; returns grad_prefix as (dK, dV) [L, S, d] or None."""
        if not self._lens:
            raise ValueError("backward_segment: empty stack")
        S_below = sum(self._lens[:-1])
        gl = None
        if grad_logits is not None:
            gl = np.ascontiguousarray(grad_logits, dtype=np.float32)
            if gl.shape != (self._lens[-1], self.cfg.vocab_size):  # model.hpp:488-490
                raise ValueError("backward_segment: grad_logits shape mismatch")
        gp = np.zeros((self.cfg.n_layers, 2, S_below, self.cfg.d_model), dtype=np.float32) if want_grad_prefix else None
        _check(_native.lib().tt_segment_pop(self._h, None if gl is None else gl.ctypes.data,
                                            None if gp is None else gp.ctypes.data))
        self._lens.pop()
        if gp is None:
            return None
        return gp[:, 0], gp[:, 1]

    def stack_depth(self):
        seg, tok = ctypes.c_uint64(), ctypes.c_uint64()
        _check(_native.lib().tt_stack_depth(self._h, ctypes.byref(seg), ctypes.byref(tok)))
        return tok.value, seg.value

    def stack_reset(self):
        _check(_native.lib().tt_stack_reset(self._h))
        self._lens = []
