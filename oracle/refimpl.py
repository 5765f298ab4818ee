"""ORACLE — TEST INFRASTRUCTURE ONLY: ctypes access to oracle/_ref/libttref.so, the reference's own
model core compiled in place from /root/reference by oracle/Makefile (see ref_driver.cpp).

Used to pin the numpy restatement (treetrain_oracle.py), to produce the golden fixtures in
tests/golden/, and as the CPU baseline (bench.py cpu_baseline / --impl reference).
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

from . import treetrain_oracle as O

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(HERE, "_ref", "libttref.so")
REF_ROOT = os.environ.get("TT_REFERENCE_ROOT", "/root/reference/proj/core")

_lib = None


class Cfg(ctypes.Structure):
    _fields_ = [(n, ctypes.c_uint64) for n in ("vocab_size", "d_model", "n_heads", "n_layers", "d_ff", "max_position")]


def build(force: bool = False) -> bool:
    """Compile _ref/libttref.so when the reference tree is present (this container only)."""
    if os.path.exists(LIB) and not force:
        return True
    if not os.path.isdir(REF_ROOT):
        return False
    subprocess.run(["make", "-C", HERE, f"REF={REF_ROOT}"], check=True, capture_output=True)
    return True


def available() -> bool:
    return os.path.exists(LIB)


def lib():
    global _lib
    if _lib is None:
        if not available():
            raise RuntimeError(f"{LIB} not built (oracle/Makefile needs /root/reference)")
        L = ctypes.CDLL(LIB)
        L.ttref_last_error.restype = ctypes.c_char_p
        _lib = L
    return _lib


def _cfg(cfg: O.ModelConfig) -> Cfg:
    return Cfg(cfg.vocab_size, cfg.d_model, cfg.n_heads, cfg.n_layers, cfg.d_ff, cfg.max_position)


def _p(a, t=ctypes.c_double):
    return a.ctypes.data_as(ctypes.POINTER(t)) if a is not None else None


def _check(rc):
    if rc != 0:
        msg = lib().ttref_last_error().decode()
        raise (ValueError if rc == 1 else RuntimeError)(msg)


def init_params(cfg: O.ModelConfig, seed: int) -> np.ndarray:
    out = np.zeros(O.param_count(cfg))
    _check(lib().ttref_init_params(ctypes.byref(_cfg(cfg)), ctypes.c_uint64(seed), _p(out)))
    return out


def save_ttpm(cfg: O.ModelConfig, flat: np.ndarray, path: str, dtype: str = "f32") -> None:
    flat = np.ascontiguousarray(flat, dtype=np.float64)
    _check(lib().ttref_save_ttpm(ctypes.byref(_cfg(cfg)), _p(flat), 0 if dtype == "f32" else 1, path.encode()))


def load_ttpm_f64(path: str):
    c = Cfg()
    _check(lib().ttref_load_ttpm_f64(path.encode(), ctypes.byref(c), None, ctypes.c_uint64(0)))
    cfg = O.ModelConfig(*(int(getattr(c, n)) for n, _ in Cfg._fields_))
    out = np.zeros(O.param_count(cfg))
    _check(lib().ttref_load_ttpm_f64(path.encode(), ctypes.byref(c), _p(out), ctypes.c_uint64(out.size)))
    return cfg, out


def forward_segment(cfg, flat, pk, pv, tokens, S):
    tok = np.ascontiguousarray(tokens, dtype=np.int32)
    n = tok.size
    logits = np.zeros((n, cfg.vocab_size))
    k = np.zeros((cfg.n_layers, n, cfg.d_model))
    v = np.zeros_like(k)
    pk = np.ascontiguousarray(pk, dtype=np.float64)
    pv = np.ascontiguousarray(pv, dtype=np.float64)
    _check(lib().ttref_forward_segment_f64(ctypes.byref(_cfg(cfg)), _p(np.ascontiguousarray(flat)), _p(pk), _p(pv),
                                           ctypes.c_uint64(S), _p(tok, ctypes.c_int32), ctypes.c_uint64(n),
                                           _p(logits), _p(k), _p(v)))
    return logits, k, v


def backward_segment(cfg, flat, pk, pv, tokens, S, grad_logits=None, gnk=None, gnv=None, grads=None):
    tok = np.ascontiguousarray(tokens, dtype=np.int32)
    g = np.zeros(O.param_count(cfg)) if grads is None else grads
    gpk = np.zeros((cfg.n_layers, S, cfg.d_model))
    gpv = np.zeros_like(gpk)
    c = lambda a: None if a is None else np.ascontiguousarray(a, dtype=np.float64)
    _check(lib().ttref_backward_segment_f64(ctypes.byref(_cfg(cfg)), _p(np.ascontiguousarray(flat)), _p(c(pk)),
                                            _p(c(pv)), ctypes.c_uint64(S), _p(tok, ctypes.c_int32),
                                            ctypes.c_uint64(tok.size), _p(c(grad_logits)), _p(c(gnk)), _p(c(gnv)),
                                            _p(g), _p(gpk), _p(gpv)))
    return g, gpk, gpv


def weighted_nll(logits, targets, weights):
    logits = np.ascontiguousarray(logits, dtype=np.float64)
    n, V = logits.shape
    t = np.ascontiguousarray(targets, dtype=np.int32)
    w = np.ascontiguousarray(weights, dtype=np.float64)
    loss = ctypes.c_double()
    grad = np.zeros_like(logits)
    _check(lib().ttref_weighted_nll_f64(_p(logits), ctypes.c_uint64(n), ctypes.c_uint64(V), _p(t, ctypes.c_int32),
                                        _p(w), ctypes.byref(loss), _p(grad)))
    return loss.value, grad


class EventList:
    """PUSH/POP event list of a DFS over an (ordered) oracle tree, with the §3.3 loss pairs."""

    def __init__(self, root: O.TreeNode, seqs):
        by_id = {s.seq_id: s for s in seqs}
        types, tok_off, toks, pair_off, rows, tgts, ws = [], [0], [], [0], [], [], []

        def push(n):
            types.append(0)
            toks.extend(n.tokens)
            tok_off.append(len(toks))
            pair_off.append(len(rows))

        def pop(n, S):
            types.append(1)
            tok_off.append(len(toks))
            r, t, w = O.node_loss_pairs(n, S, by_id)
            rows.extend(r)
            tgts.extend(t)
            ws.extend(w)
            pair_off.append(len(rows))

        def rec(n, S):
            push(n)
            for c in n.children:
                rec(c, S + len(n.tokens))
            pop(n, S)

        for c in root.children:
            rec(c, 0)
        self.types = np.array(types, dtype=np.int32)
        self.tok_off = np.array(tok_off, dtype=np.uint64)
        self.tokens = np.array(toks, dtype=np.int32)
        self.pair_off = np.array(pair_off, dtype=np.uint64)
        self.rows = np.array(rows, dtype=np.int32)
        self.tgts = np.array(tgts, dtype=np.int32)
        self.ws = np.array(ws, dtype=np.float64)

    def args(self):
        return (ctypes.c_uint64(self.types.size), _p(self.types, ctypes.c_int32), _p(self.tok_off, ctypes.c_uint64),
                _p(self.tokens, ctypes.c_int32), _p(self.pair_off, ctypes.c_uint64), _p(self.rows, ctypes.c_int32),
                _p(self.tgts, ctypes.c_int32), _p(self.ws))


def run_events(cfg, flat, events: EventList, precision: str = "f64"):
    """Reference-arithmetic DFS step: (total_loss, grads flat)."""
    g = np.zeros(O.param_count(cfg))
    loss = ctypes.c_double()
    _check(lib().ttref_run_events(0 if precision == "f32" else 1, ctypes.byref(_cfg(cfg)),
                                  _p(np.ascontiguousarray(flat)), *events.args(), ctypes.byref(loss), _p(g)))
    return loss.value, g


def run_events_threads(cfg, flat, events: EventList, n_threads: int):
    """CPU baseline: n_threads concurrent copies of the tree step at T=float. Returns seconds."""
    secs, loss = ctypes.c_double(), ctypes.c_double()
    _check(lib().ttref_run_events_threads(ctypes.byref(_cfg(cfg)), _p(np.ascontiguousarray(flat)), *events.args(),
                                          ctypes.c_int(n_threads), ctypes.byref(secs), ctypes.byref(loss)))
    return secs.value, loss.value


class RefModel:
    """init_params<float> of the reference held in C++ (made once), for repeated timed slices."""

    def __init__(self, cfg: O.ModelConfig, seed: int = 7):
        L = lib()
        L.ttref_model_create.restype = ctypes.c_void_p
        L.ttref_model_create.argtypes = [ctypes.POINTER(Cfg), ctypes.c_uint64]
        L.ttref_model_destroy.argtypes = [ctypes.c_void_p]
        L.ttref_model_slice.argtypes = [ctypes.c_void_p, ctypes.c_uint64, ctypes.c_uint64, ctypes.c_int,
                                        ctypes.c_uint64, ctypes.POINTER(ctypes.c_double)]
        self.cfg = cfg
        self._h = L.ttref_model_create(ctypes.byref(_cfg(cfg)), seed)
        if not self._h:
            raise RuntimeError(L.ttref_last_error().decode())

    def slice(self, S: int, n: int, threads: int, seed: int = 7) -> float:
        """Slowest worker's seconds for forward+NLL+backward of n tokens at prefix S, per thread."""
        secs = ctypes.c_double()
        _check(lib().ttref_model_slice(self._h, S, n, threads, seed, ctypes.byref(secs)))
        return secs.value

    def __del__(self):
        if getattr(self, "_h", None):
            lib().ttref_model_destroy(self._h)
            self._h = None
