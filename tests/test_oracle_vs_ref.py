"""Live cross-check of the numpy oracle against the reference compiled from /root/reference
(oracle/_ref/libttref.so). Skipped where the library was not built."""
import numpy as np
import pytest

from oracle import refimpl as R
from oracle import treetrain_oracle as O

pytestmark = pytest.mark.skipif(not R.available(), reason="oracle/_ref/libttref.so not built")

CFG = O.ModelConfig(vocab_size=64, d_model=32, n_heads=4, n_layers=2, d_ff=64, max_position=512)


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_segment_fwd_bwd(seed):
    rng = np.random.default_rng(seed)
    flat = R.init_params(CFG, 100 + seed)
    P = O.unflatten(CFG, flat)
    S, n = int(rng.integers(0, 20)), int(rng.integers(1, 25))
    pk = rng.normal(size=(CFG.n_layers, S, CFG.d_model))
    pv = rng.normal(size=(CFG.n_layers, S, CFG.d_model))
    toks = rng.integers(0, CFG.vocab_size, n)
    lo, (k, v), acts = O.forward_segment(CFG, P, pk, pv, toks, S)
    lr, kr, vr = R.forward_segment(CFG, flat, pk, pv, toks, S)
    np.testing.assert_allclose(lo, lr, rtol=1e-12, atol=1e-14)
    gl = rng.normal(size=lo.shape)
    gnk, gnv = rng.normal(size=k.shape), rng.normal(size=v.shape)
    G = O.zero_like_params(CFG)
    gpk, gpv = O.backward_segment(CFG, P, acts, pk, pv, G, gl, gnk, gnv)
    gr, gpkr, gpvr = R.backward_segment(CFG, flat, pk, pv, toks, S, gl, gnk, gnv)
    assert np.abs(O.flatten(CFG, G) - gr).max() <= 1e-11 * np.abs(gr).max()
    np.testing.assert_allclose(gpk, gpkr, rtol=1e-9, atol=1e-13)
    np.testing.assert_allclose(gpv, gpvr, rtol=1e-9, atol=1e-13)


def test_tree_step_events_f64():
    seqs = O.grouped_corpus(5, 6, 8, 14, CFG.vocab_size, 7, shared_response=3, weight_jitter=True)
    flat = R.init_params(CFG, 7)
    for pol in ("subtree_tokens_desc", "as_built"):
        root = O.order_children(O.build_prefix_tree(seqs), pol)
        r = O.tree_train_step(CFG, flat, root, seqs)
        lref, gref = R.run_events(CFG, flat, R.EventList(root, seqs))
        assert r.total_loss == pytest.approx(lref, rel=1e-12)
        assert O.compare_grads(r.grads, gref)[1] <= 1e-9


def test_ttpm_roundtrip(tmp_path):
    flat = R.init_params(CFG, 3)
    p = str(tmp_path / "m.ttpm")
    R.save_ttpm(CFG, flat, p, "f64")
    cfg2, flat2 = R.load_ttpm_f64(p)
    assert cfg2 == CFG
    np.testing.assert_array_equal(flat, flat2)


def test_reference_init_distribution():
    flat = R.init_params(CFG, 1)
    P = O.unflatten(CFG, flat)
    e = P["embedding"]
    assert abs(e.mean()) < 3 * 0.02 / np.sqrt(e.size)
    assert np.all(P["layers.0.attn_norm_gain"] == 1.0)
    np.testing.assert_array_equal(flat, R.init_params(CFG, 1))  # SPEC.md:59 determinism
