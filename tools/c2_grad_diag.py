"""Per-tensor gradient error of the engine at the c2 model shape vs the f64 oracle (GPU diagnostic):
prints the 20 worst tensors (rel-Frobenius, cosine) for two engine runs (run-to-run spread of the
fp32 red.add accumulation) and the errors grouped by tensor kind."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
import paper_2602_00482_b200 as tt  # noqa: E402
from oracle import treetrain_oracle as O  # noqa: E402
from test_parity_headline_gpu import C2, lean_params  # noqa: E402


def per_tensor(cfg, got, ref):
    out, o = [], 0
    for name, shape in O.tensor_specs(cfg):
        n = int(np.prod(shape))
        g, r = got[o:o + n].astype(np.float64), ref[o:o + n]
        o += n
        rn = np.linalg.norm(r)
        if rn == 0:
            continue
        out.append((float(np.linalg.norm(g - r) / rn), float(g @ r / (np.linalg.norm(g) * rn + 1e-300)), name))
    return out


if __name__ == "__main__":
    cfg = O.ModelConfig(*C2)
    flat = lean_params(cfg, 2602)
    seqs = O.grouped_corpus(1, 4, 96, 64, cfg.vocab_size, 482, weight_jitter=True)
    root = O.order_children(O.build_prefix_tree(seqs), "subtree_tokens_desc")
    ref = O.tree_train_step(cfg, flat, root, seqs)
    eng = tt.Engine(tt.ModelConfig(*C2))
    eng.upload_params(flat)
    runs = []
    for hc in (6144, 120, 6144):
        eng.set_option("head_chunk_mb", hc)
        eng.zero_gradients()
        r = eng.tree_train_step(tt.build_prefix_tree([tt.TokenSequence(s.seq_id, s.tokens, s.weights) for s in seqs]),
                                tt.SchedulerConfig())
        runs.append(eng.gradients())
        pt = per_tensor(cfg, runs[-1], ref.grads)
        print(f"head_chunk_mb={hc}: loss {r.total_loss:.6f} vs {ref.total_loss:.6f}")
        for e, c, n in sorted(pt, reverse=True)[:12]:
            print(f"   {n:28s} rel {e:.3e} cos {c:.6f}")
        kinds = {}
        for e, c, n in pt:
            kinds.setdefault(n.split(".")[-1], []).append(e)
        print("   by kind (median / max): " + ", ".join(f"{k} {np.median(v):.1e}/{max(v):.1e}" for k, v in kinds.items()))
    print("run-to-run rel (auto chunks twice):", float(np.linalg.norm(runs[0] - runs[2]) / np.linalg.norm(runs[0])))
