"""A/B of programmatic dependent launch (engine option "pdl", kernels/launch.cuh) on one prepared
plan: the same CUDA-graph step replayed with PDL on and off, interleaved so both arms see the same
clocks, plus the loss / gradient difference between the arms. Usage:
    python tools/pdl_ab.py [config] [reps] [prompts] [lib]   (default: c2 3 0 = the config's own count;
                                                              lib: an experiment build of the library)"""
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_2602_00482_b200 as tt  # noqa: E402


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "c2"
    reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
    prompts = int(sys.argv[3]) if len(sys.argv) > 3 else 0
    if len(sys.argv) > 4:
        tt._native.LIB_PATH = os.path.abspath(sys.argv[4])
    c = dict(bench.CONFIGS[name])
    V, d, H, L, F = bench.MODELS[c["model"]]
    prompts = prompts or c["prompts"]
    seqs = bench.config_corpus(c, prompts, V)
    tree = tt.build_prefix_tree(seqs)
    eng = tt.Engine(tt.ModelConfig(V, d, H, L, F, tree.stats()['max_path_tokens'] + 16), device=0)
    eng.init_params_random(7)
    ext = torch.cuda.ExternalStream(eng.stream_ptr)
    plan = eng.plan(tree, tt.SchedulerConfig())

    def step():
        eng.zero_gradients()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(ext)
        res = plan.execute()
        e1.record(ext)
        torch.cuda.synchronize()
        return e0.elapsed_time(e1), res.total_loss

    times = {0: [], 1: []}
    out = {}
    prev_off = None
    for arm in (1, 0):  # capture both graphs and warm up
        eng.set_option("pdl", arm)
        step()
        step()
    for r in range(reps):
        for arm in (1, 0):
            eng.set_option("pdl", arm)
            ms, loss = step()
            times[arm].append(ms)
            if arm == 0 and arm in out:
                prev_off = out[0][1]
            out[arm] = (loss, eng.gradients().copy())
    t1, t0 = np.median(times[1]), np.median(times[0])
    g1, g0 = out[1][1].astype(np.float64), out[0][1].astype(np.float64)
    print(f"{name} ({prompts} prompts): "
          f"pdl on {t1:.2f} ms, off {t0:.2f} ms per step ({(t0 / t1 - 1) * 100:+.2f}% from PDL); "
          f"all on {['%.2f' % x for x in times[1]]} off {['%.2f' % x for x in times[0]]}")
    print(f"loss on {out[1][0]:.9f} off {out[0][0]:.9f}; grad rel diff "
          f"{np.linalg.norm(g1 - g0) / np.linalg.norm(g0):.3e} (run-to-run with PDL off: "
          f"{np.linalg.norm(prev_off.astype(np.float64) - g0) / np.linalg.norm(g0) if prev_off is not None else float('nan'):.3e})")
    eng.close()


if __name__ == "__main__":
    t = time.time()
    main()
    print(f"wall {time.time() - t:.1f} s")
