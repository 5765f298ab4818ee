"""c2 step time of a prepared plan executed eagerly (the first execution of every plan, and what the
pipelined e2e loop runs) vs replayed as one CUDA graph (bench.py's timed loop), plus the host cost of
planning. Usage: python tools/eager_vs_graph.py [prompts]"""
import os
import sys
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_2602_00482_b200 as tt  # noqa: E402


def main():
    prompts = int(sys.argv[1]) if len(sys.argv) > 1 else 64
    c = dict(bench.CONFIGS["c2"])
    V, d, H, L, F = bench.MODELS[c["model"]]
    eng = tt.Engine(tt.ModelConfig(V, d, H, L, F, 3088), device=0)
    eng.init_params_random(7)
    seqs = bench.config_corpus(c, prompts, V)
    ext = torch.cuda.ExternalStream(eng.stream_ptr)
    sched = tt.SchedulerConfig()

    def timed(fn):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0 = time.time()
        e0.record(ext)
        fn()
        e1.record(ext)
        torch.cuda.synchronize()
        return e0.elapsed_time(e1), (time.time() - t0) * 1e3

    t0 = time.time()
    plan = eng.plan(tt.build_prefix_tree(seqs), sched)
    print(f"host build + plan: {(time.time() - t0) * 1e3:.1f} ms")
    for k in range(4):
        eng.zero_gradients()
        dev, wall = timed(plan.execute)
        print(f"plan execute #{k} ({'eager' if k == 0 else 'graph'}): device {dev:.1f} ms, wall {wall:.1f} ms")
    for k in range(2):
        p2 = eng.plan(tt.build_prefix_tree(seqs), sched)
        eng.zero_gradients()
        dev, wall = timed(p2.execute)
        print(f"fresh plan eager #{k}: device {dev:.1f} ms, wall {wall:.1f} ms")
        del p2
    eng.set_option("cuda_graph", 0)
    for k in range(2):
        eng.zero_gradients()
        dev, wall = timed(plan.execute)
        print(f"cuda_graph 0 #{k}: device {dev:.1f} ms, wall {wall:.1f} ms")


if __name__ == "__main__":
    main()
