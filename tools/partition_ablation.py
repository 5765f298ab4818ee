"""Partition ablation (SPEC.md:393-410 partition-report, "disabling the load-balanced
partitioner": -11.93%), simulated K-worker data parallelism on one B200.

A heterogeneous grouped corpus (gen-corpus) is split into K groups by
partition_contiguous (the paper's min-max contiguous balancing) and by the greedy_least_loaded
baselines (raw-token and tree-token cost). Every group's DFS tree step runs on the GPU in turn
(CUDA events around plan.execute(), second execution timed); a K-GPU step takes as long as its
slowest group, so the simulated throughput is rollout tokens / max group time. The single NCCL
gradient all-reduce is identical across methods and left out.

Usage: python tools/partition_ablation.py [--K 2,4,8] [--prompts 32] [--out gpurun_out/partition_ablation.json]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_2602_00482_b200 as tt  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--K", default="2,4,8")
    ap.add_argument("--prompts", type=int, default=32)
    ap.add_argument("--group", type=int, default=16)
    ap.add_argument("--seed", type=int, default=7)
    ap.add_argument("--out", default="gpurun_out/partition_ablation.json")
    args = ap.parse_args()
    import torch

    spec = tt.CorpusSpec(num_prompts=args.prompts, group_size=args.group, prompt_len=(128, 2048),
                         response_len=(128, 2048), branch_prob=0.02, vocab_size=151936, seed=args.seed)
    seqs = tt.gen_corpus(spec)
    by_id = {s.seq_id: s for s in seqs}
    rollout = sum(len(s.tokens) for s in seqs)
    cfg = tt.ModelConfig(151936, 896, 14, 24, 4864, 4200)  # Qwen2-0.5B shape, reference architecture
    eng = tt.Engine(cfg, device=0)
    eng.init_params_random(7)
    sched = tt.SchedulerConfig(sibling_batch=True)
    ext = torch.cuda.ExternalStream(eng.stream_ptr)

    def group_ms(ids):
        tree = tt.build_prefix_tree([by_id[i] for i in ids])
        plan = eng.plan(tree, sched)
        eng.zero_gradients()
        plan.execute()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record(ext)
        plan.execute()
        e1.record(ext)
        torch.cuda.synchronize()
        return e0.elapsed_time(e1), tree.stats()["tree_tokens"]

    res = {"corpus": dict(spec.__dict__, sequences=len(seqs), rollout_tokens=rollout,
                          tree_tokens=tt.build_prefix_tree(seqs).stats()["tree_tokens"]),
           "model": "qwen2-0.5b-shape (reference architecture), random init, bf16", "runs": []}
    for K in (int(x) for x in args.K.split(",")):
        methods = {"partition_contiguous": tt.partition_contiguous(seqs, K),
                   "greedy_least_loaded(raw_tokens)": tt.greedy_least_loaded(seqs, K, "raw_tokens"),
                   "greedy_least_loaded(tree_tokens)": tt.greedy_least_loaded(seqs, K, "tree_tokens")}
        for name, plan in methods.items():
            times, toks = [], []
            for ids in plan["groups"]:
                if not ids:
                    times.append(0.0)
                    toks.append(0)
                    continue
                ms, tk = group_ms(ids)
                times.append(ms)
                toks.append(tk)
            step = max(times)
            mean_cost = sum(plan["costs"]) / K
            row = {"K": K, "method": name, "max_cost": plan["max_cost"], "duplicated_tokens": plan["duplicated_tokens"],
                   "imbalance": plan["max_cost"] / mean_cost if mean_cost else None, "group_ms": times,
                   "simulated_step_ms": step, "rollout_tokens_per_s": rollout / (step / 1e3)}
            res["runs"].append(row)
            print(json.dumps({k: v for k, v in row.items() if k != "group_ms"}), flush=True)
    os.makedirs(os.path.dirname(args.out) or ".", exist_ok=True)
    json.dump(res, open(args.out, "w"), indent=1)


if __name__ == "__main__":
    main()
