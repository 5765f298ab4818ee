#!/usr/bin/env python
"""bench.py — rollout tokens/s of the DFS prefix-tree forward/backward step on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference] [--config c2]
    python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 ... bench.py --gpus N

A step = one DFS tree fwd+bwd pass (push / visit / pop over every prefix tree of the rank's
shard) + the single NCCL gradient all-reduce (N > 1). Whole prefix trees are sharded across
ranks with the paper's min-max contiguous partitioner (partition_contiguous),
N x the per-GPU workload in total ("weak" scaling). Rank 0 prints ONE JSON line.

  value  : device-timed (CUDA events on the engine stream, barrier + synchronize on both sides,
           max over ranks); the step plan (schedule + metadata) is already resident in HBM.
  e2e    : the same metric through the public API from host sequences every step: tree build,
           plan (host->device metadata copy from pinned memory), execute, loss read-back; step k+1's
           host work overlaps step k's device execution (tt_plan_execute_async / tt_plan_wait).
  roofline: the dominant kernel (tcgen05 GEMM) from one profiled step after the timed region
           (CUDA events around every launch on the engine stream): algorithmic FLOPs / time,
           against MEASURED_PEAKS.json bf16_tflops_sustained (kernel timed inside a long step).
  cpu_baseline: the reference's own model core (oracle/_ref, compiled from /root/reference)
           timed on this box's host cores on a bounded sample; extrapolated through the FLOP model.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "rollout tokens/s (fwd+bwd, DFS tree attn) at 1/2/4/8 B200; peak HBM GB"

# model shapes keep the reference architecture (model.hpp:20-38): MHA, no bias, 2-matrix SiLU MLP,
# untied head, sinusoidal absolute PE, pre-RMSNorm. (V, d, H, L, d_ff)
MODELS = {
    "tiny": (1024, 256, 4, 2, 1024),
    "qwen2-0.5b-shape": (151936, 896, 14, 24, 4864),
    "qwen2.5-1.5b-shape": (151936, 1536, 12, 28, 8960),
    "qwen2.5-7b-shape": (152064, 3584, 28, 28, 18944),
}
CONFIGS = {
    # BASELINE.json configs[0..4]
    "c1": dict(model="tiny", prompts=1, group=8, prompt_len=512, resp_len=256,
               desc="tiny 2-layer d=256 transformer, one prefix tree (512-tok prompt, 8 branches x 256 tok)"),
    "c2": dict(model="qwen2-0.5b-shape", prompts=64, group=16, prompt_len=1024, resp_len=2048,
               desc="Qwen2-0.5B-shape random-init, 64 prompts x 16 rollouts, 1K shared prefix / 2K branches, bf16"),
    "c3": dict(model="qwen2.5-1.5b-shape", prompts=2, deep=(4, 4, 2048), prompt_len=2048, resp_len=6144,
               desc="deep multi-turn agent trees (4 levels, fan-out 4, 2048-token turns: 85 nodes, 64 leaves, "
                    "8K paths), Qwen2.5-1.5B-shape random-init, 2 trees per GPU, DFS stack-memory stress"),
    "c4": dict(model="qwen2.5-7b-shape", prompts=32, group=16, prompt_len=1024, resp_len=2048,
               desc="Qwen2.5-7B-shape random-init, 32 trees per GPU (256 on 8 GPUs), load-balanced, NCCL allreduce"),
    # c5: prefix-share sweep point (--share r): 16 rollouts of 4096 tokens sharing a prefix of r*4096
    "c5": dict(model="qwen2-0.5b-shape", prompts=64, group=16, seq_len=4096,
               desc="prefix-share sweep point: Qwen2-0.5B-shape, 64 prompts x 16 rollouts of 4096 tokens sharing "
                    "a prefix of r*4096 tokens"),
}


def make_deep_corpus(trees, levels, fanout, node_len, vocab, seed):
    """Multi-turn agent trees: a root turn (weights 0) then `levels`-1 levels of `fanout` branches of
    node_len-token turns (weights 1); every root-to-leaf path is one rollout (levels * node_len tokens)."""
    import paper_2602_00482_b200 as tt

    rng = np.random.default_rng(seed)
    seqs = []

    def rec(prefix, w, depth):
        if depth == levels:
            seqs.append(tt.TokenSequence(len(seqs), np.asarray(prefix, dtype=np.int32), np.asarray(w)))
            return
        n = fanout if depth else 1
        firsts = rng.choice(vocab, size=n, replace=False)
        for f0 in firsts:
            turn = rng.integers(0, vocab, node_len).tolist()
            turn[0] = int(f0)
            rec(prefix + turn, w + [0.0 if depth == 0 else 1.0] * node_len, depth + 1)

    for _ in range(trees):
        rec([], [], 0)
    return seqs


def config_corpus(c, n_prompts, vocab, share=0.0):
    """The config's synthetic rollouts for n_prompts prompts (trees)."""
    if "deep" in c:
        lv, fo, nl = c["deep"]
        return make_deep_corpus(n_prompts, lv, fo, nl, vocab, 3)
    if "seq_len" in c:  # c5: shared prefix of share * seq_len tokens
        p = int(round(share * c["seq_len"]))
        return make_corpus(n_prompts, c["group"], p, c["seq_len"] - p, vocab, 3)
    return make_corpus(n_prompts, c["group"], c["prompt_len"], c["resp_len"], vocab, 3)


def make_corpus(prompts, group, prompt_len, resp_len, vocab, seed, shared=0):
    """Rollout groups: a prompt (weights 0) + `group` responses (weights 1) sharing `shared` tokens."""
    import paper_2602_00482_b200 as tt

    rng = np.random.default_rng(seed)
    seqs = []
    for p in range(prompts):
        prompt = rng.integers(0, vocab, prompt_len, dtype=np.int64)
        stem = rng.integers(0, vocab, shared, dtype=np.int64)
        firsts = rng.choice(vocab, size=group, replace=False)
        for g in range(group):
            rest = rng.integers(0, vocab, resp_len - shared, dtype=np.int64)
            rest[0] = firsts[g]
            toks = np.concatenate([prompt, stem, rest]).astype(np.int32)
            w = np.concatenate([np.zeros(prompt_len), np.ones(resp_len)])
            seqs.append(tt.TokenSequence(len(seqs), toks, w))
    return seqs


def step_flops(cfg, tree_nodes):
    """Algorithmic FLOPs of one fwd+bwd step: sum over nodes of
    len*6*(L(4d^2+2d*F) + d*V) + sum over queries 12*d*L*(S+t+1). Recompute not counted."""
    V, d, H, L, F = cfg
    per_tok = 6.0 * (L * (4 * d * d + 2 * d * F) + d * V)
    fl = 0.0
    for S, n in tree_nodes:
        fl += n * per_tok + 12.0 * d * L * (n * S + n * (n + 1) / 2)
    return fl


def tree_nodes_of(seqs):
    """(S, len) of every node of the prefix tree over `seqs` (python mirror, for the FLOP model)."""
    out = []
    groups = {}
    for s in seqs:
        groups.setdefault(tuple(np.asarray(s.tokens[:1]).tolist()), []).append(np.asarray(s.tokens))

    def rec(arrs, S):
        # longest common extension
        m = min(len(a) for a in arrs)
        q = S
        while q < m and all(a[q] == arrs[0][q] for a in arrs[1:]):
            q += 1
        if len(arrs) == 1:
            q = len(arrs[0])
        out.append((S, q - S))
        rest = [a for a in arrs if len(a) > q]
        by = {}
        for a in rest:
            by.setdefault(int(a[q]), []).append(a)
        for g in by.values():
            rec(g, q)

    for g in groups.values():
        rec(g, 0)
    return out


class ClockSampler(threading.Thread):
    """SM clock + clock-event reasons every 100 ms during the timed region (NVML). NVML is opened
    before the thread starts and the first sample is taken at once, so short timed regions (c1 runs
    in ~15 ms) still carry at least one sample; result() adds a closing sample."""

    def __init__(self, dev):
        super().__init__(daemon=True)
        self.dev, self.samples, self.reasons, self.stop_evt = dev, [], set(), threading.Event()
        self.max_mhz, self.nv, self.h = None, None, None
        try:
            import pynvml as nv

            nv.nvmlInit()
            self.nv, self.h = nv, nv.nvmlDeviceGetHandleByIndex(dev)
            self.max_mhz = nv.nvmlDeviceGetMaxClockInfo(self.h, nv.NVML_CLOCK_SM)
            self.names = {getattr(nv, k): k for k in dir(nv)
                          if k.startswith("nvmlClocksEventReason") or k.startswith("nvmlClocksThrottleReason")}
        except Exception as e:  # pragma: no cover - reported, not fatal
            self.reasons.add(f"sampler-error:{type(e).__name__}")

    def sample(self):
        nv, h = self.nv, self.h
        self.samples.append(nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM))
        try:
            r = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
        except Exception:
            r = nv.nvmlDeviceGetCurrentClocksThrottleReasons(h)
        for bit, name in self.names.items():
            if isinstance(bit, int) and bit and bit not in (0xFFFFFFFFFFFFFFFF,) and (r & bit) == bit and bit & (bit - 1) == 0:
                self.reasons.add(name.replace("nvmlClocksEventReason", "").replace("nvmlClocksThrottleReason", ""))

    def run(self):
        if self.nv is None:
            return
        try:
            while not self.stop_evt.is_set():
                self.sample()
                self.stop_evt.wait(0.1)
        except Exception as e:  # pragma: no cover - reported, not fatal
            self.reasons.add(f"sampler-error:{type(e).__name__}")

    def result(self):
        self.stop_evt.set()
        self.join(timeout=2)
        if self.nv is not None and len(self.samples) < 2:
            try:
                self.sample()
            except Exception as e:  # pragma: no cover
                self.reasons.add(f"sampler-error:{type(e).__name__}")
        med = statistics.median(self.samples) if self.samples else None
        return {"sm_mhz": med, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons), "samples": len(self.samples)}


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        j = json.load(open(p))
        return j.get("bf16_tflops_sustained", 1392.8), j.get("bf16_tflops", 1662.4), j.get("hbm_gbs", 6554.6), "measured"
    return 1400.0, 1590.0, 6650.0, "fallback"


# ----------------------------------------------------------------------------- CPU reference arm
def host_cpu():
    """(model string, physical cores, logical CPUs) of this host (BASELINE.md §3 asks for both)."""
    model = "unknown"
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                model = ln.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    try:
        import psutil

        phys = psutil.cpu_count(logical=False)
    except Exception:
        phys = None
    return model, phys, os.cpu_count() or 1


def slice_flops(model, S, n, threads):
    """(GEMM, attention) algorithmic FLOPs of `threads` slices of n tokens at prefix S."""
    V, d, H, L, F = model
    gemm = threads * n * 6.0 * (L * (4 * d * d + 2 * d * F) + d * V)
    attn = threads * 12.0 * d * L * (n * S + n * (n + 1) / 2)
    return gemm, attn


def step_flops_split(model, tree_nodes):
    """step_flops split into its GEMM and attention terms."""
    g = a = 0.0
    for S, n in tree_nodes:
        dg, da = slice_flops(model, S, n, 1)
        g += dg
        a += da
    return g, a


def cpu_reference_fit(model_name, S_lo, S_hi, n_tokens, threads, repeats=1, handle=None):
    """The reference's forward_segment + weighted_nll + backward_segment (T=float, -O3) of n_tokens
    per host thread at two prefix lengths (attention share ~1% and ~25% at c2), one slice per
    thread on all threads; fits separate GEMM and attention seconds-per-FLOP.
    Returns (per-repeat seconds [(t_lo, t_hi)], (sec_per_gemm_flop, sec_per_attn_flop))."""
    from oracle import refimpl as R
    from oracle import treetrain_oracle as O

    model = MODELS[model_name]
    V, d, H, L, F = model
    cfg = O.ModelConfig(V, d, H, L, F, S_hi + n_tokens + 8)
    m = handle or R.RefModel(cfg, 7)
    secs = [(m.slice(S_lo, n_tokens, threads, seed=11 + i), m.slice(S_hi, n_tokens, threads, seed=29 + i))
            for i in range(repeats)]
    return secs, fit_rates(model, S_lo, S_hi, n_tokens, threads, secs[-1])


def fit_rates(model, S_lo, S_hi, n, threads, ts):
    gl, al = slice_flops(model, S_lo, n, threads)
    gh, ah = slice_flops(model, S_hi, n, threads)
    det = gl * ah - gh * al
    a = (ts[0] * ah - ts[1] * al) / det
    b = (gl * ts[1] - gh * ts[0]) / det
    if a <= 0 or b <= 0:  # timing noise swamped the split: one combined rate
        r = (ts[0] + ts[1]) / (gl + al + gh + ah)
        a = b = r
    return a, b


def cpu_extrapolate(model, nodes, roll, rates):
    fg, fa = step_flops_split(model, nodes)
    t = rates[0] * fg + rates[1] * fa
    return roll / t, t


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    c = dict(CONFIGS[args.config])
    if args.prompts:
        c["prompts"] = args.prompts
    model = MODELS[c["model"]]
    from oracle import refimpl as R

    cpu_model, phys, threads = host_cpu()
    if not R.available():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/libttref.so not built (needs /root/reference at build time)"}))
        return 0
    seqs = config_corpus(c, c["prompts"], model[0], args.share)
    nodes = tree_nodes_of(seqs)
    roll = sum(len(s.tokens) for s in seqs)
    seq_len = c.get("seq_len") or c["prompt_len"] + c["resp_len"]
    n_tok = 1 if model[3] > 2 else 64
    S_lo, S_hi = 64, seq_len - n_tok
    secs, _ = cpu_reference_fit(c["model"], S_lo, S_hi, n_tok, threads, repeats=args.warmup + args.steps)
    timed = secs[args.warmup:]
    ts = (float(np.mean([t[0] for t in timed])), float(np.mean([t[1] for t in timed])))
    rates = fit_rates(model, S_lo, S_hi, n_tok, threads, ts)
    value, t_step = cpu_extrapolate(model, nodes, roll, rates)
    sample = (f"reference forward_segment+weighted_nll+backward_segment (T=float) of {n_tok} token(s) per thread at "
              f"prefix S={S_lo} and S={S_hi} on {threads} threads ({ts[0]:.2f} s / {ts[1]:.2f} s per slice pair "
              f"member): fitted {1e-9 / rates[0]:.2f} GEMM-GFLOP/s and {1e-9 / rates[1]:.2f} attention-GFLOP/s, "
              f"extrapolated to the {args.config} step ({t_step / 3600:.1f} h)")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "rollout tokens/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": (ts[0] + ts[1]) * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": f"{args.config}: {c['desc']}", "model": c["model"], "global_batch": len(seqs),
                   "seq_len": seq_len, "parallelism": f"dp{args.gpus}"},
        "cpu_baseline": {"value": value, "unit": "rollout tokens/s", "cores": threads, "kind": "reference",
                         "cpu_model": cpu_model, "physical_cores": phys, "sample": sample},
        "e2e": {"value": value, "unit": "rollout tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))
    return 0


# ----------------------------------------------------------------------------- B200 arm
def product_env():
    """The product path takes no tuning from the environment; any TT_* variable is refused so that a
    number is never taken with a knob set (the line records that the check ran)."""
    bad = sorted(k for k in os.environ if k.startswith("TT_"))
    if bad:
        raise SystemExit(f"bench.py: refusing to run with {bad} set (unset every TT_* variable)")
    return {"TT_*": "none set"}


def run_b200(args):
    env = product_env()
    import torch

    import paper_2602_00482_b200 as tt

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    c = dict(CONFIGS[args.config])
    if args.prompts:
        c["prompts"] = args.prompts
    V, d, H, L, F = MODELS[c["model"]]
    seq_len = c.get("seq_len") or c["prompt_len"] + c["resp_len"]
    max_pos = seq_len + 16
    cfg = tt.ModelConfig(V, d, H, L, F, max_pos)
    # whole job: world x per-GPU prompts, sharded by the min-max contiguous partitioner
    all_seqs = config_corpus(c, c["prompts"] * world, V, args.share)
    if world > 1:
        plan = tt.partition_contiguous(all_seqs, world)
        mine = set(plan["groups"][rank])
        seqs = [s for s in all_seqs if s.seq_id in mine]
    else:
        seqs = all_seqs
    eng = tt.Engine(cfg, device=local)
    for kv in args.option:  # engine execution options (A/B runs; recorded in config.engine_options)
        k, v = kv.split("=")
        eng.set_option(k, int(v))
    eng.init_params_random(7)
    sched = tt.SchedulerConfig(sibling_batch=not args.no_sibling_batch, batch_token_budget=args.batch_budget,
                               chunk_len=args.chunk_len)
    t0 = time.time()
    tree = tt.build_prefix_tree(seqs)
    build_s = time.time() - t0
    st = tree.stats()
    t0 = time.time()
    plan = eng.plan(tree, sched)
    plan_s = time.time() - t0
    ext = torch.cuda.ExternalStream(eng.stream_ptr)
    comm = None
    if world > 1:
        # the engine's own NCCL communicator (tt_nccl_comm_init_rank); torch.distributed only ships the
        # 128-byte unique id and provides the barrier / max-over-ranks timing reduction
        uid = torch.zeros(128, dtype=torch.uint8, device="cuda")
        if rank == 0:
            uid.copy_(torch.frombuffer(bytearray(tt.nccl_unique_id()), dtype=torch.uint8))
        dist.broadcast(uid, 0)
        comm = tt.NcclComm(bytes(uid.cpu().numpy().tobytes()), world, rank, local)

    def one_step():
        eng.zero_gradients()
        r = plan.execute()
        if comm is not None:
            eng.allreduce_gradients(comm)  # ONE in-place ncclAllReduce of the GradientStore per step
        return r

    for _ in range(args.warmup):
        one_step()

    def barrier():
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()

    sampler = ClockSampler(local)
    sampler.start()
    barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(ext)
    launches = 0
    res = None
    for _ in range(args.steps):
        res = one_step()
        launches += res.num_launches
    e1.record(ext)
    barrier()
    clocks = sampler.result()
    ms = e0.elapsed_time(e1) / args.steps
    # ---- e2e through the public API from host sequences, pipelined the way a training loop runs it:
    # step k executes asynchronously (tt_plan_execute_async) while the host builds and plans step
    # k+1 (tree build, schedule, metadata H2D on the engine's copy stream); every step's metadata
    # upload and loss read-back are inside the timed region (the first step's host work included)
    e2e_ms = None
    h2d = 0
    if not args.no_e2e:
        barrier()
        f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        f0.record(ext)
        cur = eng.plan(tt.build_prefix_tree(seqs), sched)
        for k in range(args.e2e_steps):
            eng.zero_gradients()
            cur.execute_async()
            nxt = eng.plan(tt.build_prefix_tree(seqs), sched) if k + 1 < args.e2e_steps else None
            r2 = cur.wait()
            h2d = r2.h2d_bytes
            if comm is not None:
                eng.allreduce_gradients(comm)
            cur = nxt
        f1.record(ext)
        barrier()
        e2e_ms = f0.elapsed_time(f1) / args.e2e_steps
    # ---- max over ranks
    t = torch.tensor([ms, e2e_ms or 0.0], device="cuda", dtype=torch.float64)
    if dist is not None:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms, e2e_ms = float(t[0]), float(t[1])
    roll_local = sum(len(s.tokens) for s in seqs)
    roll_total = sum(len(s.tokens) for s in all_seqs)
    value = roll_total / (ms / 1e3)
    # ---- profiled step for the roofline (after the timed region)
    eng.set_profiling(True)
    eng.zero_gradients()
    plan.execute()
    eng.set_profiling(False)
    gemm_top = eng.profile_gemm_text().splitlines()[:24]
    prof = eng.profile()
    sust, burst, hbm, src = measured_peaks()
    gm = prof["gemm"]
    gemm_tflops = gm["flops"] / (gm["ms"] / 1e3) / 1e12 if gm["ms"] else 0.0
    nodes = tree_nodes_of(seqs)
    fl_step = step_flops((V, d, H, L, F), nodes)
    prof_total_ms = sum(v["ms"] for v in prof.values())
    # ncu-measured DRAM traffic of the dominant GEMM launch (the LM-head logits GEMM), committed under
    # profiles/ (the live run cannot be profiled without perturbing the timing)
    traffic, traffic_note = None, None
    tpath = os.path.join(ROOT, "profiles", "r2", "ncu_traffic.json")
    if os.path.exists(tpath) and args.config == "c2":
        tj = json.load(open(tpath))
        kname, kv = next((k, v) for k, v in tj["kernels"].items() if k.startswith("gemm LM-head"))
        traffic = kv["dram_bytes"]
        traffic_note = (f"{kname}: {kv['dram_bytes'] / 1e9:.3f} GB DRAM per launch vs "
                        f"{kv['algorithmic_bytes'] / 1e9:.3f} GB algorithmic (profiles/r2/ncu_traffic.json)")
    line = {
        "metric": METRIC, "value": value, "unit": "rollout tokens/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "bf16",
        "data": "synthetic: uniform random tokens (seed 3), prompt weights 0 / response weights 1; random-init N(0,0.02) weights",
        "config": {"workload": f"{args.config}: {c['desc']}", "model": c["model"], "global_batch": len(all_seqs),
                   "seq_len": seq_len, "parallelism": f"dp{world}",
                   "trees_per_gpu": c["prompts"], "sibling_batch": not args.no_sibling_batch,
                   "l2": "step working set (weights + activations) >> 126 MB L2; no flush needed", "env": env,
                   **({"engine_options": dict(kv.split("=") for kv in args.option)} if args.option else {})},
        "e2e": {"value": roll_total / (e2e_ms / 1e3) if e2e_ms else None, "unit": "rollout tokens/s",
                "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": 8, "ms_per_step": e2e_ms,
                "includes": "per step: host tree build + schedule + metadata H2D (pinned, copy stream) + execute + loss "
                            "D2H; step k+1's host work overlaps step k's device execution (tt_plan_execute_async)"},
        "gpu_launches": launches,
        "roofline": {"bound": "tensor", "achieved": gemm_tflops, "peak": sust, "unit": "TFLOP/s",
                     "frac": gemm_tflops / sust if sust else None, "traffic": traffic, "traffic_note": traffic_note,
                     "kernel": "tcgen05 GEMM (all projection/MLP/LM-head GEMMs of the step)",
                     "peak_source": f"MEASURED_PEAKS.json bf16_tflops_sustained ({src})",
                     "gemm_share_of_step": gm["ms"] / prof_total_ms if prof_total_ms else None},
        "step_model_tflops": fl_step / (ms / 1e3) / 1e12 * world,
        "step_frac_of_peak": fl_step / (ms / 1e3) / 1e12 / sust,
        "kernel_classes": {k: {"ms": v["ms"], "launches": v["launches"],
                               "tflops": (v["flops"] / (v["ms"] / 1e3) / 1e12) if v["ms"] and v["flops"] else None,
                               "gbs": (v["bytes"] / (v["ms"] / 1e3) / 1e9) if v["ms"] and v["bytes"] else None}
                           for k, v in prof.items()},
        "top_launch_shapes": gemm_top,
        "tree": {"tree_tokens": st["tree_tokens"], "rollout_tokens_per_gpu": roll_local, "nodes": st["num_nodes"],
                 "duplication_factor": roll_local / st["tree_tokens"], "max_path_tokens": st["max_path_tokens"],
                 "segment_batches": res.num_batches, "host_tree_build_s": build_s, "host_plan_s": plan_s},
        "peak_hbm_gb": res.peak_hbm_bytes / 1e9,
        "device_used_gb": (torch.cuda.mem_get_info()[1] - torch.cuda.mem_get_info()[0]) / 1e9,
        "clocks": clocks,
    }
    # ---- flat per-sequence baseline on the same engine (packed varlen, no prefix sharing)
    if not args.no_flat and world == 1:
        eng.zero_gradients()
        eng.dense_train_step(seqs)  # warm
        torch.cuda.synchronize()
        g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        g0.record(ext)
        eng.zero_gradients()
        rf = eng.dense_train_step(seqs)
        g1.record(ext)
        torch.cuda.synchronize()
        fms = g0.elapsed_time(g1)
        line["flat"] = {"value": roll_total / (fms / 1e3), "unit": "rollout tokens/s", "ms_per_step": fms,
                        "peak_hbm_gb": rf.peak_hbm_bytes / 1e9, "forward_tokens": rf.forward_tokens,
                        "note": "same engine, every sequence its own root (no prefix sharing), packed varlen batches"}
    # ---- CPU baseline (rank 0, N = 1 only)
    if not args.no_cpu and world == 1 and rank == 0:
        try:
            from oracle import refimpl as R

            if R.available():
                cpu_model, phys, threads = host_cpu()
                n_tok = 1 if L > 2 else 64
                S_lo, S_hi = 64, seq_len - n_tok
                secs, rates = cpu_reference_fit(c["model"], S_lo, S_hi, n_tok, threads)
                cpu_val, t_step = cpu_extrapolate((V, d, H, L, F), nodes, roll_local, rates)
                line["cpu_baseline"] = {
                    "value": cpu_val * world, "unit": "rollout tokens/s", "cores": threads, "kind": "reference",
                    "cpu_model": cpu_model, "physical_cores": phys,
                    "sample": f"reference forward_segment+weighted_nll+backward_segment (T=float) of {n_tok} token(s) "
                              f"per thread at prefix S={S_lo} and S={S_hi} on {threads} threads "
                              f"({secs[0][0]:.1f} s + {secs[0][1]:.1f} s): fitted {1e-9 / rates[0]:.2f} GEMM-GFLOP/s "
                              f"and {1e-9 / rates[1]:.2f} attention-GFLOP/s, extrapolated to the step ({t_step / 3600:.1f} h)"}
            else:
                line["cpu_baseline"] = {"value": None, "unit": "rollout tokens/s", "cores": 0, "kind": "reference",
                                        "sample": "oracle/_ref not built"}
        except Exception as e:  # the baseline is reported, never fatal
            line["cpu_baseline"] = {"value": None, "unit": "rollout tokens/s", "cores": 0, "kind": "reference",
                                    "sample": f"failed: {e}"}
    if rank == 0:
        print(json.dumps(line))
    if comm is not None:
        comm.close()
    if dist is not None:
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", default="c2", choices=sorted(CONFIGS))
    ap.add_argument("--no-flat", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=5)
    ap.add_argument("--no-sibling-batch", action="store_true")
    ap.add_argument("--batch-budget", type=int, default=0)
    ap.add_argument("--prompts", type=int, default=0, help="override the config's prompts per GPU (quick profiling only)")
    ap.add_argument("--share", type=float, default=0.5, help="c5: shared-prefix fraction r of the 4096-token rollouts")
    ap.add_argument("--chunk-len", type=int, default=0, help="chunked backward (SPEC.md:234-251); 0 = off")
    ap.add_argument("--option", action="append", default=[],
                    help="engine option key=value (tt_engine_set_option; A/B runs only), repeatable")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)
    return run_b200(args)


if __name__ == "__main__":
    sys.exit(main())
