"""Microbenchmark of the tcgen05 GEMM on the c2 (Qwen2-0.5B-shape) step shapes, timed alone with
CUDA events (burst roofline: MEASURED_PEAKS.json bf16_tflops). Usage: python tools/gemm_shapes.py"""
import ctypes
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_00482_b200 import _native  # noqa: E402

EPI_STORE_BF16, EPI_STORE_F32, EPI_ADD_F32, EPI_SILU, EPI_DSILU, EPI_RESID, EPI_STATS = range(7)
EPI_BF16_STATS = 8
n, d, F, V = 32768, 896, 4864, 151936
SHAPES = [  # (label, M, N, K, a_mn, b_mn, epi)
    ("fwd qkv", n, 3 * d, d, 0, 1, EPI_STORE_BF16),
    ("fwd o", n, d, d, 0, 1, EPI_RESID),
    ("fwd mlp_in", n, F, d, 0, 1, EPI_SILU),
    ("fwd mlp_in plain", n, F, d, 0, 1, EPI_STORE_BF16),  # same shape, one bf16 output, no SiLU
    ("fwd mlp_out", n, d, F, 0, 1, EPI_RESID),
    ("fwd head", 2048, V, d, 0, 1, EPI_STORE_F32),
    ("fwd head stats", 2304, V, d, 0, 1, EPI_STATS),
    ("fwd head stats c2", 6656, V, d, 0, 1, EPI_STATS),  # the c2 LM-head chunk (6 GB scratch budget)
    ("fwd head bf16 c2", 6656, V, d, 0, 1, EPI_BF16_STATS),  # the same with bf16 logits (the engine's default)
    ("dX mlp_out", n, F, d, 0, 0, EPI_DSILU),
    ("dX mlp_out plain", n, F, d, 0, 0, EPI_STORE_BF16),  # same shape without the SiLU' operand
    ("dX mlp_in", n, d, F, 0, 0, EPI_STORE_F32),
    ("dX o", n, d, d, 0, 0, EPI_STORE_BF16),
    ("dX qkv", n, d, 3 * d, 0, 0, EPI_STORE_F32),
    ("dX head", 2048, d, V, 0, 0, EPI_ADD_F32),
    ("dW mlp_out", F, d, n, 1, 1, EPI_ADD_F32),
    ("dW mlp_in", d, F, n, 1, 1, EPI_ADD_F32),
    ("dW o", d, d, n, 1, 1, EPI_ADD_F32),
    ("dW qkv", d, 3 * d, n, 1, 1, EPI_ADD_F32),
    ("dW head", d, V, 2048, 1, 1, EPI_ADD_F32),
]


class _Sampler:
    """SM clock (MHz) and board power (W) every 20 ms on a background thread (NVML)."""

    def __init__(self):
        import threading

        import pynvml as nv

        nv.nvmlInit()
        self.nv, self.h = nv, nv.nvmlDeviceGetHandleByIndex(torch.cuda.current_device())
        self.clk, self.pw, self.done = [], [], False
        self.t = threading.Thread(target=self._run, daemon=True)
        self.t.start()

    def _run(self):
        import time

        while not self.done:
            self.clk.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
            self.pw.append(self.nv.nvmlDeviceGetPowerUsage(self.h) / 1e3)
            time.sleep(0.02)

    def stop(self):
        self.done = True
        self.t.join()
        k = len(self.clk) // 4  # drop the ramp-up quarter
        c, w = sorted(self.clk[k:]) or [0], sorted(self.pw[k:]) or [0]
        self.stats = dict(sm_mhz=c[len(c) // 2], power_w=w[len(w) // 2], samples=len(self.clk))

    def summary(self):
        return f"  sm {self.stats['sm_mhz']} MHz  {self.stats['power_w']:.0f} W"


def main():
    if os.environ.get("GEMM_LIB"):  # experiment builds (tools/gemm_epilogue_ab.sh)
        _native.LIB_PATH = os.path.abspath(os.environ["GEMM_LIB"])
    lib = _native.lib()
    lib.tt_debug_gemm_set_2cta(int(os.environ.get("GEMM_2CTA", "1")))
    only = os.environ.get("GEMM_ONLY")
    peaks = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json"))) \
        if os.path.exists("MEASURED_PEAKS.json") else {"bf16_tflops": 1590.0}
    vp = ctypes.c_void_p
    out = []
    shapes = list(SHAPES)
    lib.tt_debug_gemm_force_bn2(int(os.environ.get("GEMM_BN2", "0")))  # 2-CTA tile width (0 = modelled)
    lib.tt_debug_gemm_force_bn1(int(os.environ.get("GEMM_BN1", "0")))  # single-CTA tile width
    for spec in filter(None, os.environ.get("GEMM_CUSTOM", "").split(";")):  # "M,N,K,a_mn,b_mn,epi;..."
        M_, N_, K_, am_, bm_, ep_ = (int(x) for x in spec.split(","))
        lab = f"custom {M_}x{N_}x{K_} a{am_} b{bm_} e{ep_}"
        shapes.append((lab, M_, N_, K_, am_, bm_, ep_))
        only = (only + "," if only else "") + lab
    if os.environ.get("GEMM_EXTRA"):  # "M,N,K" plain bf16-store GEMM (A K-major, B MN-major)
        M_, N_, K_ = (int(x) for x in os.environ["GEMM_EXTRA"].split(","))
        shapes.append(("extra", M_, N_, K_, 0, 1, EPI_STORE_BF16))
        only = only or "extra"
    for label, M, N, K, amn, bmn, epi in shapes:
        if only and label not in only.split(","):
            continue
        a = torch.randn(K, M, device="cuda").bfloat16() if amn else torch.randn(M, K, device="cuda").bfloat16()
        b = torch.randn(K, N, device="cuda").bfloat16() if bmn else torch.randn(N, K, device="cuda").bfloat16()
        o32 = torch.zeros(M, N, device="cuda")
        o16 = torch.zeros(M, N, device="cuda", dtype=torch.bfloat16)
        act = torch.zeros(M, N, device="cuda", dtype=torch.bfloat16)
        aux = torch.zeros(M, N, device="cuda", dtype=torch.float32 if epi == EPI_RESID else torch.bfloat16)
        outp = o32 if epi in (EPI_STORE_F32, EPI_ADD_F32, EPI_RESID, EPI_STATS) else o16
        lda = a.stride(0)
        ldb = b.stride(0)
        splits = lib.tt_debug_gemm_splits(M, N, K) if epi == EPI_ADD_F32 else 1
        if os.environ.get("GEMM_SPLITS"):  # split-K sweep of the accumulate shapes
            splits = int(os.environ["GEMM_SPLITS"]) if epi == EPI_ADD_F32 else 1

        def run():
            rc = lib.tt_debug_gemm_async(vp(a.data_ptr()), lda, amn, vp(b.data_ptr()), ldb, bmn, M, N, K, epi,
                                   vp(outp.data_ptr()), vp(0), vp(0), N, 0, vp(act.data_ptr()), vp(aux.data_ptr()),
                                   splits)
            assert rc == 0, lib.tt_last_error()

        for _ in range(2):
            run()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        # GEMM_ITERS > 10: a sustained run (seconds) with the SM clock and board power sampled, so a
        # variant's cost under the power cap shows up as clock, not only as time
        it = int(os.environ.get("GEMM_ITERS", "10"))
        smp = _Sampler() if it > 10 else None
        e0.record()
        for _ in range(it):
            run()
        e1.record()
        torch.cuda.synchronize()
        if smp:
            smp.stop()
        ms = e0.elapsed_time(e1) / it
        tf = 2.0 * M * N * K / (ms / 1e3) / 1e12
        out.append(dict(shape=label, M=M, N=N, K=K, ms=ms, tflops=tf, frac=tf / peaks["bf16_tflops"], splits=splits))
        clk = smp.summary() if smp else ""
        if smp:
            out[-1].update(smp.stats)
        print(f"{label:12s} M={M:6d} N={N:6d} K={K:6d} splits={splits} {ms:8.3f} ms {tf:7.1f} TFLOP/s "
              f"({100 * tf / peaks['bf16_tflops']:.0f}% of burst peak){clk}", flush=True)
        del a, b, o32, o16, act, aux
    json.dump(out, open(os.environ.get("GEMM_SHAPES_OUT", "gpurun_out/gemm_shapes.json"), "w"), indent=1)


if __name__ == "__main__":
    main()
