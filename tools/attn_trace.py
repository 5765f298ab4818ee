"""Pipeline trace of the fused dh=64 attention backward (debug library only: make -C
paper_2602_00482_b200/csrc trace). Runs the c2 leaf-batch shape (16 sibling segments of 2048
queries over a 1024-row prefix, 14 heads x 64) and prints, for head 0's first CTAs, the per-CTA
prologue / epilogue and the per-block timeline in SM clocks:
  S   = S^T_i issued (warp 1)        dP = dP^T_i issued        sw = softmax stats barrier passed
  s0  = softmax has S/dP (w8)        s1 = sub 1 start (w8)     se = p_full arrive (w8)
  se1 = p_full arrive (w12, half 1)  mm = dV/dK/dQ_i issue (warp 2)   dq = dQ_i in TMEM (drain warp)
Usage: python tools/attn_trace.py [nseg n S H]"""
import ctypes
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CT, NB, NE = 96, 33, 10
EV = ["S", "dP", "s0", "s1", "se", "mm", "dq", "se1", "sw", "-"]


def main():
    a = [int(x) for x in sys.argv[1:]]
    nseg, n, S, H = a if len(a) == 4 else (16, 32768, 1024, 14)
    dh = 64
    lib = ctypes.CDLL(os.path.join(ROOT, "paper_2602_00482_b200", "libtreetrain_b200_trace.so"))
    lib.tt_debug_attn_set_segments(nseg)
    d = H * dh
    rows = S + n
    q = torch.randn(n, d, device="cuda").bfloat16()
    K = torch.randn(rows, d, device="cuda").bfloat16()
    V = torch.randn(rows, d, device="cuda").bfloat16()
    dO = torch.randn(n, d, device="cuda").bfloat16()
    o = torch.empty(n, d, device="cuda", dtype=torch.bfloat16)
    lse = torch.empty(H, n, device="cuda")
    D = torch.empty(H, n, device="cuda")
    dq = torch.zeros(n, d, device="cuda")
    dk = torch.zeros(rows, d, device="cuda")
    dv = torch.zeros(rows, d, device="cuda")
    vp = ctypes.c_void_p
    p = lambda t: vp(t.data_ptr())
    ms = ctypes.c_float()
    assert lib.tt_debug_attn(1, 0, p(q), p(K), p(V), p(o), p(lse), vp(0), vp(0), vp(0), vp(0), vp(0), n, S, H, dh,
                             ctypes.c_long(rows), 0, None) == 0
    for it in range(3):
        lib.tt_debug_trace_clear()
        assert lib.tt_debug_attn(1, 1, p(q), p(K), p(V), p(o), p(lse), p(dO), p(D), p(dq), p(dk), p(dv), n, S, H, dh,
                                 ctypes.c_long(rows), 5 if it == 2 else 0, ctypes.byref(ms)) == 0
    lib.tt_debug_trace_clear()
    assert lib.tt_debug_attn(1, 1, p(q), p(K), p(V), p(o), p(lse), p(dO), p(D), p(dq), p(dk), p(dv), n, S, H, dh,
                             ctypes.c_long(rows), 0, None) == 0
    torch.cuda.synchronize()
    buf = np.zeros(CT * NB * NE, dtype=np.int64)
    lib.tt_debug_trace_read(buf.ctypes.data_as(ctypes.POINTER(ctypes.c_longlong)), ctypes.c_long(buf.size))
    tr = buf.reshape(CT, NB, NE)
    print(f"backward {ms.value:.3f} ms per launch (nseg {nseg}, n {n}, S {S}, H {H})")
    periods, soft, waits, mm_lag = [], [], [], []
    for c in range(CT):
        cta = tr[c, NB - 1]
        if cta[0] == 0:
            continue
        nq = int(cta[5])
        t0 = cta[0]
        blocks = tr[c, :min(nq, NB - 1)]
        if c < 6 or c in (64, 65, 80):
            print(f"CTA {c}: sm {cta[4]} nq {nq}: kv_ready +{cta[1] - t0}, first S +{blocks[0][0] - t0}, "
                  f"last se +{blocks[-1][4] - t0}, acc_done +{cta[2] - t0}, end +{cta[3] - t0}")
            for i, b in enumerate(blocks[:6]):
                print("   i=%2d " % i + " ".join(f"{EV[e]}={b[e] - t0:7d}" for e in (0, 1, 8, 2, 3, 4, 7, 5, 6)))
        for i in range(1, len(blocks)):
            periods.append(blocks[i][4] - blocks[i - 1][4])
            soft.append(blocks[i][4] - blocks[i][2])
            waits.append(blocks[i][2] - blocks[i - 1][4])
            mm_lag.append(blocks[i][5] - max(blocks[i][4], blocks[i][7]))
    pr = lambda name, v: print(f"{name:34s} median {np.median(v):7.0f}  p10 {np.percentile(v, 10):7.0f}  "
                               f"p90 {np.percentile(v, 90):7.0f}")
    pr("block period (se_i - se_{i-1})", periods)
    pr("softmax compute (se_i - s0_i)", soft)
    pr("softmax wait for S/dP (s0_i - se_{i-1})", waits)
    pr("MMA issue lag after p_full", mm_lag)
    ctas = [tr[c, NB - 1] for c in range(CT) if tr[c, NB - 1][0]]
    pr("CTA duration", [x[3] - x[0] for x in ctas])
    pr("CTA prologue (start -> first S)", [tr[c, 0][0] - tr[c, NB - 1][0] for c in range(CT) if tr[c, NB - 1][0]])
    pr("CTA epilogue (acc_done -> end)", [x[3] - x[2] for x in ctas])


if __name__ == "__main__":
    main()
