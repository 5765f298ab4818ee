"""Pipeline trace of the attention forward (debug library only: make -C paper_2602_00482_b200/csrc
trace) on the c2 leaf-batch shape. Events per key block j (SM clocks, head 0, first CTAs):
  S = S_j issued   PV = PV_j issued   pre = softmax (w2) about to wait for S_j   w = has S_j
  ld = S_j in registers   mx = row max done   ex = exponentials done (before the P store)   ar = p_full arrive
Usage: python tools/attn_ftrace.py [nseg n S H]"""
import ctypes
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CT, NB, NE = 64, 32, 8
EV = ["S", "PV", "w", "ld", "mx", "ex", "ar", "pre"]


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
    o = torch.empty(n, d, device="cuda", dtype=torch.bfloat16)
    lse = torch.empty(H, n, device="cuda")
    vp = ctypes.c_void_p
    p = lambda t: vp(t.data_ptr())
    ms = ctypes.c_float()
    for it in range(3):
        assert lib.tt_debug_attn(1, 0, p(q), p(K), p(V), p(o), p(lse), vp(0), vp(0), vp(0), vp(0), vp(0), n, S, H, dh,
                                 ctypes.c_long(rows), 5 if it == 1 else 0, ctypes.byref(ms)) == 0
    torch.cuda.synchronize()
    buf = np.zeros(CT * NB * NE, dtype=np.int64)
    lib.tt_debug_ftrace_read(buf.ctypes.data_as(ctypes.POINTER(ctypes.c_longlong)), ctypes.c_long(buf.size))
    tr = buf.reshape(CT, NB, NE)
    print(f"forward {ms.value:.3f} ms per launch (nseg {nseg}, n {n}, S {S}, H {H})")
    per, ld, mx, ex, st, wait, loop = [], [], [], [], [], [], []
    for c in range(CT):
        b = tr[c]
        nb = int((b[:, 6] != 0).sum())
        t0 = b[0][0]
        if c < 3:
            for j in range(min(nb, 8)):
                print(f"CTA {c} j={j:2d} " + " ".join(f"{EV[e]}={b[j][e] - t0:7d}" for e in range(NE)))
        for j in range(1, nb):
            per.append(b[j][6] - b[j - 1][6])
            wait.append(b[j][2] - b[j][7])
            loop.append(b[j][7] - b[j - 1][6])
            ld.append(b[j][3] - b[j][2])
            mx.append(b[j][4] - b[j][3])
            ex.append(b[j][5] - b[j][4])
            st.append(b[j][6] - b[j][5])
    cta = np.zeros(CT * 4, dtype=np.int64)
    lib.tt_debug_fcta_read(cta.ctypes.data_as(ctypes.POINTER(ctypes.c_longlong)))
    cta = cta.reshape(CT, 4)
    setup = cta[:, 1] - cta[:, 0]
    first = tr[:, 0, 2] - cta[:, 1]
    body = cta[:, 2] - tr[:, 0, 2]
    tail = cta[:, 3] - cta[:, 2]
    tot = cta[:, 3] - cta[:, 0]
    nbk = (tr[:, :, 6] != 0).sum(1)
    print(f"CTA: total median {np.median(tot):.0f} clk for median {np.median(nbk):.0f} blocks; setup {np.median(setup):.0f}, "
          f"to first S {np.median(first):.0f}, blocks {np.median(body):.0f}, tail {np.median(tail):.0f}")
    for name, v in (("period (ar_j - ar_j-1)", per), ("loop head (ar -> pre-wait)", loop), ("wait for S_j", wait), ("S load", ld), ("max", mx),
                    ("exp + pack", ex), ("P store + arrive", st)):
        print(f"{name:26s} median {np.median(v):7.0f}  p10 {np.percentile(v, 10):7.0f}  p90 {np.percentile(v, 90):7.0f}")


if __name__ == "__main__":
    main()
