"""Per-tile pipeline trace of the tcgen05 GEMM (debug library only: make -C paper_2602_00482_b200/csrc
trace). Runs one GEMM shape of tools/gemm_shapes.py and prints, for the first CTAs, per tile in SM clocks:
  MMA warp (leader):  wait = waiting for a free accumulator slot (the epilogue), main = main loop
  epilogue (draining warps): tf = waiting for the accumulator, rel = accumulator in -> slot released,
                      st = accumulator in -> last store issued; summed over the tile's chunks:
                      opw = operand-load waits, stg = staging (math + smem), tmw = TMEM-load waits,
                      sw = staging-slot waits (bulk_wait_read)
Usage: python tools/gemm_trace.py ["fwd mlp_in"]"""
import ctypes
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from tools.gemm_shapes import SHAPES, EPI_STORE_F32, EPI_ADD_F32, EPI_RESID, EPI_STATS  # noqa: E402

CT, NW, NT, NE = 4, 18, 48, 8


def main():
    label = sys.argv[1] if len(sys.argv) > 1 else "fwd mlp_in"
    _, M, N, K, amn, bmn, epi = next(s for s in SHAPES if s[0] == label)
    from paper_2602_00482_b200 import _native

    _native.LIB_PATH = os.path.join(ROOT, "paper_2602_00482_b200", "libtreetrain_b200_trace.so")
    lib = _native.lib()  # argtypes of the debug entry points
    vp = ctypes.c_void_p
    a = torch.randn(K, M, device="cuda").bfloat16() if amn else torch.randn(M, K, device="cuda").bfloat16()
    b = torch.randn(K, N, device="cuda").bfloat16() if bmn else torch.randn(N, K, device="cuda").bfloat16()
    f32 = epi in (EPI_STORE_F32, EPI_ADD_F32, EPI_RESID, EPI_STATS)
    out = torch.zeros(M, N, device="cuda", dtype=torch.float32 if f32 else torch.bfloat16)
    act = torch.zeros(M, N, device="cuda", dtype=torch.bfloat16)
    aux = torch.zeros(M, N, device="cuda", dtype=torch.float32 if epi == EPI_RESID else torch.bfloat16)

    def run():
        rc = lib.tt_debug_gemm_async(vp(a.data_ptr()), a.stride(0), amn, vp(b.data_ptr()), b.stride(0), bmn, M, N, K,
                                     epi, vp(out.data_ptr()), vp(0), vp(0), N, 0, vp(act.data_ptr()),
                                     vp(aux.data_ptr()), 1)
        assert rc == 0, lib.tt_last_error()

    for _ in range(3):
        run()
    torch.cuda.synchronize()
    lib.tt_debug_gemm_trace_clear()
    run()
    torch.cuda.synchronize()
    buf = np.zeros(CT * NW * NT * NE, dtype=np.int64)
    lib.tt_debug_gemm_trace_read(buf.ctypes.data_as(ctypes.POINTER(ctypes.c_longlong)), ctypes.c_long(buf.size))
    tr = buf.reshape(CT, NW, NT, NE)
    print(f"{label}: M={M} N={N} K={K} epi={epi}")
    agg = {k: [] for k in ("wait", "main", "tf", "rel", "st", "opw", "stg", "tmw", "sw", "period")}
    for c in range(CT):
        print(f"-- CTA {c}")
        mma = tr[c, 1]
        for t in range(NT):
            e = tr[c, 2:NW, t]
            e = e[e[:, 1] != 0]  # the draining epilogue warps of this mode
            if len(e) == 0:
                break
            tf = e[:, 1] - e[:, 0]
            rel = e[:, 2] - e[:, 1]
            st = e[:, 3] - e[:, 1]
            line = f"  tile {t:2d}"
            if mma[t, 1]:
                w, mn = mma[t, 1] - mma[t, 0], mma[t, 2] - mma[t, 1]
                per = mma[t, 1] - mma[t - 1, 1] if t else 0
                line += f" | MMA wait {w:6d} main {mn:6d} period {per:6d}"
                if t >= 2:
                    agg["wait"].append(w)
                    agg["main"].append(mn)
                    agg["period"].append(per)
            line += (f" | epi tf {int(tf.mean()):6d} rel {int(rel.mean()):6d} (max {int(rel.max()):6d})"
                     f" st {int(st.mean()):6d} (max {int(st.max()):6d}) opw {int(e[:, 4].mean())} stg {int(e[:, 5].mean())}"
                     f" tmw {int(e[:, 6].mean())} sw {int(e[:, 7].mean())}")
            if t >= 2:
                agg["tf"].append(tf.mean())
                agg["rel"].append(rel.max())
                agg["st"].append(st.max())
                for k, j in (("opw", 4), ("stg", 5), ("tmw", 6), ("sw", 7)):
                    agg[k].append(e[:, j].mean())
            if t < 12:
                print(line)
    print("median over tiles >= 2: " + "  ".join(f"{k} {int(np.median(v)) if v else 0}" for k, v in agg.items()))


if __name__ == "__main__":
    main()
