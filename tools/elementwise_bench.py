"""Times the HBM-bound elementwise kernels alone at the c2 leaf-batch shape (32768 x 896 rows) with CUDA
events over back-to-back launches (debug entry points; each call synchronises, so the per-call figure
includes ~10 us of launch + sync). Usage: python tools/elementwise_bench.py [n d]"""
import ctypes
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_00482_b200 import _native  # noqa: E402


def main():
    n, d = (int(a) for a in sys.argv[1:3]) if len(sys.argv) > 2 else (32768, 896)
    if os.environ.get("EW_LIB"):  # experiment builds
        _native.LIB_PATH = os.path.abspath(os.environ["EW_LIB"])
    lib = _native.lib()
    vp = ctypes.c_void_p
    gy, x, gres = (torch.randn(n, d, device="cuda") for _ in range(3))
    g = torch.rand(d, device="cuda") + 0.5
    inv = torch.rand(n, device="cuda") + 0.5
    gx = torch.empty(n, d, device="cuda")
    gxb = torch.empty(n, d, device="cuda", dtype=torch.bfloat16)
    gg = torch.zeros(d, device="cuda")
    call = lambda: lib.tt_debug_rmsnorm_bwd(vp(gy.data_ptr()), vp(x.data_ptr()), vp(inv.data_ptr()), vp(g.data_ptr()),
                                            vp(gres.data_ptr()), vp(gx.data_ptr()), vp(gxb.data_ptr()),
                                            vp(gg.data_ptr()), n, d)
    for _ in range(3):
        call()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    it = 50
    e0.record()
    for _ in range(it):
        call()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / it
    algo = n * d * (4 * 3 + 4 + 2)  # gy, x, gres fp32 in; gx fp32 + gxb bf16 out
    print(f"rmsnorm_bwd n={n} d={d}: {ms * 1e3:.1f} us/call, {algo / ms / 1e6:.0f} GB/s algorithmic (18 B/elem)")


if __name__ == "__main__":
    main()
