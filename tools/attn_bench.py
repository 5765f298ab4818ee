"""Times the segment-attention kernels alone (CUDA events) on a c2-like segment batch: n queries in
nseg sibling segments over a prefix of S stack rows + own causal rows, H heads of dh. Usage:
    python tools/attn_bench.py [nseg] [n S H dh]      (c2 leaf batch: 16 32768 1024 14 64)"""
import ctypes
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_00482_b200 import _native  # noqa: E402


def main():
    nseg = int(sys.argv[1]) if len(sys.argv) > 1 else 1
    n, S, H, dh = (int(x) for x in sys.argv[2:6]) if len(sys.argv) > 5 else (2048, 1024, 14, 64)
    impl_f = impl_b = 1
    if os.environ.get("ATTN_LIB"):  # experiment builds (tools/attn_bwd_ab.sh)
        _native.LIB_PATH = os.path.abspath(os.environ["ATTN_LIB"])
    lib = _native.lib()
    vp = ctypes.c_void_p
    d = H * dh
    rows = S + n
    q = torch.randn(n, d, device="cuda").bfloat16()
    K = torch.randn(rows, d, device="cuda").bfloat16()
    V = torch.randn(rows, d, device="cuda").bfloat16()
    dO = torch.randn(n, d, device="cuda").bfloat16()
    o = torch.empty(n, d, device="cuda", dtype=torch.bfloat16)
    lse = torch.empty(H, n, device="cuda")
    D = torch.empty(H, n, device="cuda")
    dq = torch.empty(n, d, device="cuda")
    dk = torch.zeros(rows, d, device="cuda")
    dv = torch.zeros(rows, d, device="cuda")
    p = lambda t: vp(t.data_ptr())

    ms = ctypes.c_float()

    def fwd(impl, iters=0):
        assert lib.tt_debug_attn(impl, 0, p(q), p(K), p(V), p(o), p(lse), vp(0), vp(0), vp(0), vp(0), vp(0), n, S, H,
                                 dh, rows, iters, ctypes.byref(ms)) == 0, lib.tt_last_error()
        return ms.value

    def bwd(impl, iters=0):
        assert lib.tt_debug_attn(impl, 1, p(q), p(K), p(V), p(o), p(lse), p(dO), p(D), p(dq), p(dk), p(dv), n, S, H,
                                 dh, rows, iters, ctypes.byref(ms)) == 0, lib.tt_last_error()
        return ms.value

    lib.tt_debug_attn_set_segments(nseg)
    seg = (n + nseg - 1) // nseg
    ctx = n * S + sum(m * (m + 1) / 2 for m in [min(seg, n - i) for i in range(0, n, seg)])
    for name, fn, impl, fl in (("fwd", fwd, impl_f, 4.0 * d * ctx), ("bwd", bwd, impl_b, 8.0 * d * ctx)):
        t = fn(impl, iters=10)
        print(f"attn {name} impl={impl} n={n} S={S} H={H} dh={dh}: {t:.3f} ms/launch, "
              f"{fl / (t / 1e3) / 1e12:.1f} TFLOP/s algorithmic", flush=True)


if __name__ == "__main__":
    main()
