"""Timeline of one mid-grid CTA of the tcgen05 attention dq kernel (TT_ATTN_DBG=3 clock64 trace).
Usage: TT_ATTN_DBG=3 python tools/attn_trace.py [n S H dh]"""
import ctypes
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_00482_b200 import _native  # noqa: E402


def main():
    assert os.environ.get("TT_ATTN_DBG") in ("3", "5")
    subprocess.run([sys.executable, os.path.join(os.path.dirname(__file__), "attn_bench.py"), "1", "1"] + sys.argv[1:],
                   check=True)
    # attn_bench ran in a child process; rerun one bwd here to fill the trace
    import torch

    n, S, H, dh = (int(x) for x in sys.argv[1:5]) if len(sys.argv) > 4 else (8192, 1024, 14, 64)
    lib = _native.lib()
    vp = ctypes.c_void_p
    d = H * dh
    rows = S + n
    t = lambda *s: torch.randn(*s, device="cuda").bfloat16()
    q, K, V, dO = t(n, d), t(rows, d), t(rows, d), t(n, d)
    o = torch.empty(n, d, device="cuda", dtype=torch.bfloat16)
    lse, D = torch.empty(H, n, device="cuda"), torch.empty(H, n, device="cuda")
    dq, dk, dv = torch.empty(n, d, device="cuda"), torch.zeros(rows, d, device="cuda"), torch.zeros(rows, d, device="cuda")
    p = lambda x: vp(x.data_ptr())
    for dirn in (0, 1):
        assert lib.tt_debug_attn(1, dirn, p(q), p(K), p(V), p(o), p(lse), p(dO), p(D), p(dq), p(dk), p(dv), n, S, H, dh,
                                 rows, 0, None) == 0
    torch.cuda.synchronize()
    buf = (ctypes.c_longlong * 1536)()
    assert lib.tt_debug_attn_trace(buf, 1536) == 1536
    tr = [list(buf[i * 256:(i + 1) * 256]) for i in range(6)]
    t0 = tr[2][0]
    print(" j   mma_wake  mma_done  smx_wake  smx_arrive | smx_busy  mma_wait_gap  period | dQ_issue kv_wait S_issue")
    for j in range(1, 120):
        if tr[2][j] == 0:
            break
        print(f"{j:3d} {tr[0][j]-t0:9d} {tr[1][j]-t0:9d} {tr[2][j]-t0:9d} {tr[3][j]-t0:9d} | {tr[3][j]-tr[2][j]:8d} "
              f"{tr[0][j]-tr[3][j]:12d} {tr[3][j]-tr[3][j-1]:7d} | {tr[4][j]-tr[0][j]:8d} {tr[5][j]-tr[4][j]:7d} {tr[1][j]-tr[5][j]:7d}")


if __name__ == "__main__":
    main()
