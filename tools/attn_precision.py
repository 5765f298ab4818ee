"""Attention-backward precision diagnostic (GPU): the tcgen05 kernels' dQ/dK/dV error against an fp32
torch reference, next to the error of an fp32 torch emulation that rounds the MMA operands the
kernels round (P and dS to bf16, D from bf16 O). Regimes: unit-scale scores and the near-uniform
softmax of a random-init model (q, k ~ N(0, 0.05^2))."""
import ctypes
import sys

import torch

sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__))))
from paper_2602_00482_b200 import _native  # noqa: E402


def rel(a, b):
    return ((a.float() - b.float()).norm() / b.float().norm()).item()


def run(n, S, H, dh, qk_scale, seed=0):
    torch.manual_seed(seed)
    lib = _native.lib()
    d = H * dh
    rows = S + n
    q = (torch.randn(n, d, device="cuda") * qk_scale).bfloat16()
    K = (torch.randn(rows, d, device="cuda") * qk_scale).bfloat16()
    V = torch.randn(rows, d, device="cuda").bfloat16()
    dO = torch.randn(n, d, device="cuda").bfloat16()
    o = torch.empty(n, d, device="cuda", dtype=torch.bfloat16)
    lse = torch.empty(H, n, device="cuda")
    D = torch.empty(H, n, device="cuda")
    dq = torch.empty(n, d, device="cuda")
    dk = torch.zeros(rows, d, device="cuda")
    dv = torch.zeros(rows, d, device="cuda")
    vp = ctypes.c_void_p
    p = lambda t: vp(t.data_ptr()) if t is not None else vp(0)
    for dirn in (0, 1):
        rc = lib.tt_debug_attn(1, dirn, p(q), p(K), p(V), p(o), p(lse), p(dO), p(D), p(dq), p(dk), p(dv),
                               n, S, H, dh, ctypes.c_long(rows), 0, None)
        assert rc == 0, lib.tt_last_error().decode()
    scale = dh ** -0.5
    qh = q.float().view(n, H, dh).transpose(0, 1)
    kh = K.float().view(rows, H, dh).transpose(0, 1)
    vh = V.float().view(rows, H, dh).transpose(0, 1)
    doh = dO.float().view(n, H, dh).transpose(0, 1)
    s = qh @ kh.transpose(1, 2) * scale
    mask = torch.arange(rows, device="cuda")[None, :] > (S + torch.arange(n, device="cuda"))[:, None]
    s = s.masked_fill(mask[None], float("-inf"))
    P = torch.softmax(s.double(), -1)
    O = P @ vh.double()
    dP = doh.double() @ vh.double().transpose(1, 2)
    Dx = (doh.double() * O).sum(-1, keepdim=True)
    dS = P * (dP - Dx)
    ex = dict(dq=(dS @ kh.double()) * scale, dk=(dS.transpose(1, 2) @ qh.double()) * scale,
              dv=P.transpose(1, 2) @ doh.double())
    # emulation of the kernels' rounding: P, dS bf16 operands; D from the bf16 O the forward stored
    Pf = P.float()
    P16 = Pf.bfloat16().float()
    O16 = o.float().view(n, H, dh).transpose(0, 1)
    D16 = (doh * O16).sum(-1, keepdim=True)
    dPf = doh @ vh.transpose(1, 2)
    dS16 = (Pf * (dPf - D16)).bfloat16().float()
    em = dict(dq=(dS16 @ kh) * scale, dk=(dS16.transpose(1, 2) @ qh) * scale, dv=P16.transpose(1, 2) @ doh)
    dSx = (Pf * (dPf - Dx.float())).bfloat16().float()  # exact D, bf16 dS
    emx = dict(dk=(dSx.transpose(1, 2) @ qh) * scale)
    got = dict(dq=dq.view(n, H, dh).transpose(0, 1), dk=dk.view(rows, H, dh).transpose(0, 1),
               dv=dv.view(rows, H, dh).transpose(0, 1))
    out = {}
    for k in ("dq", "dk", "dv"):
        out[k] = (rel(got[k], ex[k]), rel(em[k], ex[k]))
    out["dk_exactD"] = rel(emx["dk"], ex["dk"])
    out["D_rel"] = rel(D.view(H, n, 1), Dx)
    return out


if __name__ == "__main__":
    for (n, S, H, dh) in [(2048, 1024, 2, 64), (256, 96, 14, 64), (1200, 1024, 2, 128)]:
        for sc in (1.0, 0.3, 0.05):
            r = run(n, S, H, dh, sc)
            print(f"n={n} S={S} H={H} dh={dh} qk_scale={sc}: " +
                  "  ".join(f"{k} kernel {v[0]:.2e} emul {v[1]:.2e}" for k, v in r.items() if isinstance(v, tuple)) +
                  f"  dk(exact D, bf16 dS) {r['dk_exactD']:.2e}  D_rel {r['D_rel']:.2e}", flush=True)
