"""Diagnose the tcgen05 attention forward on one small shape with progress prints."""
import ctypes
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_00482_b200 import _native  # noqa: E402

n, S, H, dh, impl = (int(x) for x in sys.argv[1:6])
print("start", n, S, H, dh, impl, flush=True)
lib = _native.lib()
vp = ctypes.c_void_p
d = H * dh
rows = S + n + 37
torch.manual_seed(0)
q = torch.randn(n, d, device="cuda").bfloat16()
K = torch.randn(rows, d, device="cuda").bfloat16()
V = torch.randn(rows, d, device="cuda").bfloat16()
o = torch.zeros(n, d, device="cuda", dtype=torch.bfloat16)
lse = torch.zeros(H, n, device="cuda")
torch.cuda.synchronize()
print("inputs ready", flush=True)
t = time.time()
p = lambda x: vp(x.data_ptr())
rc = lib.tt_debug_attn(impl, 0, p(q), p(K), p(V), p(o), p(lse), vp(0), vp(0), vp(0), vp(0), vp(0), n, S, H, dh, rows, 0, None)
print("rc", rc, lib.tt_last_error(), "secs", time.time() - t, flush=True)
ctx = S + n
qh = q.float().view(n, H, dh).transpose(0, 1)
kh = K[:ctx].float().view(ctx, H, dh).transpose(0, 1)
vh = V[:ctx].float().view(ctx, H, dh).transpose(0, 1)
s = qh @ kh.transpose(1, 2) / dh ** 0.5
mask = torch.arange(ctx, device="cuda")[None, :] > (S + torch.arange(n, device="cuda"))[:, None]
s = s.masked_fill(mask[None], float("-inf"))
ref = (torch.softmax(s, -1) @ vh).transpose(0, 1).reshape(n, d)
err = ((o.float() - ref).norm() / ref.norm()).item()
rowerr = ((o.float() - ref).norm(dim=1) / ref.norm(dim=1)).cpu()
print("rel err", err, "worst rows", torch.topk(rowerr, 5), flush=True)
