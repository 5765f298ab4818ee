"""Kernel-level checks of the sm_100a CUDA kernels against plain PyTorch fp32 references.

These call the debug entry points of libtreetrain_b200.so with torch device pointers.
"""
import ctypes

import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu


def _lib():
    from paper_2602_00482_b200 import _native

    return _native.lib()


EPI_STORE_BF16, EPI_STORE_F32, EPI_ADD_F32, EPI_SILU, EPI_DSILU, EPI_RESID_F32, EPI_STORE_F32_STATS = range(7)


@pytest.fixture(params=[1, 0], ids=["2cta", "1cta"], autouse=True)
def gemm_mode(request):
    """Run every kernel test with the CTA-pair (cta_group::2) GEMM and with the single-CTA GEMM."""
    _lib().tt_debug_gemm_set_2cta(request.param)
    yield request.param
    _lib().tt_debug_gemm_set_2cta(1)


def _gemm(a, a_mn, b, b_mn, M, N, K, mode, outs, ldo, split_w=0, act=None, aux=None, splits=1):
    lib = _lib()
    vp = ctypes.c_void_p
    o = [vp(t.data_ptr()) if t is not None else vp(0) for t in (outs + [None, None, None])[:3]]
    rc = lib.tt_debug_gemm(
        vp(a.data_ptr()), ctypes.c_long(a.stride(0)), a_mn,
        vp(b.data_ptr()), ctypes.c_long(b.stride(0)), b_mn,
        M, N, K, mode, o[0], o[1], o[2], ctypes.c_long(ldo), split_w,
        vp(act.data_ptr()) if act is not None else vp(0),
        vp(aux.data_ptr()) if aux is not None else vp(0), splits)
    assert rc == 0, lib.tt_last_error().decode()


def _rel(x, y):
    return ((x.float() - y.float()).norm() / (y.float().norm() + 1e-30)).item()


@pytest.mark.parametrize("M,N,K", [(128, 256, 64), (200, 384, 192), (1, 512, 256), (300, 896, 896), (129, 4864, 896),
                                   (260, 2688, 896), (64, 576, 128)])
def test_gemm_fwd_kmajor_mnmajor(M, N, K):
    torch.manual_seed(0)
    x = torch.randn(M, K, device="cuda").bfloat16()
    w = torch.randn(K, N, device="cuda").bfloat16()
    out = torch.empty(M, N, device="cuda", dtype=torch.float32)
    _gemm(x, 0, w, 1, M, N, K, EPI_STORE_F32, [out], N)
    ref = x.float() @ w.float()
    assert _rel(out, ref) < 1e-5


@pytest.mark.parametrize("M,N,K", [(300, 896, 896), (129, 4864, 896), (77, 448, 512), (1000, 896, 4864), (64, 256, 128),
                                   (4096, 896, 896)])
def test_gemm_residual_epilogue(M, N, K):
    # x_mid = x + attn W_o / x_out = x_mid + act W_out (model.hpp:427-428,447-448): fp32 residual in, fp32 out
    torch.manual_seed(5)
    a = torch.randn(M, K, device="cuda").bfloat16()
    w = torch.randn(K, N, device="cuda").bfloat16()
    res = torch.randn(M, N, device="cuda")
    out = torch.full((M, N), float("nan"), device="cuda")
    _gemm(a, 0, w, 1, M, N, K, EPI_RESID_F32, [out], N, aux=res)
    ref = res + a.float() @ w.float()
    assert torch.isfinite(out).all()
    assert _rel(out, ref) < 1e-5


@pytest.mark.parametrize("M,N,K", [(128, 128, 256), (77, 896, 4864), (513, 256, 896), (100, 2688, 256),
                                   (512, 896, 256), (4096, 896, 2688), (300, 448, 512), (1000, 672, 896)])
def test_gemm_dx_kmajor_kmajor(M, N, K):
    torch.manual_seed(1)
    dy = torch.randn(M, K, device="cuda").bfloat16()        # [tokens x N_w]
    w = torch.randn(N, K, device="cuda").bfloat16()         # [K_w x N_w]
    out = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    _gemm(dy, 0, w, 0, M, N, K, EPI_STORE_BF16, [out], N)
    ref = dy.float() @ w.float().t()
    assert _rel(out, ref) < 1e-2


@pytest.mark.parametrize("T,Kw,Nw,splits", [(64, 128, 128, 1), (1000, 256, 384, 1), (2048, 896, 896, 4), (333, 128, 512, 2),
                                            (700, 896, 2688, 2)])
def test_gemm_dw_mnmajor_mnmajor(T, Kw, Nw, splits):
    torch.manual_seed(2)
    x = torch.randn(T, Kw, device="cuda").bfloat16()
    dy = torch.randn(T, Nw, device="cuda").bfloat16()
    g = torch.randn(Kw, Nw, device="cuda")
    g0 = g.clone()
    _gemm(x, 1, dy, 1, Kw, Nw, T, EPI_ADD_F32, [g], Nw, splits=splits)
    ref = g0 + x.float().t() @ dy.float()
    assert _rel(g, ref) < 1e-5


@pytest.mark.parametrize("T,Kw,Nw,splits", [(2048, 4864, 896, 1), (512, 896, 4864, 1), (700, 256, 896, 2),
                                            (333, 4864, 128, 1), (96, 1000, 48, 1)])
@pytest.mark.parametrize("tmode", [2, 1], ids=["forced", "model"])
def test_gemm_dw_transposed_epilogue(T, Kw, Nw, splits, tmode):
    """dW += X^T dY computed as dW^T = dY^T X with the transposed reduce-add epilogue (EPI_ADD_F32_T)."""
    torch.manual_seed(3)
    x = torch.randn(T, Kw, device="cuda").bfloat16()
    dy = torch.randn(T, Nw, device="cuda").bfloat16()
    g = torch.randn(Kw, Nw + 16, device="cuda")  # padded pitch
    g0 = g.clone()
    _lib().tt_debug_gemm_set_transpose(tmode)
    try:
        _gemm(x, 1, dy, 1, Kw, Nw, T, EPI_ADD_F32, [g], Nw + 16, splits=splits)
    finally:
        _lib().tt_debug_gemm_set_transpose(1)
    ref = g0[:, :Nw] + x.float().t() @ dy.float()
    assert _rel(g[:, :Nw], ref) < 1e-5
    assert torch.equal(g[:, Nw:], g0[:, Nw:])


@pytest.mark.parametrize("M,N,K", [(512, 896, 320), (776, 448, 64)])  # MN-major A: M * 2 bytes % 16 == 0
def test_gemm_amn_bk_224_wide_pair_tiles(M, N, K):
    """A MN-major, B K-major, N a multiple of 224 but not of 256: the 224-wide CTA-pair tiles."""
    torch.manual_seed(4)
    a = torch.randn(K, M, device="cuda").bfloat16()  # A(m, k) at a[k, m]
    b = torch.randn(N, K, device="cuda").bfloat16()
    out = torch.empty(M, N + 32, device="cuda", dtype=torch.float32)
    _gemm(a, 1, b, 0, M, N, K, EPI_STORE_F32, [out], N + 32)
    ref = a.float().t() @ b.float().t()
    assert _rel(out[:, :N], ref) < 1e-5


def test_gemm_split_columns_qkv():
    torch.manual_seed(3)
    M, d = 200, 256
    x = torch.randn(M, d, device="cuda").bfloat16()
    w = torch.randn(d, 3 * d, device="cuda").bfloat16()
    q, k, v = (torch.empty(M, d, device="cuda", dtype=torch.bfloat16) for _ in range(3))
    _gemm(x, 0, w, 1, M, 3 * d, d, EPI_STORE_BF16, [q, k, v], d, split_w=d)
    ref = x.float() @ w.float()
    assert _rel(torch.cat([q, k, v], 1), ref) < 1e-2


def test_gemm_silu_and_dsilu():
    torch.manual_seed(4)
    M, K, N = 150, 256, 1024
    x = torch.randn(M, K, device="cuda").bfloat16()
    w = (0.1 * torch.randn(K, N, device="cuda")).bfloat16()
    h = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    a = torch.empty_like(h)
    _gemm(x, 0, w, 1, M, N, K, EPI_SILU, [h], N, act=a)
    href = x.float() @ w.float()
    assert _rel(h, href) < 1e-2
    assert _rel(a, torch.nn.functional.silu(h.float())) < 1e-2
    g = torch.randn(M, K, device="cuda").bfloat16()
    w2 = torch.randn(N, K, device="cuda").bfloat16()
    gh = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    _gemm(g, 0, w2, 0, M, N, K, EPI_DSILU, [gh], N, aux=h)
    s = torch.sigmoid(h.float())
    ref = (g.float() @ w2.float().t()) * s * (1 + h.float() * (1 - s))
    assert _rel(gh, ref) < 1e-2


@pytest.mark.parametrize("M,N,K", [(150, 1024, 256), (300, 4864, 896), (512, 4864, 896), (513, 1040, 256), (256, 576, 128)])
def test_gemm_dsilu_epilogue_warp_variants(M, N, K):
    """EPI_DSILU on shapes that launch the 16-epilogue-warp kernel (CTA-pair 256 / 128-wide tiles,
    single-CTA 192-wide tiles) and the 8-warp one (single-CTA 256-wide), with M and N edges."""
    torch.manual_seed(40 + M)
    g = torch.randn(M, K, device="cuda").bfloat16()
    w2 = torch.randn(N, K, device="cuda").bfloat16()
    h = (2 * torch.randn(M, N, device="cuda")).bfloat16()
    gh = torch.full((M, N), float("nan"), device="cuda").bfloat16()
    _gemm(g, 0, w2, 0, M, N, K, EPI_DSILU, [gh], N, aux=h)
    s = torch.sigmoid(h.float())
    ref = (g.float() @ w2.float().t()) * s * (1 + h.float() * (1 - s))
    assert torch.isfinite(gh.float()).all()
    assert _rel(gh, ref) < 1e-2


EPI_STORE_BF16_STATS = 8


@pytest.mark.parametrize("M,N", [(256, 151936), (77, 1040), (300, 4864), (130, 1040), (512, 576)])
def test_gemm_bf16_logits_with_group_stats(M, N):
    """EPI_STORE_BF16_STATS (the engine's LM-head logits): bf16(l - m_g) with m_g the row's 32-column
    group max, plus fp32 (m_g, sum exp(l - m_g)); 16- and 8-epilogue-warp launches, M / N edges."""
    torch.manual_seed(7 + M)
    K = 896
    x = torch.randn(M, K, device="cuda").bfloat16()
    w = (0.05 * torch.randn(K, N, device="cuda")).bfloat16()
    out = torch.full((M, N), float("nan"), device="cuda").bfloat16()
    G = (N + 31) // 32
    stats = torch.full((M, G, 2), float("nan"), device="cuda")
    _gemm(x, 0, w, 1, M, N, K, EPI_STORE_BF16_STATS, [out], N, act=stats)
    ref = x.float() @ w.float()
    pad = torch.full((M, G * 32), float("-inf"), device="cuda")
    pad[:, :N] = ref
    grp = pad.view(M, G, 32)
    mx = grp.max(-1).values
    assert torch.allclose(stats[..., 0], mx, rtol=1e-4, atol=1e-4)
    se = torch.exp(grp - mx[..., None]).sum(-1)
    assert torch.allclose(stats[..., 1], se, rtol=1e-3)
    rec = out.float() + stats[..., 0].repeat_interleave(32, dim=1)[:, :N]
    assert _rel(rec, ref) < 1e-2
    assert (out.float() <= 0).all()  # every entry is relative to its group's max


def test_gemm_large_vocab_head():
    torch.manual_seed(5)
    M, K, N = 256, 896, 151936
    x = torch.randn(M, K, device="cuda").bfloat16()
    w = (0.02 * torch.randn(K, N, device="cuda")).bfloat16()
    out = torch.empty(M, N, device="cuda", dtype=torch.float32)
    _gemm(x, 0, w, 1, M, N, K, EPI_STORE_F32, [out], N)
    ref = x.float() @ w.float()
    assert _rel(out, ref) < 1e-5


@pytest.mark.parametrize("M,N", [(256, 151936), (77, 1024), (300, 4864), (130, 1040)])
def test_gemm_logits_with_softmax_stats(M, N):
    """EPI_STORE_F32_STATS: fp32 logits plus (max, sum exp) per row and 32-column group."""
    torch.manual_seed(6)
    K = 896
    x = torch.randn(M, K, device="cuda").bfloat16()
    w = (0.05 * torch.randn(K, N, device="cuda")).bfloat16()
    out = torch.empty(M, N, device="cuda", dtype=torch.float32)
    G = (N + 31) // 32
    stats = torch.full((M, G, 2), float("nan"), device="cuda")
    _gemm(x, 0, w, 1, M, N, K, EPI_STORE_F32_STATS, [out], N, act=stats)
    ref = x.float() @ w.float()
    assert _rel(out, ref) < 1e-5
    pad = torch.full((M, G * 32), float("-inf"), device="cuda")
    pad[:, :N] = out
    grp = pad.view(M, G, 32)
    mx = grp.max(-1).values
    se = torch.exp(grp - mx[..., None]).sum(-1)
    assert torch.allclose(stats[..., 0], mx)
    assert torch.allclose(stats[..., 1], se, rtol=1e-5)
    # combined log-sum-exp equals the row's
    lse = stats[..., 0].max(-1).values
    lse = lse + torch.log((stats[..., 1] * torch.exp(stats[..., 0] - lse[:, None])).sum(-1))
    assert torch.allclose(lse, torch.logsumexp(out, -1), atol=1e-5)


@pytest.mark.parametrize("n,d", [(1, 256), (37, 896), (4099, 896), (32768, 896), (150, 512), (300, 1536), (129, 3584),
                                 (1001, 3584), (33, 2048), (77, 4096), (5, 8192), (2000, 1024)])
@pytest.mark.parametrize("inplace", [False, True], ids=["gres", "inplace"])
def test_rmsnorm_bwd_matches_torch(n, d, inplace):
    torch.manual_seed(7)
    lib = _lib()
    vp = ctypes.c_void_p
    gy = torch.randn(n, d, device="cuda")
    x = torch.randn(n, d, device="cuda")
    g = torch.rand(d, device="cuda") + 0.5
    inv = 1.0 / torch.sqrt((x * x).mean(-1) + 1e-6)
    gres = torch.randn(n, d, device="cuda")
    gx = torch.empty(n, d, device="cuda")
    gxb = torch.empty(n, d, device="cuda", dtype=torch.bfloat16)
    gg = torch.randn(d, device="cuda")
    gg0 = gg.clone()
    if inplace:  # the engine's call: the residual gradient is accumulated in place (gres == gx)
        gx.copy_(gres)
    rc = lib.tt_debug_rmsnorm_bwd(vp(gy.data_ptr()), vp(x.data_ptr()), vp(inv.data_ptr()), vp(g.data_ptr()),
                                  vp((gx if inplace else gres).data_ptr()), vp(gx.data_ptr()), vp(gxb.data_ptr()),
                                  vp(gg.data_ptr()), n, d)
    assert rc == 0, lib.tt_last_error().decode()
    xr = x.clone().requires_grad_(True)
    gr = g.clone().requires_grad_(True)
    y = xr * torch.rsqrt((xr * xr).mean(-1, keepdim=True) + 1e-6) * gr
    y.backward(gy)
    assert _rel(gx, gres + xr.grad) < 1e-5
    assert _rel(gxb, gres + xr.grad) < 1e-2
    assert _rel(gg, gg0 + gr.grad) < 1e-5


@pytest.mark.parametrize("n,d", [(1, 256), (37, 896), (4099, 896), (32768, 896), (300, 1536), (1001, 3584), (77, 4096),
                                 (150, 448)])
def test_rmsnorm_bwd_bf16_gy_matches_torch(n, d):
    # the engine's grad_normed path: gy (a dX GEMM output) in bf16, residual gradient in place (fp32)
    torch.manual_seed(8)
    lib = _lib()
    vp = ctypes.c_void_p
    gy = torch.randn(n, d, device="cuda").bfloat16()
    x = torch.randn(n, d, device="cuda")
    g = torch.rand(d, device="cuda") + 0.5
    inv = 1.0 / torch.sqrt((x * x).mean(-1) + 1e-6)
    gres = torch.randn(n, d, device="cuda")
    gx = gres.clone()
    gxb = torch.empty(n, d, device="cuda", dtype=torch.bfloat16)
    gg = torch.randn(d, device="cuda")
    gg0 = gg.clone()
    rc = lib.tt_debug_rmsnorm_bwd16(vp(gy.data_ptr()), vp(x.data_ptr()), vp(inv.data_ptr()), vp(g.data_ptr()),
                                    vp(gx.data_ptr()), vp(gx.data_ptr()), vp(gxb.data_ptr()), vp(gg.data_ptr()), n, d)
    assert rc == 0, lib.tt_last_error().decode()
    xr = x.clone().requires_grad_(True)
    gr = g.clone().requires_grad_(True)
    y = xr * torch.rsqrt((xr * xr).mean(-1, keepdim=True) + 1e-6) * gr
    y.backward(gy.float())
    assert _rel(gx, gres + xr.grad) < 1e-5
    assert _rel(gxb, gres + xr.grad) < 1e-2
    assert _rel(gg, gg0 + gr.grad) < 1e-5


def test_rmsnorm_bwd_bf16_gy_rejects_unsupported_width():
    lib = _lib()
    t = torch.zeros(8, 8200, device="cuda")
    vp = ctypes.c_void_p
    rc = lib.tt_debug_rmsnorm_bwd16(vp(t.data_ptr()), vp(t.data_ptr()), vp(t.data_ptr()), vp(t.data_ptr()), vp(0),
                                    vp(t.data_ptr()), vp(t.data_ptr()), vp(t.data_ptr()), 8, 8200)
    assert rc != 0


# ----------------------------------------------------------------------------- segment attention
def _attn_ref(q, K, V, S, H, dh):
    """fp32 reference of one segment's attention over stack rows [0,S) + own rows (causal)."""
    n = q.shape[0]
    ctx = S + n
    qh = q.float().view(n, H, dh).transpose(0, 1)
    kh = K[:ctx].float().view(ctx, H, dh).transpose(0, 1)
    vh = V[:ctx].float().view(ctx, H, dh).transpose(0, 1)
    s = qh @ kh.transpose(1, 2) / dh ** 0.5
    mask = torch.arange(ctx, device=q.device)[None, :] > (S + torch.arange(n, device=q.device))[:, None]
    s = s.masked_fill(mask[None], float("-inf"))
    lse = torch.logsumexp(s, -1)
    p = torch.softmax(s, -1)
    o = (p @ vh).transpose(0, 1).reshape(n, H * dh)
    return o, lse


def _attn(impl, dirn, q, K, V, o, lse, dO=None, D=None, dq=None, dk=None, dv=None, S=0, H=1, dh=64):
    lib = _lib()
    vp = ctypes.c_void_p
    p = lambda t: vp(t.data_ptr()) if t is not None else vp(0)
    rc = lib.tt_debug_attn(impl, dirn, p(q), p(K), p(V), p(o), p(lse), p(dO), p(D), p(dq), p(dk), p(dv),
                           q.shape[0], S, H, dh, ctypes.c_long(K.shape[0]), 0, None)
    assert rc == 0, lib.tt_last_error().decode()


@pytest.mark.parametrize("impl", [1])
@pytest.mark.parametrize("n,S,H,dh", [(128, 0, 2, 64), (300, 200, 2, 64), (77, 1000, 4, 64), (513, 129, 2, 128),
                                      (64, 64, 3, 128), (1000, 1024, 1, 64)])
def test_attention_forward(impl, n, S, H, dh):
    torch.manual_seed(n + S)
    d = H * dh
    rows = S + n + 37
    q = torch.randn(n, d, device="cuda").bfloat16()
    K = torch.randn(rows, d, device="cuda").bfloat16()
    V = torch.randn(rows, d, device="cuda").bfloat16()
    o = torch.empty(n, d, device="cuda", dtype=torch.bfloat16)
    lse = torch.empty(H, n, device="cuda", dtype=torch.float32)
    _attn(impl, 0, q, K, V, o, lse, S=S, H=H, dh=dh)
    oref, lref = _attn_ref(q, K, V, S, H, dh)
    assert _rel(o, oref) < 1e-2, _rel(o, oref)
    assert (lse - lref).abs().max().item() < 1e-2


@pytest.mark.parametrize("impl", [1])
@pytest.mark.parametrize("n,S,H,dh", [(300, 200, 2, 64), (513, 129, 2, 128), (100, 0, 2, 64), (1200, 1024, 2, 64),
                                      (64, 300, 1, 128), (40, 100, 2, 64), (33, 0, 2, 128)])
def test_attention_backward(impl, n, S, H, dh):
    torch.manual_seed(7 + n)
    d = H * dh
    rows = S + n + 11
    q = torch.randn(n, d, device="cuda").bfloat16()
    K = torch.randn(rows, d, device="cuda").bfloat16()
    V = torch.randn(rows, d, device="cuda").bfloat16()
    dO = torch.randn(n, d, device="cuda").bfloat16()
    o = torch.empty(n, d, device="cuda", dtype=torch.bfloat16)
    lse = torch.empty(H, n, device="cuda", dtype=torch.float32)
    _attn(1, 0, q, K, V, o, lse, S=S, H=H, dh=dh)
    D = torch.empty(H, n, device="cuda")
    dq = torch.empty(n, d, device="cuda")
    dk = torch.zeros(rows, d, device="cuda")
    dv = torch.zeros(rows, d, device="cuda")
    _attn(impl, 1, q, K, V, o, lse, dO, D, dq, dk, dv, S=S, H=H, dh=dh)
    qf, Kf, Vf = (t.float().requires_grad_() for t in (q, K, V))
    of, _ = _attn_ref(qf, Kf, Vf, S, H, dh)
    of.backward(dO.float())
    assert _rel(dq, qf.grad) < 2e-2
    assert _rel(dk, Kf.grad) < 2e-2
    assert _rel(dv, Vf.grad) < 2e-2
