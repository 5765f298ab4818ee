"""CPU emulation (torch f64) of why the w_q / w_k gradients carry ~5x the relative error of every
other tensor under bf16 activations (tests/test_engine_gpu.py tolerance note).

One attention head over the random-init residual stream of the reference model (sinusoidal PE +
N(0, 0.02) embeddings, RMS-normalised, model.hpp:239-271): dW_q = X^T dQ and dW_k = X^T dK with
dQ = scale dS K, dK = scale dS^T Q, dS = P (dP - D). dS rows sum to zero, so the common component of
the PE-dominated x / q / k cancels in the exact gradient but not in its rounding errors.

Rows printed:
  * the oracle (f64 activations) vs an engine-like pipeline whose activations (x, q, k, v, O, dO)
    are bf16: the dominant error;
  * the same plus bf16 dS (the attention kernels' MMA operand): adds little;
  * error-feedback rounding of dS along each row (carry the rounding residual into the next column)
    restores the zero row sums but does not move the total, so the kernels keep plain rounding.
"""
import torch

torch.manual_seed(0)
d, dh, n = 896, 64, 352
sc = dh ** -0.5
pos = torch.arange(n, dtype=torch.float64)[:, None]
i = torch.arange(0, d, 2, dtype=torch.float64)
pe = torch.zeros(n, d, dtype=torch.float64)
pe[:, 0::2] = torch.sin(pos / 10000 ** (i / d))
pe[:, 1::2] = torch.cos(pos / 10000 ** (i / d))
Wq, Wk, Wv = ((0.02 * torch.randn(d, dh)).bfloat16().double() for _ in range(3))
causal = torch.triu(torch.ones(n, n, dtype=torch.bool), 1)


def bf16(t):
    return t.float().bfloat16().double()


def fb_round(a, chunk):
    """bf16 rounding with the residual carried along the row (reset every `chunk` columns)."""
    a = a.float()
    out = torch.empty_like(a)
    carry = torch.zeros(a.shape[0], dtype=torch.float32)
    for j in range(a.shape[1]):
        if j % chunk == 0:
            carry.zero_()
        t = a[:, j] + carry
        r = t.bfloat16().float()
        carry = t - r
        out[:, j] = r
    return out.double()


def grads(x, dO, act_bf16, round_dS):
    R = bf16 if act_bf16 else (lambda t: t)
    xx = R(x)
    q, k, v, g = R(xx @ Wq), R(xx @ Wk), R(xx @ Wv), R(dO)
    P = torch.softmax((q @ k.T * sc).masked_fill(causal, float("-inf")), -1)
    D = (g * R(P @ v)).sum(-1, keepdim=True)
    dS = round_dS(P * (g @ v.T - D))
    return xx.T @ (dS @ k * sc), xx.T @ (dS.T @ q * sc)


def rel(a, b):
    return ((a - b).norm() / b.norm()).item()


if __name__ == "__main__":
    x = pe + 0.02 * torch.randn(n, d, dtype=torch.float64)
    x = x / x.pow(2).mean(-1, keepdim=True).sqrt()
    dO = 1e-3 * torch.randn(n, dh, dtype=torch.float64)
    ex = grads(x, dO, False, lambda t: t)
    for name, act, rd in [("bf16 dS only (f64 activations)", False, bf16),
                          ("bf16 activations", True, lambda t: t),
                          ("bf16 activations + bf16 dS (the kernels)", True, bf16),
                          ("bf16 activations + error-feedback dS (32-col chains)", True, lambda t: fb_round(t, 32))]:
        gq, gk = grads(x, dO, act, rd)
        print(f"{name:55s} dW_q rel {rel(gq, ex[0]):.2e}  dW_k rel {rel(gk, ex[1]):.2e}")
