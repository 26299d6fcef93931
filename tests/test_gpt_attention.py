"""The fused-QKV attention autograd functions (gpt.py) against plain torch
attention on CPU: same forward, same gradients (float64, dropout off)."""

import torch

from paper_2508_00806_b200.gpt import _causal_softmax, _context


def _reference(qkv, n_head, scale):
    b, s, three_h = qkv.shape
    h = three_h // 3
    q, k, v = qkv.view(b, s, 3, n_head, h // n_head).permute(2, 0, 3, 1, 4)
    scores = (q @ k.transpose(-2, -1)) * scale
    causal = torch.ones(s, s, dtype=torch.bool).triu_(1)
    p = torch.softmax(scores.masked_fill(causal, float("-inf")), dim=-1)
    return (p @ v).transpose(1, 2).reshape(b, s, h), p


def test_fused_qkv_attention_matches_torch():
    torch.manual_seed(0)
    b, s, h, nh = 2, 16, 32, 4
    scale = 1.0 / (h // nh) ** 0.5
    qkv = torch.randn(b, s, 3 * h, dtype=torch.float64, requires_grad=True)
    qkv_ref = qkv.detach().clone().requires_grad_(True)
    p = _causal_softmax(qkv, nh, scale)
    out = _context(p, qkv, nh)
    ref, p_ref = _reference(qkv_ref, nh, scale)
    assert torch.allclose(p, p_ref, atol=1e-12)
    assert torch.allclose(out, ref, atol=1e-12)
    w = torch.randn_like(out)
    (out * w).sum().backward()
    (ref * w).sum().backward()
    assert torch.allclose(qkv.grad, qkv_ref.grad, atol=1e-10)


def test_fused_qkv_gradcheck():
    torch.manual_seed(1)
    b, s, h, nh = 1, 5, 8, 2
    qkv = torch.randn(b, s, 3 * h, dtype=torch.float64, requires_grad=True)

    def f(t):
        return _context(_causal_softmax(t, nh, 0.7), t, nh)

    assert torch.autograd.gradcheck(f, (qkv,))
