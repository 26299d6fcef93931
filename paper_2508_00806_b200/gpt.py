"""GPT training model instrumented for Adacc policies (BASELINE configs[1], [3]).

A decoder-only transformer with EXPLICIT attention, so the attention score /
softmax / dropout-mask activations the reference profiles
(/root/reference/pkg/profiles/example_block.json:7-97) exist as tensors
(fused SDPA would hide them).  Every block reports the
activations autograd saves, as operators with a LayerKind:

  1 block_input  linear        LN1 input (the block checkpoint; never recomputed)
  2 ln1_out      layer_norm    LN1 output, saved by the QKV projection
  3 qkv          qkv_matrix    the fused QKV projection [b, s, 3h] (per-channel over 3h)
  4 attn_softmax softmax       softmax probabilities
  5 attn_mask    dropout_mask  attention-dropout keep mask (bool)
  6 attn_weights score         dropped probabilities, saved by probs @ v
  7 attn_context linear        merged heads, saved by the output projection
  8 ln2_in       linear        residual stream after attention (LN2 input)
  9 ln2_out      layer_norm    LN2 output, saved by the MLP up projection
 10 mlp_up       linear        up-projection output (GELU input)
 11 mlp_gelu     gelu          GELU output, saved by the down projection

Each operator's output is tagged with its recompute recipe, so an
``ActivationPolicy`` can retain, compress or recompute it per the plan.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import torch
import torch.nn as nn
import torch.nn.functional as F

from .hooks import ActivationPolicy, OpInfo
from .profiles import LayerKind

BLOCK_OPS = [
    OpInfo(1, "block_input", LayerKind.LINEAR),
    OpInfo(2, "ln1_out", LayerKind.LAYER_NORM),
    OpInfo(3, "qkv", LayerKind.QKV_MATRIX),
    OpInfo(4, "attn_softmax", LayerKind.SOFTMAX),
    OpInfo(5, "attn_mask", LayerKind.DROPOUT_MASK),
    OpInfo(6, "attn_weights", LayerKind.SCORE),
    OpInfo(7, "attn_context", LayerKind.LINEAR),
    OpInfo(8, "ln2_in", LayerKind.LINEAR),
    OpInfo(9, "ln2_out", LayerKind.LAYER_NORM),
    OpInfo(10, "mlp_up", LayerKind.LINEAR),
    OpInfo(11, "mlp_gelu", LayerKind.GELU),
]


@dataclass
class GPTConfig:
    vocab: int = 50304
    n_layer: int = 24
    n_head: int = 16
    d_model: int = 1024
    seq: int = 1024
    attn_dropout: float = 0.1

    @classmethod
    def named(cls, name: str) -> "GPTConfig":
        return {
            "gpt-tiny": cls(vocab=512, n_layer=2, n_head=4, d_model=128, seq=128),
            "gpt-small-test": cls(vocab=512, n_layer=4, n_head=4, d_model=256, seq=256),
            "gpt-117m": cls(n_layer=12, n_head=12, d_model=768),
            "gpt-345m": cls(n_layer=24, n_head=16, d_model=1024),
            "gpt-1.3b": cls(n_layer=24, n_head=16, d_model=2048),
        }[name]


class _DropMask(torch.autograd.Function):
    """p * mask / keep that saves only the boolean mask (operator 5)."""

    @staticmethod
    def forward(ctx, p, mask, keep):
        ctx.keep = keep
        ctx.save_for_backward(mask)
        return p * mask / keep

    @staticmethod
    def backward(ctx, g):
        (mask,) = ctx.saved_tensors
        return g * mask / ctx.keep, None, None


class _Softmax(torch.autograd.Function):
    """softmax that tags its output (operator 4) BEFORE saving it, so the saved
    probabilities carry their recompute recipe (the stock softmax saves its
    output before the caller could tag it)."""

    @staticmethod
    def forward(ctx, scores, tag):
        p = torch.softmax(scores, dim=-1)
        if tag is not None:
            tag(p)
        ctx.save_for_backward(p)
        return p

    @staticmethod
    def backward(ctx, g):
        (p,) = ctx.saved_tensors
        return p * (g - (g * p).sum(dim=-1, keepdim=True)), None


def head_parts(qkv, n_head):
    """[b, s, 3h] -> q, k, v as strided [b, nh, s, hd] views (no copies)."""
    b, s, three_h = qkv.shape
    h = three_h // 3
    parts = qkv.view(b, s, 3, n_head, h // n_head).permute(2, 0, 3, 1, 4)
    return parts[0], parts[1], parts[2]


def _causal(s, device):
    return torch.ones(s, s, dtype=torch.bool, device=device).triu_(1)


def _qkv_grad(qkv, n_head, dq=None, dk=None, dv=None):
    """[b, s, 3h] gradient with the q / k / v slots given in head layout."""
    g = torch.zeros_like(qkv)
    gq, gk, gv = head_parts(g, n_head)
    for slot, d in ((gq, dq), (gk, dk), (gv, dv)):
        if d is not None:
            slot.copy_(d)
    return g


class _QKScores(torch.autograd.Function):
    """Causal attention scores q k^T * scale from the FUSED qkv activation.

    Saves qkv itself (operator 3, the reference's [tokens, 3h] QKV matrix,
    compressed per channel over its 3h columns), not per-head q / k copies."""

    @staticmethod
    def forward(ctx, qkv, n_head, scale):
        q, k, _ = head_parts(qkv, n_head)
        scores = torch.matmul(q, k.transpose(-2, -1)) * scale
        ctx.save_for_backward(qkv)
        ctx.n_head, ctx.scale = n_head, scale
        return scores.masked_fill(_causal(scores.shape[-1], scores.device), float("-inf"))

    @staticmethod
    def backward(ctx, g):
        (qkv,) = ctx.saved_tensors
        q, k, _ = head_parts(qkv, ctx.n_head)
        g = g.masked_fill(_causal(g.shape[-1], g.device), 0.0) * ctx.scale
        return _qkv_grad(qkv, ctx.n_head, dq=torch.matmul(g, k), dk=torch.matmul(g.transpose(-2, -1), q)), None, None


class _Context(torch.autograd.Function):
    """probs @ v (v from the fused qkv), heads merged to [b, s, h]; saves the
    dropped probabilities (operator 6) and qkv (operator 3)."""

    @staticmethod
    def forward(ctx, pd, qkv, n_head):
        _, _, v = head_parts(qkv, n_head)
        ctx.save_for_backward(pd, qkv)
        ctx.n_head = n_head
        b, nh, s, hd = v.shape
        return torch.matmul(pd, v).transpose(1, 2).reshape(b, s, nh * hd)

    @staticmethod
    def backward(ctx, g):
        pd, qkv = ctx.saved_tensors
        _, _, v = head_parts(qkv, ctx.n_head)
        b, s, h = g.shape
        g = g.view(b, s, ctx.n_head, h // ctx.n_head).transpose(1, 2)
        return torch.matmul(g, v.transpose(-2, -1)), _qkv_grad(qkv, ctx.n_head, dv=torch.matmul(pd.transpose(-2, -1), g)), None


def _causal_softmax(qkv, n_head, scale, tag=None):
    return _Softmax.apply(_QKScores.apply(qkv, n_head, scale), tag)


def _context(pd, qkv, n_head):
    return _Context.apply(pd, qkv, n_head)


class Block(nn.Module):
    def __init__(self, cfg: GPTConfig, layer: int):
        super().__init__()
        d = cfg.d_model
        self.cfg, self.layer = cfg, layer
        self.ln1 = nn.LayerNorm(d)
        self.qkv = nn.Linear(d, 3 * d)
        self.proj = nn.Linear(d, d)
        self.ln2 = nn.LayerNorm(d)
        self.up = nn.Linear(d, 4 * d)
        self.down = nn.Linear(4 * d, d)
        self.scale = 1.0 / math.sqrt(d // cfg.n_head)

    def _mask(self, shape, device, seed):
        g = torch.Generator(device=device)
        g.manual_seed(seed)
        return torch.rand(shape, generator=g, device=device) >= self.cfg.attn_dropout

    def forward(self, x, pol: ActivationPolicy, seed: int):
        nh = self.cfg.n_head
        keep = 1.0 - self.cfg.attn_dropout
        pol.tag(1, x)
        with pol.op(2):
            h = pol.tag(2, self.ln1(x), self.ln1, (x,))
        with pol.op(3):
            qkv = pol.tag(3, self.qkv(h), self.qkv, (h,))  # saved once, as [tokens, 3h]
        with pol.op(4):
            fn4 = lambda a: _causal_softmax(a, nh, self.scale)  # noqa: E731
            p = _causal_softmax(qkv, nh, self.scale, tag=lambda out: pol.tag(4, out, fn4, (qkv,)))
        with pol.op(5):
            mseed = seed * 1000003 + self.layer
            pshape, pdev = tuple(p.shape), p.device
            fn5 = lambda: self._mask(pshape, pdev, mseed)  # noqa: E731  (no tensor captured)
            mask = pol.tag(5, fn5(), fn5, ())
            pd = _DropMask.apply(p, mask, keep) if self.training else p
        with pol.op(6):
            fn6 = lambda a, m: a * m / keep  # noqa: E731
            pol.tag(6, pd, fn6, (p, mask))
            ctx = _context(pd, qkv, nh)
        with pol.op(7):
            fn7 = lambda a, b: _context(a, b, nh)  # noqa: E731
            pol.tag(7, ctx, fn7, (pd, qkv))
            fn8 = lambda r, c: r + self.proj(c)  # noqa: E731
            a = pol.tag(8, fn8(x, ctx), fn8, (x, ctx))
        with pol.op(9):
            h2 = pol.tag(9, self.ln2(a), self.ln2, (a,))
        with pol.op(10):
            u = pol.tag(10, self.up(h2), self.up, (h2,))
        with pol.op(11):
            g = pol.tag(11, F.gelu(u), F.gelu, (u,))
            out = a + self.down(g)
        return out


class GPT(nn.Module):
    def __init__(self, cfg: GPTConfig):
        super().__init__()
        self.cfg = cfg
        self.wte = nn.Embedding(cfg.vocab, cfg.d_model)
        self.wpe = nn.Embedding(cfg.seq, cfg.d_model)
        self.blocks = nn.ModuleList([Block(cfg, i) for i in range(cfg.n_layer)])
        self.ln_f = nn.LayerNorm(cfg.d_model)
        self.head = nn.Linear(cfg.d_model, cfg.vocab, bias=False)
        self.head.weight = self.wte.weight
        self.apply(self._init)
        self.channel_scale = None  # policy-evolution drift: per-channel scale of the residual stream

    @staticmethod
    def _init(m):
        if isinstance(m, nn.Linear):
            nn.init.normal_(m.weight, std=0.02)
            if m.bias is not None:
                nn.init.zeros_(m.bias)
        elif isinstance(m, nn.Embedding):
            nn.init.normal_(m.weight, std=0.02)

    def forward(self, idx, targets, pol: ActivationPolicy, seed: int = 0):
        b, s = idx.shape
        x = self.wte(idx) + self.wpe(torch.arange(s, device=idx.device))
        if self.channel_scale is not None:
            x = x * self.channel_scale
        with pol.hooks():
            for blk in self.blocks:
                x = blk(x, pol, seed)
        logits = self.head(self.ln_f(x))
        return F.cross_entropy(logits.float().reshape(-1, logits.size(-1)), targets.reshape(-1))

    def n_params(self) -> int:
        return sum(p.numel() for p in self.parameters())


def synthetic_batch(step: int, rank: int, batch: int, seq: int, vocab: int, device):
    """Deterministic learnable token stream: a seeded first-order Markov chain
    with a sparse transition table (no dataset download is possible)."""
    g = torch.Generator(device="cpu")
    g.manual_seed(1234)
    # each token has 4 likely successors
    succ = torch.randint(0, vocab, (vocab, 4), generator=g)
    g.manual_seed(10007 * step + 31 * rank + 7)
    toks = torch.empty(batch, seq + 1, dtype=torch.long)
    toks[:, 0] = torch.randint(0, vocab, (batch,), generator=g)
    choice = torch.randint(0, 4, (batch, seq), generator=g)
    noise = torch.rand(batch, seq, generator=g) < 0.1
    rnd = torch.randint(0, vocab, (batch, seq), generator=g)
    for t in range(seq):
        nxt = succ[toks[:, t], choice[:, t]]
        toks[:, t + 1] = torch.where(noise[:, t], rnd[:, t], nxt)
    toks = toks.to(device, non_blocking=True)
    return toks[:, :-1], toks[:, 1:]
