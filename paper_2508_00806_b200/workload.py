"""Synthetic activation sets of the BASELINE.json configurations.

``gpt_block_ops`` lists the nine saved activations of one GPT transformer
block in the operator order of the reference's profile
(/root/reference/pkg/profiles/example_block.json:7-97), each with the layer
kind that ``scheme_for`` maps to a compressor (codec.py:72-82).  Shapes follow
explicit (non-fused) attention so the score / softmax / dropout-mask tensors
exist.

Values are synthetic but shaped like real activations: normal channels with a
few injected outlier channels (Fig. 4a: outliers cluster by channel),
scores ~ N(0, 3), softmax rows that sum to one, dropout masks with keep 0.9.
"""

from __future__ import annotations

from dataclasses import dataclass

import torch

from .profiles import LayerKind


@dataclass(frozen=True)
class OpSpec:
    id: int
    name: str
    kind: LayerKind
    rows: int
    cols: int

    @property
    def numel(self) -> int:
        return self.rows * self.cols


def gpt_block_ops(batch: int = 8, seq: int = 1024, hidden: int = 1024, heads: int = 16,
                  ffn: int | None = None) -> list[OpSpec]:
    ffn = ffn or 4 * hidden
    t = batch * seq
    att = batch * heads * seq
    return [
        OpSpec(1, "block_input", LayerKind.LINEAR, t, hidden),
        OpSpec(2, "qkv_matmul", LayerKind.QKV_MATRIX, t, 3 * hidden),
        OpSpec(3, "attn_score", LayerKind.SCORE, att, seq),
        OpSpec(4, "attn_softmax", LayerKind.SOFTMAX, att, seq),
        OpSpec(5, "attn_dropout_mask", LayerKind.DROPOUT_MASK, att, seq),
        OpSpec(6, "attn_out_proj", LayerKind.LINEAR, t, hidden),
        OpSpec(7, "mlp_up_proj", LayerKind.LINEAR, t, ffn),
        OpSpec(8, "mlp_gelu", LayerKind.GELU, t, ffn),
        OpSpec(9, "mlp_down_proj", LayerKind.LINEAR, t, hidden),
    ]


def llama_layer_ops(batch: int = 1, seq: int = 4096, hidden: int = 4096,
                    ffn: int = 11008) -> list[OpSpec]:
    """configs[2]: a Llama-2-7B-shaped layer's compressible activations (flash attention)."""
    t = batch * seq
    return [
        OpSpec(1, "rmsnorm_in", LayerKind.LAYER_NORM, t, hidden),
        OpSpec(2, "q_proj", LayerKind.QKV_MATRIX, t, hidden),
        OpSpec(3, "k_proj", LayerKind.QKV_MATRIX, t, hidden),
        OpSpec(4, "v_proj", LayerKind.QKV_MATRIX, t, hidden),
        OpSpec(5, "o_proj_in", LayerKind.LINEAR, t, hidden),
        OpSpec(6, "rmsnorm_post", LayerKind.LAYER_NORM, t, hidden),
        OpSpec(7, "gate_proj", LayerKind.LINEAR, t, ffn),
        OpSpec(8, "up_proj", LayerKind.LINEAR, t, ffn),
        OpSpec(9, "act_mul", LayerKind.GELU, t, ffn),
    ]


def synth_activation(op: OpSpec, *, seed: int, device, dtype=torch.bfloat16,
                     outlier_frac: float = 0.01, outlier_scale: float = 30.0) -> torch.Tensor:
    """Deterministic synthetic activation for ``op`` generated on ``device``."""
    g = torch.Generator(device=device)
    g.manual_seed(seed * 1000 + op.id)
    shape = (op.rows, op.cols)
    if op.kind is LayerKind.DROPOUT_MASK:
        return torch.rand(shape, generator=g, device=device) < 0.9
    if op.kind is LayerKind.SCORE:
        return (torch.randn(shape, generator=g, device=device) * 3.0).to(dtype)
    if op.kind is LayerKind.SOFTMAX:
        s = torch.randn(shape, generator=g, device=device) * 3.0
        return torch.softmax(s, dim=-1).to(dtype)
    x = torch.randn(shape, generator=g, device=device)
    if op.kind is LayerKind.QKV_MATRIX:
        x = x * torch.exp(torch.randn(op.cols, generator=g, device=device) * 0.5)
    k = max(1, int(op.cols * outlier_frac))
    hot = torch.randperm(op.cols, generator=g, device=device)[:k]
    x[:, hot] *= outlier_scale
    if op.kind is LayerKind.GELU:
        x = torch.nn.functional.gelu(x)
    return x.to(dtype)
