"""Gradient fidelity per saving plan: cosine similarity and relative error of
the full parameter gradient against retain-all, one batch, GPT-345M-shaped
(optionally after some training steps so attention is not uniform).

    python tools/grad_probe.py [model] [train_steps]
"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_2508_00806_b200.gpt import BLOCK_OPS, GPT, GPTConfig, synthetic_batch  # noqa: E402
from paper_2508_00806_b200.hooks import ActivationPolicy  # noqa: E402
from paper_2508_00806_b200.profiles import LayerKind  # noqa: E402


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "gpt-345m"
    warm = int(sys.argv[2]) if len(sys.argv) > 2 else 200
    cfg = GPTConfig.named(name)
    torch.manual_seed(0)
    model = GPT(cfg).cuda().to(torch.bfloat16)
    opt = torch.optim.AdamW(model.parameters(), lr=3e-4, betas=(0.9, 0.95), fused=True)
    keep = ActivationPolicy(BLOCK_OPS, {})
    for s in range(warm):  # train a little so the attention is not uniform
        for g in opt.param_groups:
            g["lr"] = 3e-4 * min(1.0, (s + 1) / 100)
        idx, tgt = synthetic_batch(s, 0, 8, cfg.seq, cfg.vocab, "cuda")
        model(idx, tgt, keep, seed=s).backward()
        opt.step()
        opt.zero_grad(set_to_none=True)
    idx, tgt = synthetic_batch(10**6, 0, 8, cfg.seq, cfg.vocab, "cuda")

    def grads(plan, overrides=None):
        model.zero_grad(set_to_none=True)
        pol = ActivationPolicy(BLOCK_OPS, plan, codec_overrides=overrides)
        loss = model(idx, tgt, pol, seed=7)
        loss.backward()
        return torch.cat([p.grad.float().flatten() for n, p in model.named_parameters()
                          if not n.startswith(("wte", "wpe"))])

    g0 = grads({})
    C = "compress"
    plans = [("softmax(4)", {4: C}), ("scores(6)", {6: C}), ("softmax+scores", {4: C, 6: C}),
             ("mask(5)", {5: C}), ("qkv(3)", {3: C}), ("block_input(1)", {1: C}),
             ("outlier ops 1,2,7,8,9,10,11", {i: C for i in (1, 2, 7, 8, 9, 10, 11)}),
             ("all", {i: C for i in range(1, 12)})]
    for label, plan in plans:
        g = grads(plan)
        cos = torch.nn.functional.cosine_similarity(g0, g, dim=0).item()
        rel = ((g - g0).norm() / g0.norm()).item()
        print(f"{label:32s} cos {cos:.5f}  rel err {rel:.4f}", flush=True)
    for label, plan in [("softmax(4) int8", {4: C}), ("softmax+scores int8", {4: C, 6: C})]:
        g = grads(plan, {LayerKind.SOFTMAX: "int8", LayerKind.SCORE: "int8"})
        cos = torch.nn.functional.cosine_similarity(g0, g, dim=0).item()
        rel = ((g - g0).norm() / g0.norm()).item()
        print(f"{label:32s} cos {cos:.5f}  rel err {rel:.4f}", flush=True)


if __name__ == "__main__":
    main()
