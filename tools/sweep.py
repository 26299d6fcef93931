"""Compressor bandwidth sweep (BASELINE.json configs[4]: 1 MB - 4 GB) and the
Llama-2-7B-shaped layer stack (configs[2]), bf16, on one B200.

    python tools/sweep.py [--out profiles/r1_sweep.json] [--max-mb 4096]

Sizes are powers of two of the bf16 input, cols = 4096 (rows = bytes / 8192).
Each point: the compress and the decompress of every scheme, timed as a
CUDA-graph replay of REPS calls over enough rotating inputs to exceed L2
(126 MB), so each call reads from HBM; GB/s uses the algorithmic bytes
(SURVEY.md 8(d)).  Outlier-separated inputs carry 1% hot channels.
Everything is device-generated (synthetic), one slot per rotating input.
"""
import argparse
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import torch  # noqa: E402

import paper_2508_00806_b200 as adc  # noqa: E402
from paper_2508_00806_b200.slots import CodecSlot  # noqa: E402

REPS = 10
SCHEMES = [("symmetric", adc.SchemeSpec(adc.Scheme.SYMMETRIC_GROUP)),
           ("asymmetric", adc.SchemeSpec(adc.Scheme.ASYMMETRIC_GROUP)),
           ("outlier_separated", adc.SchemeSpec(adc.Scheme.OUTLIER_SEPARATED)),
           ("per_channel", adc.SchemeSpec(adc.Scheme.SYMMETRIC_GROUP, 0)),
           ("bitmask", adc.SchemeSpec(adc.Scheme.BIT_MASK, 0))]


def graph_time(fns):
    """Mean us per call of one CUDA-graph replay of REPS calls cycling over fns."""
    sp = torch.cuda.current_stream().cuda_stream
    for f in fns:
        f(sp)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        sp = torch.cuda.current_stream().cuda_stream
        for i in range(REPS):
            fns[i % len(fns)](sp)
    g.replay()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    g.replay()
    b.record()
    b.synchronize()
    return a.elapsed_time(b) * 1e3 / REPS


def make_input(name, rows, cols, gen):
    if name == "bitmask":
        return torch.rand(rows, cols, device="cuda", generator=gen) < 0.9
    x = torch.randn(rows, cols, device="cuda", generator=gen)
    if name == "asymmetric":
        x = x * 3
    if name in ("outlier_separated", "symmetric", "per_channel"):
        x[:, ::100] *= 30
    return x.to(torch.bfloat16)


def measure(name, spec, rows, cols, nbuf, gen):
    xs = [make_input(name, rows, cols, gen) for _ in range(nbuf)]
    in_dt = torch.bool if name == "bitmask" else torch.bfloat16
    out_dt = torch.uint8 if name == "bitmask" else torch.bfloat16
    k_cap = max(16, cols // 50) if name == "outlier_separated" else None
    slots = [CodecSlot(rows, cols, spec, in_dt, out_dt, k_cap=k_cap) for _ in range(nbuf)]
    ys = [torch.empty((rows, cols), dtype=out_dt, device="cuda") for _ in range(nbuf)]
    tc = graph_time([lambda sp, s=s, x=x: s.compress_ptr(x.data_ptr(), sp) for s, x in zip(slots, xs)])
    td = graph_time([lambda sp, s=s, y=y: s.decompress_ptr(y.data_ptr(), sp) for s, y in zip(slots, ys)])
    s = slots[0]
    k = int(s.k_status[1]) if s.k_cap else 0
    bc, bd = s.algorithmic_bytes(k)
    err = int(s.status[0])
    return {"compress_us": round(tc, 2), "decompress_us": round(td, 2),
            "compress_gbs": round(bc / tc / 1e3, 1), "decompress_gbs": round(bd / td / 1e3, 1),
            "k": k, "error_word": err}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default="profiles/r1_sweep.json")
    ap.add_argument("--max-mb", type=int, default=4096)
    a = ap.parse_args()
    gen = torch.Generator(device="cuda").manual_seed(0)
    res = {"device": torch.cuda.get_device_name(0), "dtype": "bf16", "timing": "CUDA graph of %d calls, "
           "rotating inputs > L2" % REPS, "sweep": [], "llama": []}
    cols = 4096
    mb = 1
    while mb <= a.max_mb:
        rows = max(1, (mb << 20) // (2 * cols))
        nbuf = max(1, min(REPS, (256 << 20) // (rows * cols * 2) + 1))
        point = {"mb": mb, "shape": [rows, cols]}
        for name, spec in SCHEMES:
            point[name] = measure(name, spec, rows, cols, nbuf, gen)
        res["sweep"].append(point)
        print(json.dumps(point), flush=True)
        torch.cuda.empty_cache()
        mb *= 2
    # Llama-2-7B layer stack (h 4096, FFN 11008, seq 4096), batch 1, 2, 4
    for batch in (1, 2, 4):
        for label, cols_l, name in (("attn_in [4096]", 4096, "outlier_separated"),
                                    ("qkv [4096]", 4096, "per_channel"),
                                    ("mlp [11008]", 11008, "outlier_separated")):
            rows = 4096 * batch
            nbuf = max(1, min(REPS, (256 << 20) // (rows * cols_l * 2) + 1))
            spec = dict(SCHEMES)[name]
            r = measure(name, spec, rows, cols_l, nbuf, gen)
            r.update({"batch": batch, "tensor": label, "scheme": name, "shape": [rows, cols_l]})
            res["llama"].append(r)
            print(json.dumps(r), flush=True)
            torch.cuda.empty_cache()
    Path(a.out).write_text(json.dumps(res, indent=1) + "\n")


if __name__ == "__main__":
    main()
