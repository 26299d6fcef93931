"""Outlier-separated decompress: dequantise + overwrite launches vs the
one-launch shared-memory tile kernel at each tile size (graph-replayed,
rotating slots, output dtype bf16).

    python tools/odec_sweep.py
"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
sys.argv.append("--graph")

import torch  # noqa: E402

import paper_2508_00806_b200 as adc  # noqa: E402
from paper_2508_00806_b200 import _lib  # noqa: E402
from paper_2508_00806_b200.slots import CodecSlot  # noqa: E402
from op_timing import timeit  # noqa: E402


def main():
    for rows, cols in [(8192, 1024), (8192, 4096), (8192, 3072), (32768, 1024), (131072, 1024), (131072, 64)]:
        slots, ys = [], []
        for i in range(4):
            x = torch.randn(rows, cols, device="cuda", dtype=torch.bfloat16)
            x[:, ::97] *= 30
            s = CodecSlot(rows, cols, adc.SchemeSpec(adc.Scheme.OUTLIER_SEPARATED), torch.bfloat16,
                          torch.bfloat16, k_cap=max(16, cols // 32))
            s.compress(x)
            slots.append(s)
            ys.append(torch.empty_like(x))
        k = int(slots[0].k_status[1])
        bd = slots[0].algorithmic_bytes(k)[1]
        line = f"[{rows},{cols}] k={k}:"
        for mode, tile in [(0, 8192), (2, 4096), (2, 8192), (2, 16384)]:
            _lib.set_option("outlier_decompress", mode)
            _lib.set_option("outlier_tile", tile)
            t = timeit([lambda sp, s=s, y=y: s.decompress_ptr(y.data_ptr(), sp) for s, y in zip(slots, ys)])
            tag = "two" if mode == 0 else f"one/{tile}"
            line += f"  {tag} {t:6.1f} us ({bd / t / 1e3:5.0f} GB/s)"
        _lib.set_option("outlier_decompress", 2)
        _lib.set_option("outlier_tile", 8192)
        print(line, flush=True)


if __name__ == "__main__":
    main()
