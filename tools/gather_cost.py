"""Cost of the outlier side-buffer gather inside the outlier-separated compress:
the same tensors compressed with the side buffer (k_cap = cols / 8) and
without (k_cap = 0: no channel is flagged for zeroing, no gather), plus the
two paths' detection-only and symmetric-quantiser times (graph-replayed).
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
    _lib.set_option("outlier_path", 0)
    for rows, cols in [(8192, 1024), (8192, 4096), (8192, 8192)]:
        xs = []
        for i in range(max(2, (400 << 20) // (rows * cols * 2) + 1)):
            x = torch.randn(rows, cols, device="cuda", dtype=torch.bfloat16)
            x[:, ::97] *= 30
            xs.append(x)
        line = f"[{rows},{cols}]"
        for name, spec, kc in [("outlier k_cap=cols/8", adc.SchemeSpec(adc.Scheme.OUTLIER_SEPARATED), cols // 8),
                               ("outlier k_cap=0", adc.SchemeSpec(adc.Scheme.OUTLIER_SEPARATED), 0),
                               ("sym", adc.SchemeSpec(adc.Scheme.SYMMETRIC_GROUP), None)]:
            slots = [CodecSlot(rows, cols, spec, torch.bfloat16, k_cap=kc) for _ in range(min(4, len(xs)))]
            t = timeit([lambda sp, s=s, x=x: s.compress_ptr(x.data_ptr(), sp) for s, x in zip(slots, xs)])
            line += f"  {name} {t:6.1f} us"
        print(line, flush=True)
    _lib.set_option("outlier_path", 2)


if __name__ == "__main__":
    main()
