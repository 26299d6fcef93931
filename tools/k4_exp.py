"""Timing experiments on the single-pass outlier kernel (k4.cu; results invalid
for dbg != 0): graph-timed per-call time of the full kernel and of variants
that stops after phase A.

    python tools/k4_exp.py rows cols
"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

import paper_2508_00806_b200 as adc  # noqa: E402
from paper_2508_00806_b200 import _lib  # noqa: E402
from paper_2508_00806_b200.slots import CodecSlot  # noqa: E402
from k4_trace import graph_time  # noqa: E402

rows, cols = int(sys.argv[1]), int(sys.argv[2])
spec = adc.SchemeSpec(adc.Scheme.OUTLIER_SEPARATED)
nbuf = max(2, (400 << 20) // (rows * cols * 2) + 1)
xs = []
for i in range(min(nbuf, 4)):
    x = torch.randn(rows, cols, device="cuda").to(torch.bfloat16)
    x[:, ::97] *= 30
    xs.append(x)
slots = [CodecSlot(rows, cols, spec, torch.bfloat16, torch.bfloat16, k_cap=cols // 8) for _ in xs]
fns = [lambda sp, sl=sl, x=x: sl.compress_ptr(x.data_ptr(), sp) for sl, x in zip(slots, xs)]
mb = rows * cols * 2 / 1e6
for mode, name in ((0, "full"), (1, "stop after A")):
    _lib.set_option("k4_dbg", mode)
    t = graph_time(fns)
    print(f"[{rows},{cols}] {name:24s} {t:7.1f} us   ({mb / t * 1e-3 * 1e3:6.0f} GB/s of input)")
_lib.set_option("k4_dbg", 0)
_lib.set_option("outlier_path", 0)
print(f"[{rows},{cols}] two launches             {graph_time(fns):7.1f} us")
_lib.set_option("outlier_path", 1)
