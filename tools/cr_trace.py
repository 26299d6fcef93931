"""Phase timeline of the column-statistics kernel (colreduce<SUM>) inside an
outlier-separated compress: python tools/cr_trace.py [rows cols ...]

Per CTA: entry, stage A done, arrival; the last CTA: tail start, accumulators
moved, statistics done (globaltimer ns, relative to the first CTA's entry).
"""
import ctypes
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2508_00806_b200 as adc  # noqa: E402
from paper_2508_00806_b200 import _lib  # noqa: E402
from paper_2508_00806_b200.slots import CodecSlot  # noqa: E402

N = 4096 * 4 + 16


def main():
    args = [int(a) for a in sys.argv[1:]] or [8192, 1024, 8192, 4096, 8192, 8192]
    lib = _lib.lib()
    lib.adc_debug_trace_k4.argtypes = [ctypes.POINTER(ctypes.c_ulonglong), ctypes.c_int]
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    _lib.set_option("outlier_path", 0)
    for rows, cols in zip(args[::2], args[1::2]):
        x = torch.randn(rows, cols, device="cuda", dtype=torch.bfloat16)
        x[:, ::97] *= 30
        slot = CodecSlot(rows, cols, adc.SchemeSpec(adc.Scheme.OUTLIER_SEPARATED), torch.bfloat16)
        for _ in range(3):
            slot.compress(x)
        res = []
        for rep in range(5):
            flush.zero_()
            torch.cuda._sleep(1_000_000)
            _lib.set_option("cr_trace", 1)
            slot.compress(x)
            torch.cuda.synchronize()
            buf = (ctypes.c_ulonglong * N)()
            lib.adc_debug_trace_k4(buf, N)  # reads the column-statistics trace while cr_trace is on
            _lib.set_option("cr_trace", 0)
            a = np.frombuffer(buf, dtype=np.uint64).astype(np.int64)
            cta = a[: 4096 * 4].reshape(4096, 4)
            tail = a[4096 * 4: 4096 * 4 + 3]
            sm = a[4096 * 4 + 4: 4096 * 4 + 8]
            t_last = tail[0]
            live = (cta[:, 0] > t_last - 1_000_000) & (cta[:, 0] <= t_last)
            c = cta[live]
            t0 = c[:, 0].min()
            res.append([c.shape[0], c[:, 0].max() - t0, np.median(c[:, 1] - t0), c[:, 1].max() - t0,
                        c[:, 2].max() - t0, tail[0] - t0, tail[1] - t0, tail[2] - t0] + list(sm - t0))
        r = np.median(np.array(res, dtype=np.float64), axis=0)
        print(f"[{rows},{cols}] {int(r[0])} CTAs: entry spread {r[1] / 1e3:.2f} us, stage A done median "
              f"{r[2] / 1e3:.2f} / max {r[3] / 1e3:.2f} us, last arrival {r[4] / 1e3:.2f}, tail start "
              f"{r[5] / 1e3:.2f}, moved {r[6] / 1e3:.2f}, stats done {r[7] / 1e3:.2f} us (mean {r[8] / 1e3:.2f}, "
              f"var {r[9] / 1e3:.2f}, flags {r[10] / 1e3:.2f}, scan {r[11] / 1e3:.2f})", flush=True)
    _lib.set_option("outlier_path", 2)


if __name__ == "__main__":
    main()
