"""Per-phase timing of the single-launch outlier-separated kernel (fused.cu).

    python tools/fused_trace.py [rows cols [dtype]]

Enables the kernel's phase trace (adc_set_option("trace", 1)), runs one
compress after warm-up and prints, over CTAs, the median / max clock64 at the
end of each phase (us at the SM clock) and the spread of CTA start times.
"""
import ctypes
import statistics
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

import paper_2508_00806_b200 as adc  # noqa: E402
from paper_2508_00806_b200 import _lib  # noqa: E402
from paper_2508_00806_b200.slots import CodecSlot  # noqa: E402

PHASES = [(1, "A: colsum (+streamed quant)"), (2, "fold + red.f64"), (3, "grid barrier (warp 0)"), (4, "S load (warp 0)"),
          (8, "stats || resident quant"), (9, "flags + ranks"), (5, "prediction check"), (6, "requantise"), (7, "gather")]


def main():
    args = [a for a in sys.argv[1:] if not a.startswith("--")]
    shapes = [(8192, 1024), (8192, 4096)] if len(args) < 2 else [(int(args[0]), int(args[1]))]
    dtype = getattr(torch, args[2]) if len(args) > 2 else torch.bfloat16
    lib = _lib.lib()
    mhz = torch.cuda.get_device_properties(0).clock_rate / 1e3 if hasattr(torch.cuda.get_device_properties(0), "clock_rate") else 1965.0
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    for rows, cols in shapes:
        x = torch.randn(rows, cols, device="cuda").to(dtype)
        x[:, ::97] *= 30
        s = CodecSlot(rows, cols, adc.SchemeSpec(adc.Scheme.OUTLIER_SEPARATED), dtype, dtype, k_cap=cols // 8)
        sp = torch.cuda.current_stream().cuda_stream
        for _ in range(5):
            s.compress_ptr(x.data_ptr(), sp)
        torch.cuda.synchronize()
        _lib.set_option("trace", 1)
        s.compress_ptr(x.data_ptr(), sp)
        torch.cuda.synchronize()
        _lib.set_option("trace", 0)
        buf = (ctypes.c_ulonglong * (sms * 16))()
        n = lib.adc_debug_trace(ctypes.addressof(buf), sms * 16)
        rec = [list(buf[i * 16:(i + 1) * 16]) for i in range(n // 16)]
        starts = [r[0] for r in rec]
        t0 = min(starts)
        print(f"--- [{rows},{cols}] {dtype}: {len(rec)} CTAs, start spread "
              f"{(max(starts) - t0) / 1e3:.2f} us (median {(statistics.median(starts) - t0) / 1e3:.2f})")
        prev = [0] * len(rec)
        for p, name in PHASES:
            ends = [r[p] for r in rec]
            dur = [e - q for e, q in zip(ends, prev)]
            print(f"  {name:28s} end med {statistics.median(ends) / mhz:7.2f} max {max(ends) / mhz:7.2f} us"
                  f" | phase med {statistics.median(dur) / mhz:6.2f} max {max(dur) / mhz:6.2f} us")
            prev = ends
        for p, name in ((10, "  warp 0 stats done"), (11, "  warp 1 quant done"), (12, "  warp 15 quant done")):
            ends = [r[p] for r in rec]
            print(f"  {name:28s} end med {statistics.median(ends) / mhz:7.2f} max {max(ends) / mhz:7.2f} us")
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(20):
            s.compress_ptr(x.data_ptr(), sp)
        b.record()
        torch.cuda.synchronize()
        print(f"  eager compress {a.elapsed_time(b) * 1e3 / 20:.1f} us/call")


if __name__ == "__main__":
    main()
