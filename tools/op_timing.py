"""Per-entry-point device timings (CUDA events, median of N) for kernel tuning.

    python tools/op_timing.py [rows cols]
"""
import statistics
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import torch  # noqa: E402

import paper_2508_00806_b200 as adc  # noqa: E402
from paper_2508_00806_b200 import _lib  # noqa: E402
from paper_2508_00806_b200.slots import CodecSlot  # noqa: E402


def timeit(fn, n=30):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    ts = []
    # rotate a large buffer between iterations so inputs are not L2-resident
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    for _ in range(n):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        b.synchronize()
        ts.append(a.elapsed_time(b) * 1e3)
    return statistics.median(ts)


def main():
    shapes = [(8192, 1024), (8192, 4096), (8192, 3072), (131072, 1024)]
    if len(sys.argv) == 3:
        shapes = [(int(sys.argv[1]), int(sys.argv[2]))]
    sp = torch.cuda.current_stream().cuda_stream
    lib = _lib.lib()
    for rows, cols in shapes:
        x = torch.randn(rows, cols, device="cuda", dtype=torch.bfloat16)
        x[:, ::97] *= 30
        nbytes = x.numel() * 2
        print(f"--- [{rows},{cols}] bf16 ({nbytes / 1e6:.1f} MB)")
        ws_bytes = lib.adc_workspace_bytes(2, rows, cols, 128)
        ws = torch.zeros(ws_bytes, dtype=torch.uint8, device="cuda")
        idx = torch.empty(cols, dtype=torch.int32, device="cuda")
        st = torch.zeros(2, dtype=torch.int32, device="cuda")
        t = timeit(lambda: lib.adc_detect_outliers(x.data_ptr(), 1, rows, cols, 3.0, cols, idx.data_ptr(),
                                                    st.data_ptr() + 4, st.data_ptr(), ws.data_ptr(), ws_bytes, sp))
        print(f"detect_outliers (colstats+stats)  {t:8.1f} us  {nbytes / t / 1e3:7.0f} GB/s")
        for name, spec in [("sym128", adc.SchemeSpec(adc.Scheme.SYMMETRIC_GROUP)),
                           ("asym128", adc.SchemeSpec(adc.Scheme.ASYMMETRIC_GROUP)),
                           ("outlier128", adc.SchemeSpec(adc.Scheme.OUTLIER_SEPARATED)),
                           ("per-channel", adc.SchemeSpec(adc.Scheme.SYMMETRIC_GROUP, 0))]:
            s = CodecSlot(rows, cols, spec, torch.bfloat16, torch.bfloat16, k_cap=cols // 8)
            y = torch.empty_like(x)
            tc = timeit(lambda: s.compress_ptr(x.data_ptr(), sp))
            td = timeit(lambda: s.decompress_ptr(y.data_ptr(), sp))
            k = int(s.k_status[1]) if s.k_cap else 0
            bc, bd = s.algorithmic_bytes(k)
            print(f"{name:12s} compress {tc:8.1f} us {bc / tc / 1e3:7.0f} GB/s | decompress {td:8.1f} us "
                  f"{bd / td / 1e3:7.0f} GB/s  (k={k})")
        m = torch.rand(rows, cols, device="cuda") < 0.9
        s = CodecSlot(rows, cols, adc.SchemeSpec(adc.Scheme.BIT_MASK, 0), torch.bool)
        y = torch.empty((rows, cols), dtype=torch.uint8, device="cuda")
        tc = timeit(lambda: s.compress_ptr(m.data_ptr(), sp))
        td = timeit(lambda: s.decompress_ptr(y.data_ptr(), sp))
        bc, bd = s.algorithmic_bytes(0)
        print(f"{'mask':12s} compress {tc:8.1f} us {bc / tc / 1e3:7.0f} GB/s | decompress {td:8.1f} us "
              f"{bd / td / 1e3:7.0f} GB/s")


if __name__ == "__main__":
    main()
