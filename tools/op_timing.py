"""Per-entry-point device timings for kernel tuning.

    python tools/op_timing.py [rows cols]

Each measurement runs REPS back-to-back launches over a rotation of input
buffers whose total exceeds L2, between one pair of CUDA events, and reports
the mean per launch (so launch gaps are included, event overhead is not).
With --graph the REPS calls are captured once in a CUDA graph and replayed,
which removes the host-side submission cost (ctypes + launch) from the
measurement -- the way a captured training step or bench step runs them.
"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import torch  # noqa: E402

import paper_2508_00806_b200 as adc  # noqa: E402
from paper_2508_00806_b200 import _lib  # noqa: E402
from paper_2508_00806_b200.slots import CodecSlot  # noqa: E402

REPS = 20
GRAPH = "--graph" in sys.argv
# --opt=KEY=VALUE: adc_set_option tuning switch for this run (repeatable)
for _a in sys.argv[1:]:
    if _a.startswith("--opt="):
        _k, _v = _a[len("--opt="):].split("=", 1)
        _lib.set_option(_k, int(_v))


def _sp():
    return torch.cuda.current_stream().cuda_stream


def timeit(fns):
    """fns take the raw stream handle; mean us per call over REPS calls."""
    for f in fns[:3]:
        f(_sp())
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if GRAPH:
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            for i in range(REPS):
                fns[i % len(fns)](_sp())
        g.replay()
        torch.cuda.synchronize()
        a.record()
        g.replay()
        b.record()
    else:
        a.record()
        for i in range(REPS):
            fns[i % len(fns)](_sp())
        b.record()
    b.synchronize()
    return a.elapsed_time(b) * 1e3 / REPS


def main():
    shapes = [(8192, 1024), (8192, 4096), (8192, 3072), (131072, 1024), (131072, 64)]
    args = [a for a in sys.argv[1:] if not a.startswith("--")]
    if len(args) == 2:
        shapes = [(int(args[0]), int(args[1]))]
    lib = _lib.lib()
    for rows, cols in shapes:
        nbytes = rows * cols * 2
        nbuf = max(2, (400 << 20) // nbytes + 1)
        xs = []
        for i in range(nbuf):
            x = torch.randn(rows, cols, device="cuda", dtype=torch.bfloat16)
            x[:, ::97] *= 30
            xs.append(x)
        print(f"--- [{rows},{cols}] bf16 ({nbytes / 1e6:.1f} MB), {nbuf} rotating inputs")
        ws_bytes = lib.adc_workspace_bytes(2, rows, cols, 128)
        ws = torch.zeros(ws_bytes, dtype=torch.uint8, device="cuda")
        idx = torch.empty(cols, dtype=torch.int32, device="cuda")
        st = torch.zeros(2, dtype=torch.int32, device="cuda")
        t = timeit([lambda sp, x=x: lib.adc_detect_outliers(x.data_ptr(), 1, rows, cols, 3.0, cols, idx.data_ptr(),
                                                             st.data_ptr() + 4, st.data_ptr(), ws.data_ptr(),
                                                             ws_bytes, sp) for x in xs])
        print(f"detect_outliers (colstats+stats)  {t:8.1f} us  {nbytes / t / 1e3:7.0f} GB/s")
        sums = torch.empty(cols, dtype=torch.float64, device="cuda")
        t = timeit([lambda sp, x=x: lib.adc_channel_abs_sums(x.data_ptr(), 1, rows, cols, sums.data_ptr(),
                                                              st.data_ptr(), ws.data_ptr(), ws_bytes, sp) for x in xs])
        print(f"channel_abs_sums (colstats only)  {t:8.1f} us  {nbytes / t / 1e3:7.0f} GB/s")
        for name, spec in [("sym128", adc.SchemeSpec(adc.Scheme.SYMMETRIC_GROUP)),
                           ("asym128", adc.SchemeSpec(adc.Scheme.ASYMMETRIC_GROUP)),
                           ("outlier128", adc.SchemeSpec(adc.Scheme.OUTLIER_SEPARATED)),
                           ("per-channel", adc.SchemeSpec(adc.Scheme.SYMMETRIC_GROUP, 0))]:
            slots = [CodecSlot(rows, cols, spec, torch.bfloat16, torch.bfloat16, k_cap=cols // 8)
                     for _ in range(min(nbuf, 4))]
            ys = [torch.empty_like(xs[0]) for _ in range(len(slots))]
            tc = timeit([lambda sp, s=s, x=x: s.compress_ptr(x.data_ptr(), sp)
                         for s, x in zip(slots, xs)])
            td = timeit([lambda sp, s=s, y=y: s.decompress_ptr(y.data_ptr(), sp)
                         for s, y in zip(slots, ys)])
            s = slots[0]
            k = int(s.k_status[1]) if s.k_cap else 0
            bc, bd = s.algorithmic_bytes(k)
            print(f"{name:12s} compress {tc:8.1f} us {bc / tc / 1e3:7.0f} GB/s | decompress {td:8.1f} us "
                  f"{bd / td / 1e3:7.0f} GB/s  (k={k})")
        # extensions with float32 scales (int8 codes, int4 codes), g = 128
        n = rows * cols
        for name, fn_c, fn_d, cbytes in [("int8/f32", lib.adc_compress_int8, lib.adc_decompress_int8, n),
                                        ("int4/f32", lib.adc_compress_int4f32, lib.adc_decompress_int4f32,
                                         (n + 1) // 2)]:
            bufs = [(torch.empty(cbytes, dtype=torch.uint8, device="cuda"),
                     torch.empty(n // 128, dtype=torch.float32, device="cuda"),
                     torch.zeros(1, dtype=torch.int32, device="cuda")) for _ in range(min(nbuf, 4))]
            ys = [torch.empty_like(xs[0]) for _ in bufs]
            tc = timeit([lambda sp, b=b, x=x: fn_c(x.data_ptr(), 1, rows, cols, 128, b[0].data_ptr(),
                                                   b[1].data_ptr(), b[2].data_ptr(), sp)
                         for b, x in zip(bufs, xs)])
            td = timeit([lambda sp, b=b, y=y: fn_d(b[0].data_ptr(), b[1].data_ptr(), rows, cols, 128,
                                                   y.data_ptr(), 1, sp) for b, y in zip(bufs, ys)])
            bc = nbytes + cbytes + 4 * (n // 128)
            print(f"{name:12s} compress {tc:8.1f} us {bc / tc / 1e3:7.0f} GB/s | decompress {td:8.1f} us "
                  f"{bc / td / 1e3:7.0f} GB/s")
        ms = [torch.rand(rows, cols, device="cuda") < 0.9 for _ in range(min(nbuf, 4))]
        slots = [CodecSlot(rows, cols, adc.SchemeSpec(adc.Scheme.BIT_MASK, 0), torch.bool) for _ in ms]
        ys = [torch.empty((rows, cols), dtype=torch.uint8, device="cuda") for _ in ms]
        tc = timeit([lambda sp, s=s, m=m: s.compress_ptr(m.data_ptr(), sp) for s, m in zip(slots, ms)])
        td = timeit([lambda sp, s=s, y=y: s.decompress_ptr(y.data_ptr(), sp) for s, y in zip(slots, ys)])
        bc, bd = slots[0].algorithmic_bytes(0)
        print(f"{'mask':12s} compress {tc:8.1f} us {bc / tc / 1e3:7.0f} GB/s | decompress {td:8.1f} us "
              f"{bd / td / 1e3:7.0f} GB/s")
        del xs


if __name__ == "__main__":
    main()
