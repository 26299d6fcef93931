"""Per-phase timing of the single-pass outlier-separated kernel (k4.cu).

    python tools/k4_trace.py [rows cols [dtype]]

Enables the kernel's phase trace (adc_set_option("k4_trace", 1)), runs one
compress after warm-up and prints, over CTAs, the median / max clock64 at the
end of each phase (us at the max SM clock), then times the three outlier
paths (two launches, single pass, single pass + speculation) as CUDA-graph
replays of 20 calls over rotating inputs.
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

PHASES = [(14, "setup: mbarrier init"), (15, "setup: chunk issue (warp 0)"), (18, "setup: prediction scan"),
          (16, "setup: prediction masks"), (9, "setup: nibble masks"), (1, "A: sums + quantise (warp 0)"),
          (17, "A: all warps done"), (2, "B: fold"), (3, "B: reduce + arrive"), (13, "B: barrier wait"),
          (4, "C: load sums"), (10, "C: mean"), (11, "C: variance tree"), (5, "C: sqrt"),
          (19, "C: flags + scan"), (20, "C: idx / k"), (6, "C: tile list + prediction"),
          (7, "D: re-quantise"), (8, "E: side buffer")]


def graph_time(fns, reps=20):
    sp = torch.cuda.current_stream().cuda_stream
    for f in fns[:3]:
        f(sp)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for i in range(reps):
            fns[i % len(fns)](torch.cuda.current_stream().cuda_stream)
    g.replay()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    g.replay()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) * 1e3 / reps


def main():
    args = [a for a in sys.argv[1:] if not a.startswith("--")]
    shapes = [(8192, 1024), (8192, 4096), (131072, 1024)] if len(args) < 2 else [(int(args[0]), int(args[1]))]
    dtype = getattr(torch, args[2]) if len(args) > 2 else torch.bfloat16
    lib = _lib.lib()
    mhz = 1965.0
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    spec = adc.SchemeSpec(adc.Scheme.OUTLIER_SEPARATED)
    for rows, cols in shapes:
        nbytes = rows * cols * torch.empty((), dtype=dtype).element_size()
        nbuf = max(2, (400 << 20) // nbytes + 1)
        xs = []
        for i in range(nbuf):
            x = torch.randn(rows, cols, device="cuda").to(dtype)
            x[:, ::97] *= 30
            xs.append(x)
        s = CodecSlot(rows, cols, spec, dtype, dtype, k_cap=cols // 8)
        sp = torch.cuda.current_stream().cuda_stream
        _lib.set_option("outlier_path", 1)
        for _ in range(3):
            s.compress_ptr(xs[0].data_ptr(), sp)
        torch.cuda.synchronize()
        _lib.set_option("k4_trace", 1)
        s.compress_ptr(xs[1].data_ptr(), sp)
        torch.cuda.synchronize()
        _lib.set_option("k4_trace", 0)
        NS = 64
        buf = (ctypes.c_ulonglong * (sms * NS))()
        n = lib.adc_debug_trace_k4(ctypes.addressof(buf), sms * NS)
        rec = [list(buf[i * NS:(i + 1) * NS]) for i in range(n // NS)]
        rec = [r for r in rec if r[8] > 0]
        starts = [r[0] for r in rec]
        t0 = min(starts)
        print(f"--- [{rows},{cols}] {dtype}: {len(rec)} CTAs, start spread "
              f"{(max(starts) - t0) / 1e3:.2f} us (median {(statistics.median(starts) - t0) / 1e3:.2f})")
        ends_gt = [r[12] for r in rec]
        print(f"  globaltimer entry->exit: med {statistics.median([e - s for e, s in zip(ends_gt, starts)]) / 1e3:.2f} us, "
              f"first entry -> last exit {(max(ends_gt) - t0) / 1e3:.2f} us; clock64 at exit med "
              f"{statistics.median([r[8] for r in rec]):.0f} cycles")
        wen = [min(r[32:48]) for r in rec]
        wex = [max(r[48:64]) for r in rec]
        print(f"  warps: first entry -> last exit {(max(wex) - min(wen)) / 1e3:.2f} us; per CTA warp-entry spread med "
              f"{statistics.median([max(r[32:48]) - min(r[32:48]) for r in rec]) / 1e3:.2f} us, warp-exit spread med "
              f"{statistics.median([max(r[48:64]) - min(r[48:64]) for r in rec]) / 1e3:.2f} us")
        r0_ = rec[0]
        print("  CTA 0 warp exits (us after CTA entry):", " ".join(f"{(r0_[48 + w] - r0_[0]) / 1e3:.1f}" for w in range(16)))
        prev = [0] * len(rec)
        for p, name in PHASES:
            ends = [r[p] for r in rec]
            dur = [e - q for e, q in zip(ends, prev)]
            print(f"  {name:26s} end med {statistics.median(ends) / mhz:7.2f} max {max(ends) / mhz:7.2f} us"
                  f" | phase med {statistics.median(dur) / mhz:6.2f} max {max(dur) / mhz:6.2f} us")
            prev = ends
        # eager single calls with a sync between (launch gaps excluded by events around each)
        for mode in (0, 1):  # 0: two launches, 1: single pass
            _lib.set_option("outlier_path", mode)
            ts = []
            for it in range(10):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                torch.cuda.synchronize()
                e0.record()
                s.compress_ptr(xs[it % len(xs)].data_ptr(), sp)
                e1.record()
                torch.cuda.synchronize()
                ts.append(e0.elapsed_time(e1) * 1e3)
            print(f"  eager mode {mode}: per call {sorted(ts)[len(ts) // 2]:.1f} us (median of 10)")
        slots = [CodecSlot(rows, cols, spec, dtype, dtype, k_cap=cols // 8) for _ in range(min(nbuf, 4))]
        # a second input family with another outlier channel set: alternating the
        # two through one slot makes every call mispredict
        alt = []
        for i in range(len(slots)):
            x = torch.randn(rows, cols, device="cuda").to(dtype)
            x[:, 5::89] *= 30
            alt.append(x)
        for mode, name, srcs in ((0, "two launches", None), (1, "single pass (hit)", None),
                                 (1, "single pass (miss)", alt)):
            _lib.set_option("outlier_path", mode)
            fns = []
            for j, (sl, x) in enumerate(zip(slots, xs)):
                fns.append(lambda sp, sl=sl, x=x: sl.compress_ptr(x.data_ptr(), sp))
                if srcs is not None:
                    fns.append(lambda sp, sl=sl, x=srcs[j]: sl.compress_ptr(x.data_ptr(), sp))
            if srcs is not None:  # interleave: slot j gets xs[j], alt[j], xs[j], ...
                fns = fns * 2
            t = graph_time(fns)
            kk = int(slots[0].k_status[1])
            bc, _ = slots[0].algorithmic_bytes(kk)
            print(f"  {name:20s} {t:7.1f} us  {bc / t / 1e3:6.0f} GB/s  (k={kk})")
        _lib.set_option("outlier_path", 1)
        del xs


if __name__ == "__main__":
    main()
