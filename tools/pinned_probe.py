"""Pinned-buffer flavours for the e2e leg: torch pin_memory vs 2 MB-aligned
anonymous memory with MADV_HUGEPAGE registered by cudaHostRegister.  Prints
H2D / D2H / concurrent GB/s for ~0.9 GB each way (the step's volume)."""
import ctypes
import mmap
import sys

import torch

SIZE = 9 * (100 << 20)
libc = ctypes.CDLL("libc.so.6", use_errno=True)


def thp_pinned(nbytes):
    buf = mmap.mmap(-1, nbytes + (2 << 20), flags=mmap.MAP_PRIVATE | mmap.MAP_ANONYMOUS)
    base = ctypes.addressof(ctypes.c_char.from_buffer(buf))
    off = (-base) % (2 << 20)
    libc.madvise(ctypes.c_void_p(base + off), ctypes.c_size_t(nbytes), 14)  # MADV_HUGEPAGE
    mv = memoryview(buf)[off:off + nbytes]
    t = torch.frombuffer(mv, dtype=torch.uint8)
    t.fill_(1)
    rc = torch.cuda.cudart().cudaHostRegister(t.data_ptr(), nbytes, 0)
    assert int(rc) == 0, rc
    return t, buf


def measure(h_in, h_out):
    d_in = torch.empty(SIZE, dtype=torch.uint8, device="cuda")
    d_out = torch.empty(SIZE, dtype=torch.uint8, device="cuda")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    res = {}
    for name in ("h2d", "d2h", "both"):
        for rep in range(3):
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            if name in ("h2d", "both"):
                with torch.cuda.stream(s1):
                    d_in.copy_(h_in, non_blocking=True)
            if name in ("d2h", "both"):
                with torch.cuda.stream(s2):
                    h_out.copy_(d_out, non_blocking=True)
            for s in (s1, s2):
                torch.cuda.current_stream().wait_stream(s)
            b.record()
            torch.cuda.synchronize()
            res[name] = SIZE / 1e9 / (a.elapsed_time(b) / 1e3)
    return res


kind = sys.argv[1]
if kind == "torch":
    hi = torch.empty(SIZE, dtype=torch.uint8, pin_memory=True)
    ho = torch.empty(SIZE, dtype=torch.uint8, pin_memory=True)
else:
    hi, _k1 = thp_pinned(SIZE)
    ho, _k2 = thp_pinned(SIZE)
r = measure(hi, ho)
print(kind, {k: round(v, 1) for k, v in r.items()}, "pinned:", hi.is_pinned())
