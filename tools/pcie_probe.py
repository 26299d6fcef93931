"""PCIe ceiling for bench.py's e2e leg: pinned H2D alone, D2H alone, and both
directions concurrently on two streams (906 MB each way, the step's volume)."""
import torch

n = 906 * (1 << 20) // 9
hs = [torch.empty(n, dtype=torch.uint8, pin_memory=True) for _ in range(9)]
ho = [torch.empty(n, dtype=torch.uint8, pin_memory=True) for _ in range(9)]
ds = [torch.empty(n, dtype=torch.uint8, device="cuda") for _ in range(9)]
do = [torch.empty(n, dtype=torch.uint8, device="cuda") for _ in range(9)]
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def timed(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    for s in (s1, s2):
        torch.cuda.current_stream().wait_stream(s)
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


def h2d():
    with torch.cuda.stream(s1):
        for h, d in zip(hs, ds):
            d.copy_(h, non_blocking=True)


def d2h():
    with torch.cuda.stream(s2):
        for h, d in zip(ho, do):
            h.copy_(d, non_blocking=True)


def both():
    h2d()
    d2h()


tot = 9 * n / 1e9
for name, f in [("H2D", h2d), ("D2H", d2h), ("both", both)]:
    ms = timed(f)
    print(f"{name:5s} {ms:7.2f} ms  {tot / (ms / 1e3):6.1f} GB/s per direction")
