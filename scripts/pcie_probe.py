"""PCIe ceiling of this box: pinned H2D, D2H and both at once (the e2e path's bound)."""
import time

import torch

n = 1 << 30
h1 = torch.empty(n, dtype=torch.uint8).pin_memory()
h2 = torch.empty(n, dtype=torch.uint8).pin_memory()
d1 = torch.empty(n, dtype=torch.uint8, device="cuda")
d2 = torch.empty(n, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def bw(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    return reps * n / (time.perf_counter() - t) / 1e9


def h2d():
    d1.copy_(h1, non_blocking=True)


def d2h():
    h2.copy_(d2, non_blocking=True)


def both():
    with torch.cuda.stream(s1):
        d1.copy_(h1, non_blocking=True)
    with torch.cuda.stream(s2):
        h2.copy_(d2, non_blocking=True)


print(f"H2D {bw(h2d):.1f} GB/s  D2H {bw(d2h):.1f} GB/s  both (each direction) {bw(both):.1f} GB/s")
