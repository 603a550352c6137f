"""Pinned host<->device copy rates on this box: H2D, D2H, and both at once (GB/s)."""
import time

import torch

n = 1 << 28
h_in = torch.empty(n, dtype=torch.int32).pin_memory()
h_out = torch.empty(n, dtype=torch.int32).pin_memory()
d_a = torch.empty(n, dtype=torch.int32, device="cuda")
d_b = torch.empty(n, dtype=torch.int32, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def timed(f):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    f()
    torch.cuda.synchronize()
    return time.perf_counter() - t0


for _ in range(2):
    th = timed(lambda: d_a.copy_(h_in, non_blocking=True))
    td = timed(lambda: h_out.copy_(d_b, non_blocking=True))

    def both():
        with torch.cuda.stream(s1):
            d_a.copy_(h_in, non_blocking=True)
        with torch.cuda.stream(s2):
            h_out.copy_(d_b, non_blocking=True)
    tb = timed(both)
    gb = n * 4 / 1e9
    print(f"H2D {gb / th:6.1f} GB/s   D2H {gb / td:6.1f} GB/s   duplex {2 * gb / tb:6.1f} GB/s (sum)", flush=True)
