"""Bench-style end-to-end step (clear, insert_host(sync=False), retrieve_host) of 2^28 keys at
load 0.95 for several host chunk sizes (capacity / div)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2009_07914_b200 import SingleValueHashTable, _lib  # noqa: E402

n = 1 << 28
keys, vals = bench.make_keys(0, n, 1, torch.device("cuda", 0))
hk, hv = keys.cpu().pin_memory(), vals.cpu().pin_memory()
t = SingleValueHashTable(int(n / 0.95) + 1, layout="packed", key_bits=32, value_bits=32, group_width=8)
st = torch.empty(n, dtype=torch.uint8).pin_memory()
ov = torch.empty(n, dtype=torch.int32).pin_memory()
of = torch.empty(n, dtype=torch.uint8).pin_memory()
c = t.capacity
divs = [int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "12,16,24,32,48,64").split(",")]
for div in divs:
    ch = max(1 << 20, -(-c // div))
    best = 1e9
    for rep in range(4):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        _lib.check(_lib.lib().ch_clear(t._dt.handle, torch.cuda.current_stream().cuda_stream))
        t.insert_host(hk, hv, chunk=ch, status_out=st, sync=False)
        t.retrieve_host(hk, chunk=ch, values_out=ov, found_out=of)
        torch.cuda.synchronize()
        ms = 1e3 * (time.perf_counter() - t0)
        if rep:
            best = min(best, ms)
    ok = bool((ov == hv).all()) and bool((of == 1).all()) and bool((st == 0).all())
    print(f"div {div:3d} chunk {ch:10d} ({t.batch_schedule(ch)}): {best:7.2f} ms  {2 * n / best / 1e6:6.2f} G ops/s  ok={ok}",
          flush=True)
