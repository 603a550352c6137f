"""Diagnose the host-buffer path: per-phase timings of insert_host / retrieve_host."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import bench
from paper_2009_07914_b200 import SingleValueHashTable
n = 1 << 28
keys, vals = bench.make_keys(0, n, 1, torch.device("cuda", 0))
hk, hv = keys.cpu().pin_memory(), vals.cpu().pin_memory()
t = SingleValueHashTable(int(n / 0.95) + 1, layout="packed", key_bits=32, value_bits=32, group_width=8)
def timed(name, f):
    torch.cuda.synchronize(); t0 = time.perf_counter(); r = f(); torch.cuda.synchronize()
    print(f"{name:40s} {1e3*(time.perf_counter()-t0):8.2f} ms", flush=True); return r
for rep in range(2):
    from paper_2009_07914_b200 import _lib
    _lib.check(_lib.lib().ch_clear(t._dt.handle, torch.cuda.current_stream().cuda_stream))
    timed("h2d keys+vals (plain)", lambda: (hk.to("cuda", non_blocking=True), hv.to("cuda", non_blocking=True)))
    st = timed("insert_host", lambda: t.insert_host(hk, hv))
    r = timed("retrieve_host", lambda: t.retrieve_host(hk))
    timed("d2h 1.3GB (plain)", lambda: (keys.to("cpu"),))
    for ch in (1 << 24, 1 << 26):
        _lib.check(_lib.lib().ch_clear(t._dt.handle, torch.cuda.current_stream().cuda_stream))
        timed(f"insert_host chunk={ch}", lambda: t.insert_host(hk, hv, chunk=ch))
        timed(f"retrieve_host chunk={ch}", lambda: t.retrieve_host(hk, chunk=ch))
print("ok", bool((r[0] == hv).all()), bool((r[1] == 1).all()))
