"""insert_host / retrieve_host time per schedule and chunk size (2^28 keys, load 0.95)."""
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


def timed(f):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    f()
    torch.cuda.synchronize()
    return 1e3 * (time.perf_counter() - t0)


c = t.capacity
for mode in ("staged", "on"):
    t.set_locality(mode)
    for div in (8, 12, 24):
        ch = max(1 << 20, -(-c // div))
        best_i, best_r = 1e9, 1e9
        for rep in range(3):
            _lib.check(_lib.lib().ch_clear(t._dt.handle, torch.cuda.current_stream().cuda_stream))
            ti = timed(lambda: t.insert_host(hk, hv, chunk=ch, status_out=st))
            tr = timed(lambda: t.retrieve_host(hk, chunk=ch, values_out=ov, found_out=of))
            if rep:
                best_i, best_r = min(best_i, ti), min(best_r, tr)
        ok = bool((ov == hv).all()) and bool((of == 1).all())
        print(f"{mode:7s} chunk=c/{div:<3d} ({ch:>10d})  insert_host {best_i:7.2f} ms  retrieve_host {best_r:7.2f} ms"
              f"  step {best_i + best_r:7.2f} ms  ok={ok}", flush=True)
