"""Per-chunk timeline of the host pipeline (_io.pipelined): H2D / kernel / D2H intervals (ms)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2009_07914_b200 import SingleValueHashTable, _lib  # noqa: E402

n = 1 << 28
keys, vals = bench.make_keys(0, n, 1, torch.device("cuda", 0))
hk, hv = keys.cpu().pin_memory(), vals.cpu().pin_memory()
t = SingleValueHashTable(int(n / 0.95) + 1, layout="packed", key_bits=32, value_bits=32, group_width=8)
ov = torch.empty(n, dtype=torch.int32).pin_memory()
of = torch.empty(n, dtype=torch.uint8).pin_memory()
st = torch.empty(n, dtype=torch.uint8).pin_memory()
dev = torch.device("cuda", 0)


def run(inputs, outputs, op, chunk):
    compute = torch.cuda.current_stream(dev)
    s_in, s_out = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
    nb = 3
    bufs = [[torch.empty(chunk, dtype=x.dtype, device=dev) for x in inputs] for _ in range(nb)]
    free = [torch.cuda.Event() for _ in range(nb)]
    ev = []
    t0 = torch.cuda.Event(enable_timing=True)
    t0.record(compute)
    s_in.wait_stream(compute)
    for c, lo in enumerate(range(0, n, chunk)):
        hi = min(n, lo + chunk)
        m = hi - lo
        b = c % nb
        e = [torch.cuda.Event(enable_timing=True) for _ in range(6)]
        with torch.cuda.stream(s_in):
            if c >= nb:
                s_in.wait_event(free[b])
            e[0].record(s_in)
            for d, x in zip(bufs[b], inputs):
                d[:m].copy_(x[lo:hi], non_blocking=True)
            e[1].record(s_in)
        compute.wait_event(e[1])
        e[2].record(compute)
        outs = op([d[:m] for d in bufs[b]], compute)
        e[3].record(compute)
        free[b].record(compute)
        with torch.cuda.stream(s_out):
            s_out.wait_event(e[3])
            e[4].record(s_out)
            for o, y in zip(outs, outputs):
                o.record_stream(s_out)
                y[lo:hi].copy_(o, non_blocking=True)
            e[5].record(s_out)
        ev.append(e)
    compute.wait_stream(s_out)
    t1 = torch.cuda.Event(enable_timing=True)
    t1.record(compute)
    torch.cuda.synchronize()
    print(f"total {t0.elapsed_time(t1):.2f} ms")
    for c, e in enumerate(ev):
        r = [t0.elapsed_time(x) for x in e]
        print(f"  chunk {c:2d}: h2d {r[0]:6.2f}-{r[1]:6.2f}  kern {r[2]:6.2f}-{r[3]:6.2f}  d2h {r[4]:6.2f}-{r[5]:6.2f}")


chunk = -(-t.capacity // 24)
for rep in range(2):
    _lib.check(_lib.lib().ch_clear(t._dt.handle, torch.cuda.current_stream().cuda_stream))
    print("insert")
    run([hk, hv], [st], lambda d, s: [t.insert_device(d[0], d[1], stream=s)], chunk)
    print("retrieve")
    run([hk], [ov, of], lambda d, s: list(t.retrieve_device(d[0], stream=s)), chunk)
