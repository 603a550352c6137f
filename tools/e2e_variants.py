"""A/B of host-pipeline variants on the bench's end-to-end step (clear, insert_host(sync=False),
retrieve_host of 2^28 keys at load 0.95), CUDA-event timed like bench.py."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2009_07914_b200 import SingleValueHashTable, _io, _lib  # noqa: E402

orig = _io.pipelined


def variant(d2h_streams=1, taper=0):
    outs_streams = {}

    def pipelined(device, inputs, outputs, run, chunk, staging=None):
        n = inputs[0].numel()
        if n == 0:
            return
        dev = torch.device("cuda", device)
        compute = torch.cuda.current_stream(dev)
        bufs, free, s_in, s_out0 = staging.get(device, min(chunk, n), tuple(x.dtype for x in inputs))
        key = (device, chunk, tuple(x.dtype for x in inputs))
        if key not in outs_streams:
            outs_streams[key] = [s_out0] + [torch.cuda.Stream(dev) for _ in range(d2h_streams - 1)]
        souts = outs_streams[key]
        bounds = list(range(0, n, chunk)) + [n]
        if taper and len(bounds) > 2:  # the last chunk in `taper` pieces: a shorter drain
            lo = bounds[-2]
            step = -(-(n - lo) // taper)
            bounds = bounds[:-2] + list(range(lo, n, step)) + [n]
        nb = len(bufs)
        for c in range(len(bounds) - 1):
            lo, hi = bounds[c], bounds[c + 1]
            m = hi - lo
            b = c % nb
            ev_in = torch.cuda.Event()
            with torch.cuda.stream(s_in):
                if free[b] is not None:
                    s_in.wait_event(free[b])
                for d, x in zip(bufs[b], inputs):
                    d[:m].copy_(x[lo:hi], non_blocking=True)
                ev_in.record(s_in)
            compute.wait_event(ev_in)
            outs = run([d[:m] for d in bufs[b]], compute)
            ev_done = torch.cuda.Event()
            ev_done.record(compute)
            free[b] = ev_done
            so = souts[c % len(souts)]
            with torch.cuda.stream(so):
                so.wait_event(ev_done)
                for o, y in zip(outs, outputs):
                    o.record_stream(so)
                    y[lo:hi].copy_(o, non_blocking=True)
        for so in souts:
            compute.wait_stream(so)
    return pipelined


n = 1 << 28
dev = torch.device("cuda", 0)
keys, vals = bench.make_keys(0, n, 1, dev)
hk, hv = keys.cpu().pin_memory(), vals.cpu().pin_memory()
t = SingleValueHashTable(int(n / 0.95) + 1, layout="packed", key_bits=32, value_bits=32, group_width=8)
st = torch.empty(n, dtype=torch.uint8).pin_memory()
ov = torch.empty(n, dtype=torch.int32).pin_memory()
of = torch.empty(n, dtype=torch.uint8).pin_memory()
stream = torch.cuda.current_stream(dev)
configs = [("baseline", None), ("d2h x2", variant(2, 0)), ("taper 4", variant(1, 4)), ("d2h x2 + taper 4", variant(2, 4)),
           ("baseline", None)]
for name, fn in configs:
    _io.pipelined = fn or orig
    t._stage = None
    for rep in range(2):
        _lib.check(_lib.lib().ch_clear(t._dt.handle, stream.cuda_stream))
        t.insert_host(hk, hv, status_out=st, sync=False)
        t.retrieve_host(hk, values_out=ov, found_out=of)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for rep in range(3):
        _lib.check(_lib.lib().ch_clear(t._dt.handle, stream.cuda_stream))
        t.insert_host(hk, hv, status_out=st, sync=False)
        t.retrieve_host(hk, values_out=ov, found_out=of)
    e1.record(stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 3
    ok = bool((ov == hv).all()) and bool((of == 1).all()) and bool((st == 0).all())
    print(f"{name:20s} {ms:7.2f} ms  {2 * n / ms / 1e6:5.2f} G ops/s  ok={ok}", flush=True)
