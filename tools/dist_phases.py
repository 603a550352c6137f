"""Per-phase device times (split = the one-pass route partition ShardedTable uses, beside the
stable split with the inverse map; back-map = coalesced gathers) of the hash-partitioned path at the headline size on ONE B200
(2^28 keys per rank, S = 8 destinations): the route + split of the insert batch (keys +
values) and of the retrieve batch, the inverse-permutation scatters of the results, and the
local insert / retrieve of a full 2^28 batch -- the inputs to the weak-scaling model in
DESIGN.md §6 (the exchange itself needs 2+ GPUs and is modelled from NVLink bandwidth)."""
import json
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2009_07914_b200 import SingleValueHashTable
from paper_2009_07914_b200.distributed import gather_device32
from paper_2009_07914_b200.workloads import unique_keys_device


def timed(fn, reps=5):
    out = None
    ts = []
    for r in range(reps + 1):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        a.record()
        out = fn()
        b.record()
        torch.cuda.synchronize()
        if r:
            ts.append(a.elapsed_time(b))
    return sum(ts) / len(ts), out


n, S = 1 << 28, 8
dev = torch.device("cuda", 0)
keys = unique_keys_device(0, n, n, dev)
vals = keys.clone()
res = {"n": n, "shards": S}
from paper_2009_07914_b200 import _lib  # noqa: E402
# outputs preallocated: the timing is the kernels', not the allocator's
perm = torch.empty(n, dtype=torch.int32, device=dev)
off = torch.empty(S + 1, dtype=torch.int64, device=dev)
ko, vo = torch.empty_like(keys), torch.empty_like(vals)
strm = lambda: torch.cuda.current_stream().cuda_stream


def split(with_vals):
    _lib.check(_lib.lib().ch_route_split32(keys.data_ptr(), 4, vals.data_ptr() if with_vals else None, 4, n, S,
                                           perm.data_ptr(), off.data_ptr(), ko.data_ptr(),
                                           vo.data_ptr() if with_vals else None, 0, strm()))


res["stable_split_insert_ms"], _ = timed(lambda: split(True))
res["stable_split_retrieve_ms"], _ = timed(lambda: split(False))
# the one-pass partition ShardedTable uses (ch_route_part32, fixed-capacity segments)
cap = int(n / S * 1.05) + 4096
kp, vp = torch.empty(S * cap, dtype=keys.dtype, device=dev), torch.empty(S * cap, dtype=vals.dtype, device=dev)
cnt = torch.empty(S, dtype=torch.int64, device=dev)
flag = torch.empty(1, dtype=torch.int32, device=dev)


def part(with_vals):
    _lib.check(_lib.lib().ch_route_part32(keys.data_ptr(), vals.data_ptr() if with_vals else None, n, S, cap,
                                          perm.data_ptr(), cnt.data_ptr(), kp.data_ptr(),
                                          vp.data_ptr() if with_vals else None, flag.data_ptr(), 0, strm()))


res["split_insert_ms"], _ = timed(lambda: part(True))
res["split_retrieve_ms"], _ = timed(lambda: part(False))
assert int(flag.item()) == 0
st = torch.zeros(n, dtype=torch.uint8, device=dev)
out8 = torch.empty_like(st)
res["scatter_status_ms"], _ = timed(lambda: gather_device32(st, perm, out8))
v = torch.zeros(n, dtype=torch.int32, device=dev)
out32 = torch.empty_like(v)
res["scatter_values_found_ms"], _ = timed(lambda: (gather_device32(v, perm, out32), gather_device32(st, perm, out8)))
t = SingleValueHashTable(math.ceil(n * 1.001 / 0.95), layout="packed", key_bits=32, value_bits=32, group_width=8)
from paper_2009_07914_b200 import _lib


stt = torch.empty(n, dtype=torch.uint8, device=dev)


def ins():
    _lib.check(_lib.lib().ch_clear(t._dt.handle, torch.cuda.current_stream().cuda_stream))
    return t.insert_device(keys, vals, status=stt)


res["local_clear_insert_ms"], _ = timed(ins)
ov = torch.empty(n, dtype=torch.int32, device=dev)
of = torch.empty(n, dtype=torch.uint8, device=dev)
res["local_retrieve_ms"], _ = timed(lambda: t.retrieve_device(keys, values_out=ov, found_out=of))
print(json.dumps(res))
