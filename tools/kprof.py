"""Per-kernel device times of the multi-value grouped insert, without a replaying profiler.

  python tools/kprof.py [log2 n] [insert|retrieve|bucket_insert|bucket_retrieve]
(CUPTI activity records via torch.profiler)
"""
import math
import os
import sys
from collections import defaultdict

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from torch.profiler import ProfilerActivity, profile

from paper_2009_07914_b200 import BucketListHashTable, GrowthPolicy, MultiValueHashTable

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from bench_configs import power_law_keys, zipf_keys  # noqa: E402

n = 1 << (int(sys.argv[1]) if len(sys.argv) > 1 else 27)
what = sys.argv[2] if len(sys.argv) > 2 else "insert"
dev = torch.device("cuda", 0)
bucket = what.startswith("bucket")
what = what.replace("bucket_", "")
if bucket:
    keys, distinct = power_law_keys(n, 7, dev)
    k32 = keys.to(torch.int32)
    v32 = torch.arange(1, n + 1, device=dev, dtype=torch.int64)
else:
    keys, _ = zipf_keys(n, 1 << 23, 0.5, 42, dev)
    k32 = keys.to(torch.int32)
    v32 = torch.arange(1, n + 1, device=dev, dtype=torch.int32)
for rep in range(3):
    if bucket:
        t = BucketListHashTable(math.ceil(distinct / 0.8), int(n * 2.5) + 64, growth=GrowthPolicy(1, 1.1),
                                key_bits=32, value_bits=64, device=0)
    else:
        t = MultiValueHashTable(math.ceil(n / 0.8), layout="packed", key_bits=32, value_bits=32, group_width=8,
                                device=0)
    torch.cuda.synchronize()
    if what == "retrieve":
        t.insert_device(k32, v32)
        q = torch.unique(keys).to(torch.int32)
        torch.cuda.synchronize()
    op = (lambda: t.retrieve_device(q)) if what == "retrieve" else (lambda: t.insert_device(k32, v32))
    if rep < 2:
        op()
        torch.cuda.synchronize()
        continue
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        op()
        torch.cuda.synchronize()
tot = defaultdict(float)
cnt = defaultdict(int)
for e in prof.events():
    if e.device_type == torch.autograd.DeviceType.CUDA:
        name = e.name[:60]
        tot[name] += e.device_time_total if hasattr(e, "device_time_total") else e.cuda_time_total
        cnt[name] += 1
s = 0.0
for k, v in sorted(tot.items(), key=lambda kv: -kv[1]):
    print(f"{v / 1000:8.3f} ms  x{cnt[k]:2d}  {k}")
    s += v
print(f"{s / 1000:8.3f} ms  total")
