"""Element inserts into a large bucket-list table: device time per insert() call (O(batch) passes)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2009_07914_b200 import BucketListHashTable

n = 1 << 23
t = BucketListHashTable(int(n / 0.8), 4 * n, key_bits=32, value_bits=32)
keys = torch.arange(1, n + 1, dtype=torch.int32, device="cuda")
t.insert_device(keys, keys)
torch.cuda.synchronize()
k1 = torch.tensor([5], dtype=torch.int32, device="cuda")
for _ in range(5):
    t.insert_device(k1, k1)
torch.cuda.synchronize()
reps = 200
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for r in range(reps):
    t.insert_device(k1, k1 + r)
e1.record()
torch.cuda.synchronize()
print(f"capacity {t.capacity}: element insert {e0.elapsed_time(e1) / reps * 1000:.1f} us of device time per call;"
      f" count(5) = {t.count(5)}")
