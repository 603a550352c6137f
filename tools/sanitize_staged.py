"""Small staged-path run for compute-sanitizer (memcheck / racecheck / synccheck)."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_2009_07914_b200 import SingleValueHashTable

n = 1 << 16
rng = np.random.default_rng(1)
keys = rng.permutation(np.unique(rng.integers(1, (1 << 32) - 3, size=2 * n, dtype=np.uint64)))[:n]
t = SingleValueHashTable(int(n / 0.95), layout="packed", key_bits=32, value_bits=32, group_width=8)
t.set_locality("staged")
st = t.insert_device(keys, keys).cpu().numpy()
v, f = t.retrieve_device(keys)
torch.cuda.synchronize()
print("ok", (st == 0).all(), f.cpu().numpy().all(), t.deferred_count())
