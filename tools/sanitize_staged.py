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

# skewed batch over several super-regions: level-1 overflow (gated exact redo) and
# over-full regions (runs handed to the COPS kernels)
from paper_2009_07914_b200.probing import mix64_array  # noqa: E402
t2 = SingleValueHashTable(2_200_000, layout="packed", key_bits=32, value_bits=32, group_width=8)
t2.set_locality("staged")
cand = np.unique(rng.integers(1, (1 << 32) - 3, size=2_000_000, dtype=np.uint64))
h = mix64_array(cand) % np.uint64(t2.capacity)
hot = cand[(h >> np.uint64(21)) == 0][:60_000]
cold = cand[(h >> np.uint64(21)) != 0][:4_000]
k2 = rng.permutation(np.concatenate([hot, cold]))
st2 = t2.insert_device(k2, k2).cpu().numpy()
v2, f2 = t2.retrieve_device(k2)
torch.cuda.synchronize()
print("skew", (st2 == 0).all(), f2.cpu().numpy().all(), (v2.cpu().numpy().view(np.uint32) == k2.astype(np.uint32)).all())

# staged bulk erase (retiring region pass, region write-back, deferred COPS erase), with duplicates
q = np.concatenate([keys[::2], keys[::2][:1000]])
er = t.erase_device(q).cpu().numpy()
v3, f3 = t.retrieve_device(keys)
torch.cuda.synchronize()
print("erase", int(er.sum()) == keys[::2].size, not f3.cpu().numpy()[::2].any(), f3.cpu().numpy()[1::2].all())
