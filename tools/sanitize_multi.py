"""Small grouped multi-value insert + count / retrieve (stash) for compute-sanitizer."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2009_07914_b200 import MultiValueHashTable  # noqa: E402

n = 1 << 15
rng = np.random.default_rng(2)
keys = np.minimum(rng.zipf(1.4, size=n), 5000).astype(np.uint64) * np.uint64(2654435761) % np.uint64(1 << 31) + 1
vals = np.arange(1, n + 1, dtype=np.uint64)
t = MultiValueHashTable(int(n / 0.8), layout="packed", key_bits=32, value_bits=32, group_width=8)
st = t.insert_device(keys, vals).cpu().numpy()
q = torch.from_numpy(np.unique(keys).astype(np.int64)).to(torch.int32).cuda()
off, flat = t.retrieve_device(q)
torch.cuda.synchronize()
print("ok", (st == 0).all(), int(off[-1]) == n)
t64 = MultiValueHashTable(int(n / 0.8), layout="soa", key_bits=64, value_bits=64, group_width=4)
st = t64.insert_device(keys * np.uint64(3), vals).cpu().numpy()
off, flat = t64.retrieve_device(np.unique(keys * np.uint64(3)))
torch.cuda.synchronize()
print("ok64", (st == 0).all(), int(off[-1]) == n)
