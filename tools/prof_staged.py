"""One staged insert + retrieve of n unique keys at load 0.95 (ncu target; n = argv[1], default 2^24)."""
import math
import sys

import torch

sys.path.insert(0, ".")
from bench import make_keys  # noqa: E402
from paper_2009_07914_b200 import SingleValueHashTable, _lib  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 24
mode = sys.argv[2] if len(sys.argv) > 2 else "staged"
dev = torch.device("cuda", 0)
keys, vals = make_keys(0, n, 1, dev)
t = SingleValueHashTable(math.ceil(n / 0.95), layout="packed", key_bits=32, value_bits=32, group_width=8)
t.set_locality(mode)
for _ in range(2):
    _lib.check(_lib.lib().ch_clear(t._dt.handle, torch.cuda.current_stream().cuda_stream), "clear")
    st = t.insert_device(keys, vals)
    v, f = t.retrieve_device(keys)
torch.cuda.synchronize()
print("ok", bool((f == 1).all().item()), bool((v == vals).all().item()))
