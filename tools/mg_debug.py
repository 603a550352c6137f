import sys; sys.path.insert(0, "/root/repo")
import numpy as np, torch
from paper_2009_07914_b200 import MultiValueHashTable
for layout, r, g in (("packed", 256, 8), ("aos", 256, 32), ("soa", 256, 8), ("packed", 64, 8)):
    n = 1 << 17
    rng = np.random.default_rng(r * 31 + g)
    keys = rng.integers(1, n // r + 1, size=n, dtype=np.uint64)
    vals = np.arange(1, n + 1, dtype=np.uint64)
    t = MultiValueHashTable(int(np.ceil(n / 0.8)), layout=layout, key_bits=32, value_bits=32 if layout == "packed" else 64, group_width=g)
    st = t.insert_device(keys, vals).cpu().numpy()
    q = np.arange(1, n // r + 1, dtype=np.uint64)
    cnt, off = t.count_device(q)
    cnt = cnt.cpu().numpy()
    true = np.bincount(keys.astype(np.int64), minlength=n // r + 1)[1:]
    bad = np.nonzero(cnt != true)[0]
    print(layout, r, "status ok", (st == 0).all(), "occupied", t.occupied, "bad", len(bad), (cnt[bad][:5], true[bad][:5]))
