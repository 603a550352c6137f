"""One multi-value insert + retrieve at 2^24 pairs, r = 1 (the reference CLI's multi-sweep point),
for an ncu launch list."""
import math, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2009_07914_b200 import MultiValueHashTable
from paper_2009_07914_b200.workloads import WorkloadSpec, gen_multiplicity

r = int(sys.argv[1]) if len(sys.argv) > 1 else 1
n = 1 << 24
keys = gen_multiplicity(WorkloadSpec(n=n, r=r, seed=42))
k = torch.from_numpy(keys.astype(np.uint32).view(np.int32)).cuda()
v = torch.arange(1, n + 1, dtype=torch.int32, device="cuda")
q = torch.arange(1, n + 1, dtype=torch.int32, device="cuda")
for rep in range(2):
    t = MultiValueHashTable(math.ceil(n / 0.8), layout="packed", key_bits=32, value_bits=32, group_width=8)
    torch.cuda.synchronize()
    e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    e[0].record()
    t.insert_device(k, v)
    e[1].record()
    off, flat = t.retrieve_device(q)
    e[2].record()
    torch.cuda.synchronize()
    print(f"r={r} rep={rep} insert {e[0].elapsed_time(e[1]):.3f} ms retrieve {e[1].elapsed_time(e[2]):.3f} ms")
    del t, off, flat
