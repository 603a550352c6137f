import math, sys, torch
sys.path[:0] = ["."]
from bench import make_keys
from paper_2009_07914_b200 import SingleValueHashTable, _lib
n = 1 << 28
keys, vals = make_keys(0, n, 1, torch.device("cuda", 0))
t = SingleValueHashTable(math.ceil(n / 0.95), layout="packed", key_bits=32, value_bits=32, group_width=8)
t.set_locality("staged")
t.reset_probe_counters()
st = t.insert_device(keys, vals); torch.cuda.synchronize()
print("insert deferred", t.deferred_count(), t.deferred_count() / n, "occupied", t.occupied)
t.reset_probe_counters()
v, f = t.retrieve_device(keys); torch.cuda.synchronize()
print("lookup deferred", t.deferred_count(), t.deferred_count() / n, bool(f.all()))
