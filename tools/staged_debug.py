"""Debug: replay golden single-table scenario steps on the staged path and report
status mismatches against the reference statuses, with table copies of each key."""
import sys
from collections import Counter
sys.path[:0] = ["tests", "."]
import numpy as np
from gold import load, ints
from paper_2009_07914_b200 import SingleValueHashTable, Sentinels, InsertStatus

for idx in [int(a) for a in sys.argv[1:]] or range(11):
    sc = load("single.json")["scenarios"][idx]
    for trial in range(5):
        t = SingleValueHashTable(sc["min_capacity"], layout=sc["layout"], key_bits=sc["key_bits"],
                                 value_bits=32 if sc["layout"] == "packed" else 64, group_width=sc["group_width"],
                                 max_outer_attempts=sc["max_outer_attempts"],
                                 sentinels=Sentinels(int(sc["empty"]), int(sc["tomb"])))
        t.set_locality("staged")
        st = sc["steps"][0]
        keys, vals = ints(st["keys"]), ints(st["vals"])
        got = t.insert_bulk(list(zip(keys, vals)))
        mult = Counter(keys)
        tk = Counter(t.slots.load_key(i) for i in range(t.capacity))
        bad = [(i, k, g.value, r, tk[k]) for i, (k, g, r) in enumerate(zip(keys, got, st["status"]))
               if mult[k] == 1 and g.value != r]
        dup_tab = [k for k, c in tk.items() if c > 1 and k not in (int(sc["empty"]), int(sc["tomb"]))]
        print(idx, sc["name"], "trial", trial, "bad", len(bad), bad[:5], "table dups", dup_tab[:5],
              "deferred", t.deferred_count())
