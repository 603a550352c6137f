"""Other single-value operations at the headline size (2^28 packed 32|32, load 0.95, g = 8):
retrieve with 0 / 50 / 100 % absent keys and bulk erase, device time (CUDA events), each
verified.  Prints one JSON line per operation.

  python tools/ops_2p28.py [--n 2^28] [--load 0.95] [--reps 3]
"""
import argparse
import json
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2009_07914_b200 import SingleValueHashTable
from paper_2009_07914_b200.workloads import unique_keys_device


def timed(fn):
    s = torch.cuda.current_stream()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    a.record(s)
    out = fn()
    b.record(s)
    torch.cuda.synchronize()
    return a.elapsed_time(b), out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=1 << 28)
    ap.add_argument("--load", type=float, default=0.95)
    ap.add_argument("--reps", type=int, default=3)
    a = ap.parse_args()
    dev = torch.device("cuda", 0)
    n = a.n
    keys = unique_keys_device(0, n, 2 * n, dev)
    absent = unique_keys_device(n, n, 2 * n + 16, dev)
    vals = keys.clone()
    half = torch.cat([keys[: n // 2], absent[: n - n // 2]])
    half = half[torch.randperm(n, device=dev)]
    t = SingleValueHashTable(math.ceil(n / a.load), layout="packed", key_bits=32, value_bits=32, group_width=8,
                             device=0)
    t.insert_device(keys, vals)
    torch.cuda.synchronize()
    for name, q, hits in (("retrieve_hits", keys, n), ("retrieve_50pct_absent", half, n // 2),
                          ("retrieve_absent", absent, 0)):
        ms = []
        for r in range(a.reps + 1):
            t.reset_probe_counters()
            dt, (v, f) = timed(lambda: t.retrieve_device(q))
            if r:
                ms.append(dt)
        c = t.probe_counters()
        ok = int(f.sum().item()) == hits
        print(json.dumps({"op": name, "n": n, "load": a.load, "ms": sum(ms) / len(ms),
                          "gops": n / (sum(ms) / len(ms)) / 1e6, "mean_attempts": c.attempts / max(1, c.ops),
                          "schedule": t.batch_schedule(n), "verified": ok}), flush=True)
    ms = []
    for r in range(a.reps):
        t2 = SingleValueHashTable(math.ceil(n / a.load), layout="packed", key_bits=32, value_bits=32,
                                  group_width=8, device=0)
        t2.insert_device(keys, vals)
        dt, er = timed(lambda: t2.erase_device(keys))
        ok = bool(er.bool().all()) and t2.occupied == 0 and t2.tombstones == n
        ms.append(dt)
        del t2
        torch.cuda.empty_cache()
    print(json.dumps({"op": "erase", "n": n, "load": a.load, "ms": sum(ms) / len(ms),
                      "gops": n / (sum(ms) / len(ms)) / 1e6, "verified": ok}), flush=True)


if __name__ == "__main__":
    main()
