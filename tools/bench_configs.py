"""BASELINE configs[2] and configs[3]: multi-value (Zipf) and bucket-list (power law), 2^27 pairs.

  python tools/bench_configs.py [--n 2^27] [--which multi,bucket] [--reps 3]
Prints one JSON line per workload: insert / count+retrieve G ops/s, verified against a
device-side multiset check (sorted per-key values vs the inserted pairs).
"""
import argparse
import json
import math
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2009_07914_b200 import BucketListHashTable, GrowthPolicy, MultiValueHashTable


def fmix32(x):
    x = x & 0xFFFFFFFF
    x = x ^ (x >> 16)
    x = (x * 0x85EBCA6B) & 0xFFFFFFFF
    x = x ^ (x >> 13)
    x = (x * 0xC2B2AE35) & 0xFFFFFFFF
    return x ^ (x >> 16)


def zipf_keys(n, universe, s, seed, dev):
    g = torch.Generator(device=dev).manual_seed(seed)
    ranks = torch.arange(1, universe + 1, device=dev, dtype=torch.float64)
    cdf = torch.cumsum(ranks ** (-s), 0)
    cdf /= cdf[-1].clone()
    u = torch.rand(n, generator=g, device=dev, dtype=torch.float64)
    r = torch.searchsorted(cdf, u).clamp_(max=universe - 1) + 1     # rank in [1, universe]
    return fmix32(r.to(torch.int64)), r


def power_law_keys(n, seed, dev, mmax=1000, alpha=1.5):
    rng = np.random.default_rng(seed)
    m = np.arange(1, mmax + 1)
    p = m ** -alpha
    p /= p.sum()
    mult = []
    total = 0
    while total < n:
        draw = rng.choice(m, size=1 << 20, p=p)
        mult.append(draw)
        total += int(draw.sum())
    mult = np.concatenate(mult)
    cs = np.cumsum(mult)
    k = int(np.searchsorted(cs, n)) + 1
    mult = mult[:k]
    mult[-1] -= int(cs[k - 1] - n)
    keys = np.repeat(np.arange(1, k + 1, dtype=np.int64), mult)
    keys = torch.from_numpy(rng.permutation(keys)).to(dev)
    return fmix32(keys), k


def check_multiset(keys, vals, offsets, flat, queries):
    """Per-query sorted value multisets equal those of the inserted pairs (device-side)."""
    order = torch.argsort(keys * (1 << 32) + vals)
    ks, vs = keys[order], vals[order]
    qo = torch.argsort(queries)
    counts = offsets[1:] - offsets[:-1]
    seg = torch.repeat_interleave(torch.arange(len(queries), device=keys.device), counts)
    fq = queries[seg]
    o2 = torch.argsort(fq * (1 << 32) + flat.to(torch.int64) % (1 << 32))
    return bool(torch.equal(fq[o2], ks) and torch.equal(flat.to(torch.int64)[o2] % (1 << 32), vs))


def timed(f):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    r = f()
    torch.cuda.synchronize()
    return time.perf_counter() - t0, r


def run_multi(n, dev, reps, s):
    keys, _ = zipf_keys(n, 1 << 23, s, 42, dev)
    vals = torch.arange(1, n + 1, device=dev, dtype=torch.int64)
    k32 = keys.to(torch.int32)
    v32 = vals.to(torch.int32)
    queries = torch.unique(keys)
    q32 = queries.to(torch.int32)
    ins, ret = [], []
    for r in range(reps + 1):
        t = MultiValueHashTable(math.ceil(n / 0.8), layout="packed", key_bits=32, value_bits=32, group_width=8,
                                device=dev.index)
        ti, st = timed(lambda: t.insert_device(k32, v32))
        tr, (off, flat) = timed(lambda: t.retrieve_device(q32))
        if r:
            ins.append(ti)
            ret.append(tr)
        del t
    ok = bool((st == 0).all()) and int(off[-1]) == n and check_multiset(
        keys, vals, off, flat.to(torch.int64) & 0xFFFFFFFF, queries)
    return {"workload": f"MultiValueHashTable packed, 2^{int(math.log2(n))} pairs, Zipf s={s} over 2^23 ranks, load 0.8",
            "insert_gops": n / np.mean(ins) / 1e9, "retrieve_gops": n / np.mean(ret) / 1e9,
            "insert_ms": 1e3 * np.mean(ins), "count_retrieve_ms": 1e3 * np.mean(ret),
            "distinct": len(queries), "verified": ok}


def run_bucket(n, dev, reps, policy):
    keys, distinct = power_law_keys(n, 7, dev)
    vals = torch.arange(1, n + 1, device=dev, dtype=torch.int64)
    queries = torch.unique(keys)
    s0, lam = policy
    ins, ret = [], []
    for r in range(reps + 1):
        t = BucketListHashTable(math.ceil(distinct / 0.8), int(n * 2.5) + 64, growth=GrowthPolicy(s0, lam),
                                key_bits=32, value_bits=64, device=dev.index)
        ti, st = timed(lambda: t.insert_device(keys.to(torch.int32), vals))
        tr, (off, flat) = timed(lambda: t.retrieve_device(queries.to(torch.int32)))
        if r:
            ins.append(ti)
            ret.append(tr)
        density = t.storage_density()
        del t
    ok = bool((st == 0).all()) and int(off[-1]) == n and check_multiset(keys, vals, off, flat, queries)
    return {"workload": f"BucketListHashTable soa, 2^{int(math.log2(n))} pairs, power-law multiplicity 1..1000 "
                        f"(alpha 1.5), growth (s0={s0}, lambda={lam})",
            "insert_gops": n / np.mean(ins) / 1e9, "retrieve_gops": n / np.mean(ret) / 1e9,
            "insert_ms": 1e3 * np.mean(ins), "count_retrieve_ms": 1e3 * np.mean(ret),
            "distinct": distinct, "storage_density": density, "verified": ok}


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=1 << 27)
    ap.add_argument("--which", default="multi,bucket")
    ap.add_argument("--reps", type=int, default=2)
    ap.add_argument("--zipf", type=float, default=0.5)
    a = ap.parse_args()
    dev = torch.device("cuda", 0)
    for w in a.which.split(","):
        if w == "multi":
            print(json.dumps(run_multi(a.n, dev, a.reps, a.zipf)), flush=True)
        elif w == "bucket":
            for pol in ((1, "1.1"), (24, "1.0")):
                print(json.dumps(run_bucket(a.n, dev, a.reps, pol)), flush=True)
