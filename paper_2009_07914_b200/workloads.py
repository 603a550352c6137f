"""Synthetic workloads of the reference benchmark (coophash/bench.py:41-84) and of the
BASELINE configurations, as numpy (reference-compatible) or CUDA tensors (full size).

  gen_unique / gen_multiplicity    bench.py:58-84, same RNG calls as the reference, so the
                                   same seed gives the same keys (numpy Generator)
  unique_keys_device               n distinct 32-bit keys as a bijection of an index range
                                   (fmix32), sentinel images replaced (configs[1], [4])
  zipf_keys_device                 bounded Zipf ranks over a universe (configs[2])
  power_law_keys                   per-key multiplicity P(m) ~ m^-alpha on [1, 1000] (configs[3])
  multiset_equal                   per-query sorted value multisets vs the inserted pairs
                                   (the reference's _verify_multi, bench.py:201-220, on device)
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch


@dataclass(frozen=True)
class WorkloadSpec:
    """bench.py:41-55 (validation and messages kept)."""
    n: int
    r: int = 1
    key_bits: int = 32
    seed: int = 42
    target_density: float = 0.8

    def __post_init__(self) -> None:
        if self.n < 1:
            raise ValueError("n must be positive")
        if not 1 <= self.r <= self.n:
            raise ValueError("multiplicity r must satisfy 1 <= r <= n")
        if self.key_bits not in (32, 64):
            raise ValueError("key_bits must be 32 or 64")
        if not 0 < self.target_density < 1:
            raise ValueError("target density must lie in (0, 1)")


def gen_unique(spec: WorkloadSpec) -> np.ndarray:
    """n pairwise-distinct non-sentinel keys (bench.py:58-71): uniform on [1, 2^kb - 3]."""
    rng = np.random.default_rng(spec.seed)
    high = (1 << spec.key_bits) - 2
    if spec.n > high - 1:
        raise ValueError("key space too small for n unique keys")
    acc = np.empty(0, dtype=np.uint64)
    while len(acc) < spec.n:
        need = spec.n - len(acc)
        draw = rng.integers(1, high, size=need + need // 8 + 16, dtype=np.uint64)
        acc = np.unique(np.concatenate([acc, draw]))
    return rng.permutation(acc)[:spec.n]


def gen_multiplicity(spec: WorkloadSpec) -> np.ndarray:
    """n keys with mean multiplicity r drawn uniformly from [1, n // r] (bench.py:74-84);
    r = 1 is a permutation of 1..n."""
    rng = np.random.default_rng(spec.seed)
    if spec.r == 1:
        return rng.permutation(np.arange(1, spec.n + 1, dtype=np.uint64))
    return rng.integers(1, spec.n // spec.r + 1, size=spec.n, dtype=np.uint64)


# ------------------------------------------------------------------ device-scale generators

def fmix32(x: torch.Tensor) -> torch.Tensor:
    """murmur3 finalizer on int64 tensors holding 32-bit values (a bijection of [0, 2^32))."""
    x = x & 0xFFFFFFFF
    x = x ^ (x >> 16)
    x = (x * 0x85EBCA6B) & 0xFFFFFFFF
    x = x ^ (x >> 13)
    x = (x * 0xC2B2AE35) & 0xFFFFFFFF
    return x ^ (x >> 16)


def _inv_xorshift(y: int, s: int) -> int:
    x = y
    for _ in range(32 // s + 1):
        x = y ^ (x >> s)
    return x & 0xFFFFFFFF


def fmix32_inverse(y: int) -> int:
    y = _inv_xorshift(y, 16)
    y = (y * pow(0xC2B2AE35, -1, 1 << 32)) & 0xFFFFFFFF
    y = _inv_xorshift(y, 13)
    y = (y * pow(0x85EBCA6B, -1, 1 << 32)) & 0xFFFFFFFF
    return _inv_xorshift(y, 16)


def fmix32_host(x: int) -> int:
    return int(fmix32(torch.tensor([x], dtype=torch.int64))[0])


def unique_keys_device(start: int, n: int, total: int, device) -> torch.Tensor:
    """fmix32 of the indices [start, start + n) as int32 bit patterns: pairwise distinct
    across any disjoint index ranges; the two sentinel images (0xFFFFFFFF, 0xFFFFFFFE)
    are replaced by images of indices >= total."""
    idx = torch.arange(start, start + n, dtype=torch.int64, device=device)
    x = fmix32(idx)
    spare = total
    for sentinel in (0xFFFFFFFF, 0xFFFFFFFE):
        pre = fmix32_inverse(sentinel)
        if start <= pre < start + n:
            while fmix32_host(spare) in (0xFFFFFFFF, 0xFFFFFFFE):
                spare += 1
            x[pre - start] = fmix32_host(spare)
            spare += 1
    return x.to(torch.int32)


def zipf_keys_device(n: int, universe: int, s: float, seed: int, device):
    """n bounded-Zipf ranks on [1, universe] (P(r) ~ r^-s), mapped through fmix32.
    Returns (keys int64 holding u32 values, ranks)."""
    g = torch.Generator(device=device).manual_seed(seed)
    ranks = torch.arange(1, universe + 1, device=device, dtype=torch.float64)
    cdf = torch.cumsum(ranks ** (-s), 0)
    cdf /= cdf[-1].clone()
    u = torch.rand(n, generator=g, device=device, dtype=torch.float64)
    r = torch.searchsorted(cdf, u).clamp_(max=universe - 1) + 1
    return fmix32(r.to(torch.int64)), r


def power_law_keys(n: int, seed: int, device, mmax: int = 1000, alpha: float = 1.5):
    """Keys whose multiplicities follow P(m) ~ m^-alpha on [1, mmax], n pairs in total,
    shuffled.  Returns (keys int64 holding u32 values, distinct key count)."""
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
    keys = torch.from_numpy(rng.permutation(keys)).to(device)
    return fmix32(keys), k


def multiset_equal(keys: torch.Tensor, vals: torch.Tensor, offsets: torch.Tensor, flat: torch.Tensor,
                   queries: torch.Tensor) -> bool:
    """Per-query sorted value multisets equal those of the inserted (key, value) pairs
    (all int64 tensors holding u32 values; every inserted key is queried once)."""
    order = torch.argsort(keys * (1 << 32) + vals)
    ks, vs = keys[order], vals[order]
    counts = offsets[1:] - offsets[:-1]
    seg = torch.repeat_interleave(torch.arange(len(queries), device=keys.device), counts)
    fq = queries[seg]
    fl = flat.to(torch.int64) & 0xFFFFFFFF
    o2 = torch.argsort(fq * (1 << 32) + fl)
    return bool(torch.equal(fq[o2], ks) and torch.equal(fl[o2], vs))
