"""Bucket-list hash table on B200 (mirrors coophash.bucket_list).

Keys live once in a device key store whose value cells hold 64-bit list
handles (state:2 | count:20 | tail:42, bucket_list.py:37-70); values live in
a device arena of growing buckets (s_i = ceil(lambda s_{i-1}), exact rational
lambda, :73-126).  A bulk insert moves each key's handle once per batch
(csrc/bucket.cu); counting reads handles only; retrieval walks the chains.

  insert / insert_bulk        ch_bucket_insert   (:228-294, :367-378)
  count / count_bulk          ch_bucket_count    (:320-326, :380-381)
  retrieve / retrieve_bulk    ch_bucket_count + ch_bucket_retrieve (:300-355, :383-397)
"""
from __future__ import annotations

import threading
from bisect import bisect_left
from enum import IntEnum
from fractions import Fraction
from math import ceil
from typing import Callable, Iterable, Sequence

import numpy as np
import torch

from . import _io, _lib
from .layout import LayoutKind, Sentinels, as_layout
from .probing import CapacityPlan, ProbingScheme
from .single_table import (InsertStatus, ProbeStats, _TableBase, statuses_from_codes)

COUNT_BITS = 20
TAIL_BITS = 42
COUNT_MAX = (1 << COUNT_BITS) - 1
TAIL_MAX = (1 << TAIL_BITS) - 1
BACKOFF_CAP = 1024
RETRY_BUDGET = 10 ** 6


class PoolExhausted(Exception):
    """The bucket arena has no room for the requested allocation."""


class ContentionTimeout(Exception):
    """A handle stayed blocked or contended past the retry budget."""


class HandleState(IntEnum):
    UNINITIALIZED = 0
    BLOCKED = 1
    READY = 2
    FULL = 3


def pack_handle(state: int, count: int, tail: int) -> int:
    if not 0 <= count <= COUNT_MAX:
        raise ValueError("handle count out of range")
    if not 0 <= tail <= TAIL_MAX:
        raise ValueError("handle tail reference out of range")
    return (state << (COUNT_BITS + TAIL_BITS)) | (count << TAIL_BITS) | tail


def unpack_handle(word: int) -> tuple[int, int, int]:
    return word >> (COUNT_BITS + TAIL_BITS), (word >> TAIL_BITS) & COUNT_MAX, word & TAIL_MAX


class GrowthPolicy:
    """Bucket sizes s_i = ceil(lambda * s_(i-1)) with lambda an exact Fraction."""

    def __init__(self, initial_size: int = 1, factor: float | str | Fraction = "1.1"):
        if initial_size < 1:
            raise ValueError("initial bucket size must be >= 1")
        factor = factor if isinstance(factor, Fraction) else Fraction(str(factor))
        if factor < 1:
            raise ValueError("growth factor must be >= 1")
        self.initial_size = initial_size
        self.factor = factor
        self._sizes = [initial_size]
        self._sums = [initial_size]
        self._lock = threading.Lock()

    def _grow_to(self, m: int) -> None:
        if len(self._sizes) >= m:
            return
        with self._lock:
            while len(self._sizes) < m:
                s = ceil(self.factor * self._sizes[-1])
                self._sizes.append(s)
                self._sums.append(self._sums[-1] + s)

    def bucket_size(self, i: int) -> int:
        self._grow_to(i + 1)
        return self._sizes[i]

    def capacity_of(self, m: int) -> int:
        if m == 0:
            return 0
        self._grow_to(m)
        return self._sums[m - 1]

    def buckets_for(self, count: int) -> int:
        if count <= 0:
            return 0
        while self._sums[-1] < count:
            self._grow_to(len(self._sizes) + 8)
        return bisect_left(self._sums, count) + 1


def next_bucket_size(policy: GrowthPolicy, previous: int) -> int:
    if previous < 1:
        raise ValueError("previous bucket size must be >= 1")
    return ceil(policy.factor * previous)


class BucketPool:
    """Bump arena.  Standalone pools are host bookkeeping; a table's pool is a
    view of its device arena (``allocated`` and ``arena`` read back from HBM)."""

    def __init__(self, capacity: int, _table=None):
        if capacity <= 0:
            raise ValueError("pool capacity must be positive")
        self.capacity = capacity
        self._table = _table
        self._bump = 0
        self._lock = threading.Lock()

    def alloc(self, slots: int) -> int:
        if self._table is not None:
            raise RuntimeError("a table's pool is allocated on the device")
        if slots < 1:
            raise ValueError("allocation must cover at least one slot")
        with self._lock:
            if self._bump + slots > self.capacity:
                raise PoolExhausted(f"need {slots} slots, {self.capacity - self._bump} left")
            off = self._bump
            self._bump += slots
            return off

    @property
    def allocated(self) -> int:
        if self._table is not None:
            return int(self._table._dt.stats().pool_allocated)
        return self._bump

    @property
    def arena(self) -> list[int]:
        if self._table is None:
            return [0] * self.capacity
        t = self._table
        out = np.empty(self.capacity, dtype=_io.np_dtype(t.value_bits))
        _lib.check(_lib.lib().ch_read_arena(t._dt.handle, out.ctypes.data, self.capacity), "read arena")
        return out.tolist()


class _KeyStore(_TableBase):
    """The bucket table's key store seen as a SingleValueHashTable (value cells = handles)."""

    def __init__(self, owner: "BucketListHashTable"):
        self.__dict__.update({k: owner.__dict__[k] for k in
                              ("config", "_dt", "layout", "workers", "device", "_packed", "slots",
                               "sentinels", "key_bits")})
        self.value_bits = 64

    @property
    def tombstones(self) -> int:
        return int(self._dt.stats().tombstones)

    def slot_of(self, key: int) -> int:
        if self._is_sentinel(key):
            return -1
        k = self._keys([key])
        slots = torch.empty(1, dtype=torch.int64, device=f"cuda:{self.device}")
        _lib.check(_lib.lib().ch_find(self._dt.handle, k.data_ptr(), 1, slots.data_ptr(), None, None, None,
                                      self._stream()), "find")
        return int(slots.item())

    def retrieve_with_stats(self, key: int):
        if self._is_sentinel(key):
            return None, ProbeStats(0, 0)
        k = self._keys([key])
        dev = f"cuda:{self.device}"
        slots = torch.empty(1, dtype=torch.int64, device=dev)
        att = torch.empty(1, dtype=torch.int32, device=dev)
        win = torch.empty(1, dtype=torch.int32, device=dev)
        vals = torch.empty(1, dtype=torch.int64, device=dev)
        _lib.check(_lib.lib().ch_find(self._dt.handle, k.data_ptr(), 1, slots.data_ptr(), att.data_ptr(),
                                      win.data_ptr(), vals.data_ptr(), self._stream()), "find")
        stats = ProbeStats(int(att.item()), int(win.item()))
        if int(slots.item()) < 0:
            return None, stats
        return int(_io.from_device(vals, 64)[0]), stats

    def retrieve(self, key: int):
        return self.retrieve_with_stats(key)[0]


class BucketListHashTable(_TableBase):
    """Multi-value table that stores each key once and chains its values (HBM-resident)."""

    _kind = _lib.CH_BUCKET

    def __init__(self, min_keys: int, pool_capacity: int, *, growth: GrowthPolicy | None = None,
                 layout: LayoutKind | str = LayoutKind.SOA, key_bits: int = 64, value_bits: int = 64,
                 sentinels: Sentinels | None = None, group_width: int = 32, workers: int = 1,
                 plan: CapacityPlan | None = None, device=None):
        layout = as_layout(layout)
        if layout == LayoutKind.PACKED_AOS:
            raise ValueError("list handles need 64-bit value cells; use the soa or aos layout")
        if pool_capacity <= 0:
            raise ValueError("pool capacity must be positive")
        self.growth = growth if growth is not None else GrowthPolicy()
        f = self.growth.factor
        self._setup(min_keys, layout=layout, key_bits=key_bits, value_bits=value_bits,
                    sentinels=sentinels, group_width=group_width, scheme=ProbingScheme.COOPERATIVE,
                    max_outer_attempts=None, workers=workers, plan=plan, device=device,
                    pool_capacity=pool_capacity,
                    growth=(self.growth.initial_size, f.numerator, f.denominator), handle_bits=64)
        self.pool = BucketPool(pool_capacity, _table=self)
        self.key_store = _KeyStore(self)

    # -- introspection (bucket_list.py:190-215) ---------------------------------
    @property
    def occupied_keys(self) -> int:
        return self.occupied

    @property
    def total_values(self) -> int:
        return int(self._dt.stats().total_values)

    def key_load_factor(self) -> float:
        return self.load_factor()

    def storage_density(self) -> float:
        s = self._dt.stats()
        kb = self.key_bits
        stored = s.occupied * kb + s.total_values * self.value_bits
        allocated = self.capacity * kb + self.capacity * 64 + self.pool.capacity * self.value_bits
        return stored / allocated

    # -- device-native API ---------------------------------------------------------
    def insert_device(self, keys, values, stream=None) -> torch.Tensor:
        k, v = self._keys(keys), self._vals(values)
        if k.numel() != v.numel():
            raise ValueError("keys and values differ in length")
        n = k.numel()
        st = self._u8(n)
        if n:
            _lib.check(_lib.lib().ch_bucket_insert(self._dt.handle, k.data_ptr(), v.data_ptr(), n,
                                                   st.data_ptr(), self._stream(stream)), "bucket insert")
            self._dt.touch()
        return st

    def count_device(self, keys, stream=None):
        """(counts int32, offsets int64[n+1], handles int64) -- handles feed retrieve_device."""
        k = self._keys(keys)
        n = k.numel()
        dev = f"cuda:{self.device}"
        counts = torch.empty(n, dtype=torch.int32, device=dev)
        offsets = torch.empty(n + 1, dtype=torch.int64, device=dev)
        handles = torch.empty(n, dtype=torch.int64, device=dev)
        _lib.check(_lib.lib().ch_bucket_count(self._dt.handle, k.data_ptr(), n, counts.data_ptr(),
                                              offsets.data_ptr(), handles.data_ptr(), self._stream(stream)),
                   "bucket count")
        return counts, offsets, handles

    def retrieve_device(self, keys, stream=None):
        k = self._keys(keys)
        n = k.numel()
        _, offsets, handles = self.count_device(k, stream)
        total = int(offsets[n].item()) if n else 0
        vals = torch.zeros(total, dtype=_io.torch_dtype(self.value_bits), device=f"cuda:{self.device}")
        if total:
            _lib.check(_lib.lib().ch_bucket_retrieve(self._dt.handle, handles.data_ptr(), n, offsets.data_ptr(),
                                                     vals.data_ptr(), self._stream(stream)), "bucket retrieve")
        return offsets, vals

    # -- element operations ------------------------------------------------------------
    def insert(self, key: int, value: int) -> InsertStatus:
        return self.insert_bulk([(key, value)])[0]

    def count(self, key: int) -> int:
        return self.count_bulk([key])[0]

    def retrieve(self, key: int) -> list[int]:
        return self.retrieve_bulk([key])[1]

    def chain_sizes(self, key: int) -> list[int]:
        n = self.count(key)
        if n == 0:
            return []
        return [self.growth.bucket_size(b) for b in range(self.growth.buckets_for(n))]

    # -- bulk operations ------------------------------------------------------------------
    def insert_bulk(self, pairs: Sequence[tuple[int, int]], workers: int | None = None) -> list[InsertStatus]:
        keys, vals = _io.split_pairs(pairs)
        if not keys:
            return []
        st = self.insert_device(keys, vals)
        return statuses_from_codes(st.cpu().numpy())

    def count_bulk(self, keys: Sequence[int]) -> list[int]:
        keys = list(keys)
        if not keys:
            return []
        counts, _, _ = self.count_device(keys)
        return counts.cpu().numpy().astype(np.int64).tolist()

    def retrieve_bulk(self, keys: Sequence[int]) -> tuple[list[int], list[int]]:
        keys = list(keys)
        if not keys:
            return [0], []
        offsets, vals = self.retrieve_device(keys)
        self._dt.stats()  # raises ContentionTimeout if a walk met a handle left BLOCKED (:300-318)
        return offsets.cpu().numpy().tolist(), _io.from_device(vals, self.value_bits).tolist()

    def for_each(self, keys: Iterable[int], callback: Callable[[int, int, int], None]) -> None:
        keys = list(keys)
        if not keys:
            return
        offsets, flat = self.retrieve_bulk(keys)
        for i, k in enumerate(keys):
            seg = flat[offsets[i]:offsets[i + 1]]
            if not seg:
                continue
            slot = self.key_store.slot_of(k)
            for v in seg:
                callback(k, v, slot)
