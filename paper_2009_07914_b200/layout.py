"""Slot layouts, sentinels and the device-resident slot array.

Mirrors coophash.layout (reference pkg/src/coophash/layout.py).  The cells
live in HBM, owned by a ch_table (csrc/api.cu); element transitions are
single-thread CUDA kernels with real 32/64-bit atomicCAS (csrc/api.cu
k_slot_op), replacing the reference's striped Python locks (layout.py:22,105).
Reads of whole windows / items are served from a host copy of the device
arrays that is refreshed whenever the table changed.

  LayoutKind, Sentinels, default_sentinels   layout.py:29-53
  pack_pair / unpack_pair                    layout.py:56-66 (value << 32 | key)
  SlotArray                                  layout.py:69-265
"""
from __future__ import annotations

import ctypes as C
import threading
from dataclasses import dataclass
from enum import Enum
from typing import Iterator

import numpy as np

from . import _lib

MASK32 = (1 << 32) - 1


class LayoutUnsupported(Exception):
    """Operation or configuration not available for this layout."""


class LayoutKind(Enum):
    SOA = "soa"
    AOS = "aos"
    PACKED_AOS = "packed"


_LAYOUT_CODE = {LayoutKind.SOA: _lib.CH_SOA, LayoutKind.AOS: _lib.CH_AOS,
                LayoutKind.PACKED_AOS: _lib.CH_PACKED}


def as_layout(layout) -> LayoutKind:
    return LayoutKind(layout) if isinstance(layout, str) else layout


@dataclass(frozen=True)
class Sentinels:
    empty_key: int
    tombstone_key: int

    def __post_init__(self) -> None:
        if self.empty_key == self.tombstone_key:
            raise ValueError("empty and tombstone sentinels must differ")
        if self.empty_key < 0 or self.tombstone_key < 0:
            raise ValueError("sentinels must be non-negative")

    def is_sentinel(self, key: int) -> bool:
        return key == self.empty_key or key == self.tombstone_key


def default_sentinels(key_bits: int = 64) -> Sentinels:
    top = (1 << key_bits) - 1
    return Sentinels(empty_key=top, tombstone_key=top - 1)


def pack_pair(key: int, value: int) -> int:
    if not 0 <= key <= MASK32:
        raise ValueError("packed key must fit in 32 bits")
    if not 0 <= value <= MASK32:
        raise ValueError("packed value must fit in 32 bits")
    return (value << 32) | key


def unpack_pair(word: int) -> tuple[int, int]:
    return word & MASK32, word >> 32


def storage_dtype(bits: int):
    return np.uint32 if bits <= 32 else np.uint64


class DeviceTable:
    """Lifetime of one ch_table (device slots, counters, optional bucket arena)."""

    def __init__(self, *, kind: int, layout: LayoutKind, key_bits: int, value_bits: int,
                 group_width: int, p: int, max_outer_attempts: int | None,
                 sentinels: Sentinels, device=None, pool_capacity: int = 0,
                 growth: tuple[int, int, int] = (0, 0, 0)):
        self.device = _lib.require_cuda(device)
        cfg = _lib.ch_config()
        cfg.kind = kind
        cfg.layout = _LAYOUT_CODE[layout]
        cfg.key_bits = key_bits
        cfg.value_bits = value_bits
        cfg.group_width = group_width
        cfg.p = p
        cfg.max_outer_attempts = max_outer_attempts or 0
        cfg.empty_key = sentinels.empty_key
        cfg.tombstone_key = sentinels.tombstone_key
        cfg.pool_capacity = pool_capacity
        cfg.growth_s0, cfg.growth_num, cfg.growth_den = growth
        cfg.device = self.device
        h = C.c_void_p()
        _lib.check(_lib.lib().ch_create(C.byref(h), C.byref(cfg)), "ch_create")
        self.handle = h.value
        self.kind = kind
        self.layout = layout
        self.key_bits, self.value_bits = key_bits, value_bits
        self.capacity = 32 * p
        self.version = 0          # bumped on every mutation (host caches key off it)
        self._lock = threading.Lock()

    def __del__(self):
        h = getattr(self, "handle", None)
        if h and _lib._lib is not None:
            _lib._lib.ch_destroy(h)
            self.handle = None

    def touch(self) -> None:
        with self._lock:
            self.version += 1

    def stats(self) -> _lib.ch_stats:
        s = _lib.ch_stats()
        _lib.check(_lib.lib().ch_get_stats(self.handle, C.byref(s)), "ch_get_stats")
        if s.device_error & 1:
            from .bucket_list import ContentionTimeout
            raise ContentionTimeout("a bucket handle stayed blocked past the retry budget")
        if s.device_error:
            raise RuntimeError(f"device error bits {s.device_error:#x}: a list handle or bucket header "
                               "points outside the arena")
        return s

    def read_slots(self, value_bits: int | None = None) -> tuple[np.ndarray, np.ndarray]:
        kd = storage_dtype(self.key_bits)
        vd = storage_dtype(self.value_bits if value_bits is None else value_bits)
        keys = np.empty(self.capacity, dtype=kd)
        vals = np.empty(self.capacity, dtype=vd)
        _lib.check(_lib.lib().ch_read_slots(self.handle, keys.ctypes.data, vals.ctypes.data),
                   "ch_read_slots")
        return keys, vals

    def read_range(self, start: int, count: int, value_bits: int | None = None) -> tuple[np.ndarray, np.ndarray]:
        """Cells [start, start + count) only (no whole-table copy)."""
        kd = storage_dtype(self.key_bits)
        vd = storage_dtype(self.value_bits if value_bits is None else value_bits)
        keys = np.empty(count, dtype=kd)
        vals = np.empty(count, dtype=vd)
        _lib.check(_lib.lib().ch_read_slot_range(self.handle, start, count, keys.ctypes.data, vals.ctypes.data),
                   "ch_read_slot_range")
        return keys, vals

    def slot_op(self, op: int, slot: int, expected: int = 0, desired: int = 0,
                value: int = 0) -> tuple[bool, int, int]:
        won = C.c_int(0)
        k = C.c_uint64(0)
        v = C.c_uint64(0)
        _lib.check(_lib.lib().ch_slot_op(self.handle, op, slot, expected, desired, value,
                                         C.byref(won), C.byref(k), C.byref(v)), "ch_slot_op")
        if op in (0, 1, 2, 3, 4) and won.value:
            self.touch()
        return bool(won.value), int(k.value), int(v.value)


class SlotArray:
    """Fixed-capacity key/value cells in HBM with atomic transitions.

    Standalone arrays own a ch_table; ``table.slots`` returns one bound to the
    table's own cells (capacity = 32 p) so the reference's introspection
    (load_key / load_value / iter_items ...) sees the device state.
    """

    def __init__(self, capacity: int, layout: LayoutKind | str = LayoutKind.SOA,
                 sentinels: Sentinels | None = None, *, key_bits: int = 64,
                 value_bits: int = 64, device=None, _table: DeviceTable | None = None):
        layout = as_layout(layout)
        if capacity <= 0:
            raise ValueError("capacity must be positive")
        if layout == LayoutKind.PACKED_AOS and (key_bits > 32 or value_bits > 32):
            raise LayoutUnsupported("packed layout needs 32-bit keys and values")
        self.sentinels = sentinels if sentinels is not None else default_sentinels(key_bits)
        self.capacity = capacity
        self.layout = layout
        self.key_bits = key_bits
        self.value_bits = value_bits
        if _table is None:
            _table = DeviceTable(kind=_lib.CH_SINGLE, layout=layout, key_bits=key_bits,
                                 value_bits=value_bits, group_width=32,
                                 p=max(2, -(-capacity // 32)), max_outer_attempts=None,
                                 sentinels=self.sentinels, device=device)
        self._t = _table
        self._cache_version = -1
        self._keys = self._vals = None
        self._lock = threading.Lock()

    # -- host view of the device cells -----------------------------------
    def _host(self) -> tuple[np.ndarray, np.ndarray]:
        with self._lock:
            if self._cache_version != self._t.version:
                v = self._t.version
                keys, vals = self._t.read_slots(self.value_bits)
                self._keys, self._vals = keys[: self.capacity], vals[: self.capacity]
                self._cache_version = v
            return self._keys, self._vals

    def _cells(self, start: int, count: int) -> tuple[np.ndarray, np.ndarray]:
        """Cells [start, start + count) (count <= capacity, wrapping): served from the
        whole-array host copy when it is current, else read from the device alone --
        element reads of a 2 GiB table move bytes, not the table."""
        with self._lock:
            cached = self._cache_version == self._t.version
        if cached:
            idx = (np.arange(count, dtype=np.int64) + start) % self.capacity
            return self._keys[idx], self._vals[idx]
        first = min(count, self.capacity - start)
        k, v = self._t.read_range(start, first, self.value_bits)
        if first < count:
            k2, v2 = self._t.read_range(0, count - first, self.value_bits)
            k, v = np.concatenate([k, k2]), np.concatenate([v, v2])
        return k, v

    def _index(self, i: int) -> int:
        if not -self.capacity <= i < self.capacity:
            raise IndexError("slot index out of range")
        return i % self.capacity

    def load_window(self, start: int, width: int) -> list[int]:
        return self._cells(start % self.capacity, width)[0].tolist()

    def load_key(self, i: int) -> int:
        return int(self._cells(self._index(i), 1)[0][0])

    def load_value(self, i: int) -> int:
        return int(self._cells(self._index(i), 1)[1][0])

    def load_pair(self, i: int) -> tuple[int, int]:
        if self.layout == LayoutKind.PACKED_AOS:  # one atomic 64-bit read (layout.py:154-157)
            _, k, v = self._t.slot_op(5, i)
            return k, v
        k, v = self._cells(self._index(i), 1)
        return int(k[0]), int(v[0])

    def store_value(self, i: int, value: int) -> None:
        self._t.slot_op(4, i, value=value)

    # -- atomic transitions (layout.py:174-243) ----------------------------
    def try_claim_key(self, i: int, expected: int, desired: int) -> tuple[bool, int]:
        won, k, _ = self._t.slot_op(0, i, expected, desired)
        return won, k

    def try_claim_pair_packed(self, i: int, key: int, value: int) -> tuple[bool, int]:
        if self.layout != LayoutKind.PACKED_AOS:
            raise LayoutUnsupported("pair claim requires the packed layout")
        won, k, _ = self._t.slot_op(1, i, desired=key, value=value)
        return won, k

    def cas_value(self, i: int, expected: int, desired: int) -> tuple[bool, int]:
        if self.layout == LayoutKind.PACKED_AOS:
            raise LayoutUnsupported("value CAS is not available on packed cells")
        won, _, v = self._t.slot_op(2, i, expected, desired)
        return won, v

    def retire_key(self, i: int, expected: int, tombstone_value: int = 0) -> tuple[bool, int]:
        won, k, _ = self._t.slot_op(3, i, expected, value=tombstone_value)
        return won, k

    def iter_items(self) -> Iterator[tuple[int, int, int]]:
        keys, vals = self._host()
        e, t = self.sentinels.empty_key, self.sentinels.tombstone_key
        live = np.nonzero((keys != keys.dtype.type(e)) & (keys != keys.dtype.type(t)))[0]
        for i, k, v in zip(live.tolist(), keys[live].tolist(), vals[live].tolist()):
            yield i, k, v


def new_slot_array(capacity: int, layout: LayoutKind = LayoutKind.SOA,
                   sentinels: Sentinels | None = None, *, key_bits: int = 64,
                   value_bits: int = 64) -> SlotArray:
    return SlotArray(capacity, layout, sentinels, key_bits=key_bits, value_bits=value_bits)
