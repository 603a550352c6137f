"""ctypes front-end of liboracle.so (CPU restatement of coophash; TEST ONLY).

Each class mirrors the sequential (workers=1) behaviour of one reference
table; every method cites the reference lines it restates through oracle.c.
Arrays are numpy uint64 in, numpy out.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from fractions import Fraction

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liboracle.so")

STATUS_NAMES = ("inserted", "duplicate_key", "table_full", "invalid_key", "out_of_memory")


def build() -> str:
    src = os.path.join(_HERE, "oracle.c")
    if (not os.path.exists(_LIB_PATH)
            or os.path.getmtime(_LIB_PATH) < os.path.getmtime(src)):
        subprocess.check_call(["make", "-s", "-C", _HERE, "liboracle.so"])
    return _LIB_PATH


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = C.CDLL(build())
        u64, i64, p = C.c_uint64, C.c_int64, C.c_void_p
        sig = {
            "orc_mix64": (u64, [u64]),
            "orc_is_prime": (C.c_int, [u64]),
            "orc_choose_p": (u64, [u64]),
            "orc_dh_step": (u64, [u64, u64]),
            "orc_single_new": (p, [u64, u64, u64, u64, u64, u64, C.c_int]),
            "orc_single_free": (None, [p]),
            "orc_single_capacity": (u64, [p]),
            "orc_single_p": (u64, [p]),
            "orc_single_insert_bulk": (None, [p, p, p, u64, p, C.c_int]),
            "orc_single_retrieve_bulk": (None, [p, p, u64, p, p, C.c_int]),
            "orc_single_find": (i64, [p, u64, C.POINTER(u64), C.POINTER(u64)]),
            "orc_single_erase_bulk": (None, [p, p, u64, p]),
            "orc_single_stats": (None, [p, p]),
            "orc_single_dump": (None, [p, p, p]),
            "orc_multi_insert_bulk": (None, [p, p, p, u64, p]),
            "orc_multi_count_bulk": (None, [p, p, u64, p]),
            "orc_multi_retrieve_bulk": (None, [p, p, u64, p, p]),
            "orc_exclusive_prefix_sum": (None, [p, u64, p]),
            "orc_pack_handle": (u64, [u64, u64, u64]),
            "orc_bucket_new": (p, [u64, u64, u64, u64, u64, u64, u64, u64]),
            "orc_bucket_free": (None, [p]),
            "orc_bucket_keystore": (p, [p]),
            "orc_bucket_insert_bulk": (None, [p, p, p, u64, p]),
            "orc_bucket_count_bulk": (None, [p, p, u64, p]),
            "orc_bucket_retrieve_bulk": (None, [p, p, u64, p, p]),
            "orc_bucket_chain_sizes": (u64, [p, u64, p, u64]),
            "orc_bucket_stats": (None, [p, p]),
            "orc_bucket_dump_arena": (None, [p, p]),
            "orc_growth_sizes": (None, [u64, u64, u64, u64, p]),
            "orc_route": (C.c_uint32, [u64, C.c_uint32]),
            "orc_multi_split": (None, [p, u64, C.c_uint32, p, p]),
            "orc_mix64_array": (None, [p, u64, u64, p]),
        }
        for name, (res, args) in sig.items():
            fn = getattr(_lib, name)
            fn.restype = res
            fn.argtypes = args
    return _lib


def _u64(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.uint64))


def _ptr(a: np.ndarray) -> int:
    return a.ctypes.data


# ---------------------------------------------------------------- L0 helpers

def mix64(key: int) -> int:
    return int(lib().orc_mix64(key))


def mix64_array(keys, seed: int = 0) -> np.ndarray:
    k = _u64(keys)
    out = np.empty_like(k)
    lib().orc_mix64_array(_ptr(k), len(k), seed, _ptr(out))
    return out


def is_prime(n: int) -> bool:
    return bool(lib().orc_is_prime(n))


def choose_p(min_slots: int) -> int:
    return int(lib().orc_choose_p(min_slots))


def dh_step(key: int, p: int) -> int:
    return int(lib().orc_dh_step(key, p))


def route(key: int, shards: int) -> int:
    return int(lib().orc_route(key, shards))


def multi_split(keys, shards: int) -> tuple[np.ndarray, np.ndarray]:
    k = _u64(keys)
    perm = np.empty(len(k), dtype=np.uint64)
    offsets = np.empty(shards + 1, dtype=np.uint64)
    lib().orc_multi_split(_ptr(k), len(k), shards, _ptr(perm), _ptr(offsets))
    return perm, offsets


def exclusive_prefix_sum(counts) -> np.ndarray:
    c = _u64(counts)
    out = np.empty(len(c) + 1, dtype=np.uint64)
    lib().orc_exclusive_prefix_sum(_ptr(c), len(c), _ptr(out))
    return out


def growth_sizes(s0: int, factor, m: int) -> np.ndarray:
    f = Fraction(str(factor)) if not isinstance(factor, Fraction) else factor
    out = np.empty(m, dtype=np.uint64)
    lib().orc_growth_sizes(s0, f.numerator, f.denominator, m, _ptr(out))
    return out


def default_sentinels(key_bits: int) -> tuple[int, int]:
    top = (1 << key_bits) - 1
    return top, top - 1


# ------------------------------------------------------------- L1 tables

class OracleSingle:
    """Sequential SingleValueHashTable (single_table.py:88-429)."""

    def __init__(self, min_capacity: int, *, group_width: int = 32, key_bits: int = 64,
                 packed: bool = False, max_outer_attempts: int = 0, p: int = 0,
                 sentinels: tuple[int, int] | None = None, _handle=None):
        e, t = sentinels if sentinels else default_sentinels(key_bits)
        self.empty_key, self.tombstone_key = e, t
        self.group_width = group_width
        if _handle is not None:
            self._h, self._owned = _handle, False
        else:
            self._h = lib().orc_single_new(min_capacity, p, group_width,
                                           max_outer_attempts, e, t, int(packed))
            self._owned = True
        self.capacity = int(lib().orc_single_capacity(self._h))
        self.p = int(lib().orc_single_p(self._h))

    def __del__(self):
        if getattr(self, "_owned", False) and _lib is not None:
            _lib.orc_single_free(self._h)
            self._owned = False

    def insert_bulk(self, keys, values, threads: int = 1) -> np.ndarray:
        k, v = _u64(keys), _u64(values)
        st = np.empty(len(k), dtype=np.uint8)
        lib().orc_single_insert_bulk(self._h, _ptr(k), _ptr(v), len(k), _ptr(st), threads)
        return st

    def retrieve_bulk(self, keys, threads: int = 1) -> tuple[np.ndarray, np.ndarray]:
        k = _u64(keys)
        out = np.empty(len(k), dtype=np.uint64)
        found = np.empty(len(k), dtype=np.uint8)
        lib().orc_single_retrieve_bulk(self._h, _ptr(k), len(k), _ptr(out), _ptr(found), threads)
        return out, found

    def find(self, key: int) -> tuple[int, int, int]:
        pr, wi = C.c_uint64(0), C.c_uint64(0)
        slot = lib().orc_single_find(self._h, key, C.byref(pr), C.byref(wi))
        return int(slot), int(pr.value), int(wi.value)

    def erase_bulk(self, keys) -> np.ndarray:
        k = _u64(keys)
        out = np.empty(len(k), dtype=np.uint8)
        lib().orc_single_erase_bulk(self._h, _ptr(k), len(k), _ptr(out))
        return out

    def stats(self) -> dict:
        out = np.zeros(5, dtype=np.int64)
        lib().orc_single_stats(self._h, _ptr(out))
        return dict(zip(("occupied", "tombstones", "ops", "attempts", "windows"),
                        (int(x) for x in out)))

    def dump(self) -> tuple[np.ndarray, np.ndarray]:
        keys = np.empty(self.capacity, dtype=np.uint64)
        vals = np.empty(self.capacity, dtype=np.uint64)
        lib().orc_single_dump(self._h, _ptr(keys), _ptr(vals))
        return keys, vals

    def items(self) -> dict:
        keys, vals = self.dump()
        live = (keys != np.uint64(self.empty_key)) & (keys != np.uint64(self.tombstone_key))
        return dict(zip(keys[live].tolist(), vals[live].tolist()))


class OracleMulti(OracleSingle):
    """Sequential MultiValueHashTable (multi_table.py:33-339)."""

    def insert_bulk(self, keys, values, threads: int = 1) -> np.ndarray:
        k, v = _u64(keys), _u64(values)
        st = np.empty(len(k), dtype=np.uint8)
        lib().orc_multi_insert_bulk(self._h, _ptr(k), _ptr(v), len(k), _ptr(st))
        return st

    def count_bulk(self, keys) -> np.ndarray:
        k = _u64(keys)
        out = np.empty(len(k), dtype=np.uint64)
        lib().orc_multi_count_bulk(self._h, _ptr(k), len(k), _ptr(out))
        return out

    def retrieve_bulk(self, keys, threads: int = 1) -> tuple[np.ndarray, np.ndarray]:
        k = _u64(keys)
        offsets = exclusive_prefix_sum(self.count_bulk(k))
        flat = np.zeros(int(offsets[-1]), dtype=np.uint64)
        lib().orc_multi_retrieve_bulk(self._h, _ptr(k), len(k), _ptr(offsets), _ptr(flat))
        return offsets, flat


class OracleBucket:
    """Sequential BucketListHashTable (bucket_list.py:164-407)."""

    def __init__(self, min_keys: int, pool_capacity: int, *, s0: int = 1, factor="1.1",
                 group_width: int = 32, key_bits: int = 64,
                 sentinels: tuple[int, int] | None = None):
        f = Fraction(str(factor)) if not isinstance(factor, Fraction) else factor
        e, t = sentinels if sentinels else default_sentinels(key_bits)
        self.pool_capacity = pool_capacity
        self._h = lib().orc_bucket_new(min_keys, pool_capacity, s0, f.numerator,
                                       f.denominator, group_width, e, t)
        self.key_store = OracleSingle(0, sentinels=(e, t), group_width=group_width,
                                      _handle=lib().orc_bucket_keystore(self._h))

    def __del__(self):
        if getattr(self, "_h", None) and _lib is not None:
            _lib.orc_bucket_free(self._h)
            self._h = None

    def insert_bulk(self, keys, values) -> np.ndarray:
        k, v = _u64(keys), _u64(values)
        st = np.empty(len(k), dtype=np.uint8)
        lib().orc_bucket_insert_bulk(self._h, _ptr(k), _ptr(v), len(k), _ptr(st))
        return st

    def count_bulk(self, keys) -> np.ndarray:
        k = _u64(keys)
        out = np.empty(len(k), dtype=np.uint64)
        lib().orc_bucket_count_bulk(self._h, _ptr(k), len(k), _ptr(out))
        return out

    def retrieve_bulk(self, keys) -> tuple[np.ndarray, np.ndarray]:
        k = _u64(keys)
        offsets = exclusive_prefix_sum(self.count_bulk(k))
        flat = np.zeros(int(offsets[-1]), dtype=np.uint64)
        lib().orc_bucket_retrieve_bulk(self._h, _ptr(k), len(k), _ptr(offsets), _ptr(flat))
        return offsets, flat

    def chain_sizes(self, key: int) -> list[int]:
        out = np.zeros(4096, dtype=np.uint64)
        m = lib().orc_bucket_chain_sizes(self._h, key, _ptr(out), 4096)
        return out[:m].tolist()

    def stats(self) -> dict:
        out = np.zeros(3, dtype=np.uint64)
        lib().orc_bucket_stats(self._h, _ptr(out))
        return {"occupied_keys": int(out[0]), "total_values": int(out[1]),
                "allocated": int(out[2])}

    def arena(self) -> np.ndarray:
        out = np.empty(self.pool_capacity, dtype=np.uint64)
        lib().orc_bucket_dump_arena(self._h, _ptr(out))
        return out


def pack_handle(state: int, count: int, tail: int) -> int:
    return int(lib().orc_pack_handle(state, count, tail))
