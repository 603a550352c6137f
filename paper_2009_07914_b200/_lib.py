"""ctypes binding of libcoophash_b200.so (include/coophash_b200.h).

The shared library is the product: every table operation below is a CUDA
kernel launch through this C ABI.  There is no CPU fallback -- if the
library or a GPU is missing, constructing a table raises.
"""
from __future__ import annotations

import ctypes as C
import os
import threading

_HERE = os.path.dirname(os.path.abspath(__file__))
# CH_LIB_PATH: an alternative build of the same library (A/B measurements, tools/ab.sh)
LIB_PATH = os.environ.get("CH_LIB_PATH") or os.path.join(_HERE, "libcoophash_b200.so")

CH_OK, CH_EINVAL, CH_ENOMEM, CH_EIO, CH_ETIMEDOUT = 0, -22, -12, -5, -110
CH_SINGLE, CH_MULTI, CH_BUCKET = 0, 1, 2
CH_SOA, CH_AOS, CH_PACKED = 0, 1, 2
CH_DIST_AUTO, CH_DIST_NCCL, CH_DIST_COPY = 0, 1, 2


class ch_config(C.Structure):
    _fields_ = [
        ("kind", C.c_int), ("layout", C.c_int), ("key_bits", C.c_int), ("value_bits", C.c_int),
        ("group_width", C.c_int), ("p", C.c_uint64), ("max_outer_attempts", C.c_uint64),
        ("empty_key", C.c_uint64), ("tombstone_key", C.c_uint64), ("pool_capacity", C.c_uint64),
        ("growth_s0", C.c_uint64), ("growth_num", C.c_uint64), ("growth_den", C.c_uint64),
        ("device", C.c_int),
    ]


class ch_stats(C.Structure):
    _fields_ = [
        ("capacity", C.c_uint64), ("occupied", C.c_int64), ("tombstones", C.c_int64),
        ("ops", C.c_uint64), ("attempts", C.c_uint64), ("windows", C.c_uint64),
        ("total_values", C.c_int64), ("pool_allocated", C.c_uint64), ("device_error", C.c_uint64),
        ("deferred", C.c_uint64),
    ]


_P = C.c_void_p
_U64 = C.c_uint64
_SIGS = {
    "ch_last_error": (C.c_char_p, []),
    "ch_version": (C.c_int, []),
    "ch_kernel_launches": (C.c_uint64, []),
    "ch_create": (C.c_int, [C.POINTER(_P), C.POINTER(ch_config)]),
    "ch_destroy": (C.c_int, [_P]),
    "ch_clear": (C.c_int, [_P, _P]),
    "ch_get_stats": (C.c_int, [_P, C.POINTER(ch_stats)]),
    "ch_reset_probe_counters": (C.c_int, [_P, _P]),
    "ch_synchronize": (C.c_int, [_P]),
    "ch_set_locality": (C.c_int, [_P, C.c_int]),
    "ch_batch_schedule": (C.c_int, [_P, _U64]),
    "ch_set_multi_grouping": (C.c_int, [_P, C.c_int]),
    "ch_kernel_timing": (C.c_int, [_P, C.c_int]),
    "ch_kernel_time": (C.c_int, [_P, C.POINTER(C.c_double), C.c_uint64, C.POINTER(C.c_uint64)]),
    "ch_insert": (C.c_int, [_P, _P, _P, _U64, _P, _P]),
    "ch_find_or_claim": (C.c_int, [_P, _P, _U64, _P, _P, _P]),
    "ch_retrieve": (C.c_int, [_P, _P, _U64, _P, _P, _P]),
    "ch_erase": (C.c_int, [_P, _P, _U64, _P, _P]),
    "ch_find": (C.c_int, [_P, _P, _U64, _P, _P, _P, _P, _P]),
    "ch_multi_insert": (C.c_int, [_P, _P, _P, _U64, _P, _P]),
    "ch_multi_count": (C.c_int, [_P, _P, _U64, _P, _P, _P]),
    "ch_multi_retrieve": (C.c_int, [_P, _P, _U64, _P, _P, _P]),
    "ch_multi_retrieve_slots": (C.c_int, [_P, _P, _U64, _P, _P, _P, _P]),
    "ch_for_all": (C.c_int, [_P, _P, _P, _P, _U64, _P, _P]),
    "ch_reduce_live": (C.c_int, [_P, _P, _P]),
    "ch_bucket_insert": (C.c_int, [_P, _P, _P, _U64, _P, _P]),
    "ch_bucket_count": (C.c_int, [_P, _P, _U64, _P, _P, _P, _P]),
    "ch_bucket_retrieve": (C.c_int, [_P, _P, _U64, _P, _P, _P]),
    "ch_read_slots": (C.c_int, [_P, _P, _P]),
    "ch_write_slots": (C.c_int, [_P, _P, _P]),
    "ch_read_slot_range": (C.c_int, [_P, _U64, _U64, _P, _P]),
    "ch_read_arena": (C.c_int, [_P, _P, _U64]),
    "ch_slot_op": (C.c_int, [_P, C.c_int, _U64, _U64, _U64, _U64, C.POINTER(C.c_int),
                             C.POINTER(_U64), C.POINTER(_U64)]),
    "ch_exclusive_scan_u32": (C.c_int, [_P, _U64, _P, C.c_int, _P]),
    "ch_mix64": (C.c_int, [_P, _U64, _U64, _P, C.c_int, _P]),
    "ch_multi_split": (C.c_int, [_P, C.c_int, _P, C.c_int, _U64, C.c_uint32, _P, _P, _P, _P,
                                 C.c_int, _P]),
    "ch_partition": (C.c_int, [_P, _U64, C.c_uint32, _P, _P, C.c_int, _P]),
    "ch_scatter": (C.c_int, [_P, C.c_int, _P, _U64, _P, C.c_int, _P]),
    "ch_gather": (C.c_int, [_P, C.c_int, _P, _U64, _P, C.c_int, _P]),
    "ch_segment_copy": (C.c_int, [_P, C.c_int, _P, _P, _U64, _P, _P, C.c_int, _P]),
    "ch_get_config": (C.c_int, [_P, C.POINTER(ch_config)]),
    "ch_dist_create": (C.c_int, [C.POINTER(_P), C.POINTER(_P), C.c_int, C.c_int]),
    "ch_dist_destroy": (C.c_int, [_P]),
    "ch_dist_info": (C.c_int, [_P, C.POINTER(C.c_int), C.POINTER(C.c_int)]),
    "ch_dist_insert": (C.c_int, [_P, C.POINTER(_P), C.POINTER(_P), C.POINTER(_U64), C.POINTER(_P),
                                 C.POINTER(_P)]),
    "ch_dist_retrieve": (C.c_int, [_P, C.POINTER(_P), C.POINTER(_U64), C.POINTER(_P), C.POINTER(_P),
                                   C.POINTER(_P)]),
    "ch_kmer_sketch": (C.c_int, [_P, _P, _P, _P, _U64, _U64, C.c_int, C.c_uint32, _P, _P, _P, C.c_int, _P]),
    "ch_multi_split32": (C.c_int, [_P, C.c_int, _P, C.c_int, _U64, C.c_uint32, _P, _P, _P, _P,
                                   C.c_int, _P]),
    "ch_scatter32": (C.c_int, [_P, C.c_int, _P, _U64, _P, C.c_int, _P]),
    "ch_route_split32": (C.c_int, [_P, C.c_int, _P, C.c_int, _U64, C.c_uint32, _P, _P, _P, _P, C.c_int, _P]),
    "ch_route_part32": (C.c_int, [_P, _P, _U64, C.c_uint32, _U64, _P, _P, _P, _P, _P, C.c_int, _P]),
    "ch_gather32": (C.c_int, [_P, C.c_int, _P, _U64, _P, C.c_int, _P]),
}

_lib = None
_lock = threading.Lock()


class ExtensionMissing(RuntimeError):
    """The CUDA library is not built or cannot be loaded (no CPU fallback exists)."""


def lib():
    """Load the CUDA library once; raise loudly if it is missing."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise ExtensionMissing(
                    f"{LIB_PATH} is not built; run __graft_entry__.build() "
                    "(there is no CPU fallback)")
            handle = C.CDLL(LIB_PATH)
            for name, (res, args) in _SIGS.items():
                fn = getattr(handle, name)
                fn.restype = res
                fn.argtypes = args
            _lib = handle
    return _lib


def exported_symbols() -> list[str]:
    return sorted(_SIGS)


def last_error() -> str:
    msg = lib().ch_last_error()
    return msg.decode() if msg else ""


def check(rc: int, what: str = "") -> None:
    """Map negative ABI codes to Python exceptions (mirrors the reference's)."""
    if rc == CH_OK:
        return
    msg = last_error() or what
    if rc == CH_EINVAL:
        from .layout import LayoutUnsupported
        if msg.startswith("packed layout needs") or "requires the packed layout" in msg \
                or "not available on packed" in msg:
            raise LayoutUnsupported(msg)
        raise ValueError(msg)
    if rc == CH_ENOMEM:
        raise MemoryError(msg)
    if rc == CH_ETIMEDOUT:
        from .bucket_list import ContentionTimeout
        raise ContentionTimeout(msg)
    raise RuntimeError(f"CUDA error in {what}: {msg}")


def require_cuda(device) -> int:
    """Resolve a CUDA device ordinal; raise when no GPU is present."""
    import torch
    if not torch.cuda.is_available():
        raise ExtensionMissing("no CUDA device: the B200 tables have no CPU fallback")
    lib()
    if device is None:
        return torch.cuda.current_device()
    if isinstance(device, torch.device):
        return device.index if device.index is not None else torch.cuda.current_device()
    if isinstance(device, str):
        d = torch.device(device)
        return d.index if d.index is not None else torch.cuda.current_device()
    return int(device)
