"""Single-value hash table on B200 (mirrors coophash.single_table).

Every operation is a CUDA kernel (csrc/single.cu) reached through the C ABI:
  insert / insert_bulk          K1 ch_insert        (single_table.py:273-290, 355-374)
  find_or_claim                 K1 ch_find_or_claim (:292-311)
  retrieve / retrieve_bulk      K2 ch_retrieve      (:313-327, 376-408)
  retrieve_with_stats / slot_of ch_find             (:317-336)
  erase                         K3 ch_erase         (:338-351)
  for_each / for_all            ch_find / slot read-back (:412-429)
Gauges (occupied, tombstones, probe counters) are device counters reduced per
CTA and read back on demand (ch_get_stats).

The list API keeps the reference's signatures and return types.  The
``*_device`` methods take and return CUDA tensors (no host round trip).
"""
from __future__ import annotations

from dataclasses import dataclass
from enum import Enum
from typing import Callable, Iterable, Optional, Sequence

import numpy as np
import torch

from . import _io, _lib
from .layout import DeviceTable, LayoutKind, Sentinels, SlotArray, as_layout, default_sentinels
from .probing import CapacityPlan, ProbingConfig, ProbingScheme, choose_capacity


class InsertStatus(Enum):
    INSERTED = "inserted"
    DUPLICATE_KEY = "duplicate_key"
    TABLE_FULL = "table_full"
    INVALID_KEY = "invalid_key"
    OUT_OF_MEMORY = "out_of_memory"


STATUS_BY_CODE = tuple(InsertStatus)


@dataclass(frozen=True)
class ProbeStats:
    attempts: int
    windows_visited: int


@dataclass
class ProbeCounters:
    ops: int = 0
    attempts: int = 0
    windows_visited: int = 0

    @property
    def mean_attempts(self) -> float:
        return self.attempts / self.ops if self.ops else 0.0


def statuses_from_codes(codes: np.ndarray) -> list[InsertStatus]:
    return [STATUS_BY_CODE[c] for c in codes.tolist()]


def _host_tensor(x, bits: int) -> torch.Tensor:
    """Host data as a pinned integer tensor of the storage width."""
    dt = _io.torch_dtype(bits)
    if isinstance(x, torch.Tensor) and not x.is_cuda and x.dtype == dt:
        return x if x.is_pinned() else x.pin_memory()
    if isinstance(x, torch.Tensor):
        x = x.cpu().numpy()
    arr = _io.to_numpy(x, bits)
    return torch.from_numpy(arr.view(np.int32 if bits <= 32 else np.int64)).pin_memory()


class _TableBase:
    """Construction and gauges shared by the three table kinds."""

    _kind = _lib.CH_SINGLE

    def _setup(self, min_capacity, *, layout, key_bits, value_bits, sentinels, group_width,
               scheme, max_outer_attempts, workers, plan, device, pool_capacity=0,
               growth=(0, 0, 0), handle_bits=None):
        layout = as_layout(layout)
        if plan is None:
            plan = choose_capacity(max(min_capacity, 32))
        self.config = ProbingConfig(plan=plan, scheme=scheme, group_width=group_width,
                                    max_outer_attempts=max_outer_attempts)
        if sentinels is None:
            sentinels = default_sentinels(key_bits)
        vbits = handle_bits if handle_bits is not None else value_bits
        if layout == LayoutKind.PACKED_AOS and (key_bits > 32 or vbits > 32):
            from .layout import LayoutUnsupported
            raise LayoutUnsupported("packed layout needs 32-bit keys and values")
        self._dt = DeviceTable(kind=self._kind, layout=layout, key_bits=key_bits, value_bits=value_bits,
                               group_width=group_width, p=plan.p,
                               max_outer_attempts=self.config.max_outer_attempts,
                               sentinels=sentinels, device=device, pool_capacity=pool_capacity,
                               growth=growth)
        self.key_bits, self.value_bits = key_bits, value_bits
        self.layout = layout
        self.workers = workers
        self.device = self._dt.device
        self._packed = layout == LayoutKind.PACKED_AOS
        self.slots = SlotArray(plan.c, layout, sentinels, key_bits=key_bits, value_bits=vbits,
                               _table=self._dt)
        self.sentinels = sentinels

    # -- introspection ---------------------------------------------------
    @property
    def capacity(self) -> int:
        return self._dt.capacity

    @property
    def occupied(self) -> int:
        return int(self._dt.stats().occupied)

    def load_factor(self) -> float:
        return self.occupied / self.capacity

    def probe_counters(self) -> ProbeCounters:
        s = self._dt.stats()
        return ProbeCounters(ops=int(s.ops), attempts=int(s.attempts), windows_visited=int(s.windows))

    # -- device functors (single_table.py:412-429) -------------
    def _cell_value_dtype(self) -> torch.dtype:
        bits = 64 if self._kind == _lib.CH_BUCKET else self.value_bits  # bucket cells hold handles
        return _io.torch_dtype(bits)

    def for_all_device(self, fn: Callable | None = None, stream=None):
        """The live cells (neither empty nor tombstone) in slot order, compacted on the
        device by ch_for_all: CUDA tensors (keys, values, slots).  With ``fn``, returns
        fn(keys, values, slots) -- a functor applied on the device (tensor ops or another
        kernel) instead of one host callback per slot."""
        n = self.occupied
        dev = f"cuda:{self.device}"
        keys = torch.empty(n, dtype=_io.torch_dtype(self.key_bits), device=dev)
        vals = torch.empty(n, dtype=self._cell_value_dtype(), device=dev)
        slots = torch.empty(n, dtype=torch.int64, device=dev)
        _lib.check(_lib.lib().ch_for_all(self._dt.handle, keys.data_ptr(), vals.data_ptr(), slots.data_ptr(), n,
                                         None, self._stream(stream)), "for_all")
        return fn(keys, vals, slots) if fn is not None else (keys, vals, slots)

    def reduce_live(self, stream=None) -> dict:
        """Built-in device functors folded over the live cells in one pass (ch_reduce_live)."""
        out = torch.empty(5, dtype=torch.int64, device=f"cuda:{self.device}")
        _lib.check(_lib.lib().ch_reduce_live(self._dt.handle, out.data_ptr(), self._stream(stream)), "reduce")
        c, sm, kx, mn, mx = (int(x) & ((1 << 64) - 1) for x in out.cpu().tolist())
        return {"count": c, "value_sum": sm, "key_xor": kx, "min_value": mn if c else None,
                "max_value": mx if c else None}

    def deferred_count(self) -> int:
        """Keys the staged-region pass (csrc/staged.cu) handed to the COPS probe kernels
        since the last reset_probe_counters() (window 0 could not decide them)."""
        return int(self._dt.stats().deferred)

    def reset_probe_counters(self) -> None:
        _lib.check(_lib.lib().ch_reset_probe_counters(self._dt.handle, self._stream()),
                   "reset_probe_counters")

    def set_locality(self, mode) -> None:
        """Schedule of big batches: "auto" (default), "off" (direct probes), "on" (L2 region
        order, csrc/locality.cu) or "staged" (shared-memory staged regions, csrc/staged.cu;
        packed tables, other layouts run direct)."""
        code = {"auto": 0, "off": 1, "on": 2, "staged": 3}.get(mode, mode)
        _lib.check(_lib.lib().ch_set_locality(self._dt.handle, int(code)), "set_locality")

    def batch_schedule(self, n: int) -> str:
        """Schedule a bulk insert / retrieve of n keys takes: "direct", "l2_order" or "staged"."""
        code = _lib.lib().ch_batch_schedule(self._dt.handle, int(n))
        if code < 0:
            _lib.check(code, "batch_schedule")
        return {1: "direct", 2: "l2_order", 3: "staged"}[code]

    def kernel_timing(self, enable: bool = True) -> None:
        """Record CUDA events around every probe-kernel launch of this table."""
        _lib.check(_lib.lib().ch_kernel_timing(self._dt.handle, int(bool(enable))), "kernel_timing")

    def kernel_times(self) -> list[float]:
        """Device time (ms) of each timed probe-kernel launch, in launch order; resets."""
        import ctypes as C
        cnt = C.c_uint64(0)
        buf = (C.c_double * 4096)()
        _lib.check(_lib.lib().ch_kernel_time(self._dt.handle, buf, 4096, C.byref(cnt)), "kernel_time")
        return [buf[i] for i in range(min(cnt.value, 4096))]

    def synchronize(self) -> None:
        _lib.check(_lib.lib().ch_synchronize(self._dt.handle), "synchronize")

    # -- helpers -----------------------------------------------------------
    def _stream(self, stream=None) -> int:
        return _io.stream_of(self.device, stream)

    def _keys(self, keys) -> torch.Tensor:
        return _io.to_device(keys, self.key_bits, self.device, "key")

    def _vals(self, vals) -> torch.Tensor:
        return _io.to_device(vals, self.value_bits, self.device, "value")

    def _empty_vals(self, n: int) -> torch.Tensor:
        return torch.empty(n, dtype=_io.torch_dtype(self.value_bits), device=f"cuda:{self.device}")

    def _u8(self, n: int) -> torch.Tensor:
        return torch.empty(n, dtype=torch.uint8, device=f"cuda:{self.device}")

    def _is_sentinel(self, key: int) -> bool:
        return self.sentinels.is_sentinel(key)


class SingleValueHashTable(_TableBase):
    """Concurrent open-addressing table mapping each key to one value (HBM-resident)."""

    _kind = _lib.CH_SINGLE

    def __init__(self, min_capacity: int, *, layout: LayoutKind | str = LayoutKind.SOA,
                 key_bits: int = 64, value_bits: int = 64, sentinels: Sentinels | None = None,
                 group_width: int = 32, scheme: ProbingScheme = ProbingScheme.COOPERATIVE,
                 max_outer_attempts: int | None = None, workers: int = 1,
                 plan: CapacityPlan | None = None, device=None):
        self._setup(min_capacity, layout=layout, key_bits=key_bits, value_bits=value_bits,
                    sentinels=sentinels, group_width=group_width, scheme=scheme,
                    max_outer_attempts=max_outer_attempts, workers=workers, plan=plan, device=device)

    @property
    def tombstones(self) -> int:
        return int(self._dt.stats().tombstones)

    # -- device-native bulk API -----------------------------------------------
    def insert_device(self, keys, values, status: torch.Tensor | None = None, stream=None) -> torch.Tensor:
        """K1 over CUDA tensors; returns the uint8 InsertStatus codes."""
        k, v = self._keys(keys), self._vals(values)
        if k.numel() != v.numel():
            raise ValueError("keys and values differ in length")
        n = k.numel()
        st = status if status is not None else self._u8(n)
        _lib.check(_lib.lib().ch_insert(self._dt.handle, k.data_ptr(), v.data_ptr(), n, st.data_ptr(),
                                        self._stream(stream)), "insert")
        self._dt.touch()
        return st

    def retrieve_device(self, keys, values_out: torch.Tensor | None = None,
                        found_out: torch.Tensor | None = None, stream=None):
        """K2 over CUDA tensors; returns (values, found) (values of misses are 0)."""
        k = self._keys(keys)
        n = k.numel()
        vals = values_out if values_out is not None else self._empty_vals(n)
        found = found_out if found_out is not None else self._u8(n)
        _lib.check(_lib.lib().ch_retrieve(self._dt.handle, k.data_ptr(), n, vals.data_ptr(),
                                          found.data_ptr(), self._stream(stream)), "retrieve")
        return vals, found

    def erase_device(self, keys, stream=None) -> torch.Tensor:
        k = self._keys(keys)
        n = k.numel()
        out = self._u8(n)
        _lib.check(_lib.lib().ch_erase(self._dt.handle, k.data_ptr(), n, out.data_ptr(),
                                       self._stream(stream)), "erase")
        self._dt.touch()
        return out

    def find_device(self, keys, *, with_stats: bool = False, with_values: bool = False, stream=None):
        k = self._keys(keys)
        n = k.numel()
        dev = f"cuda:{self.device}"
        slots = torch.empty(n, dtype=torch.int64, device=dev)
        att = torch.empty(n, dtype=torch.int32, device=dev) if with_stats else None
        win = torch.empty(n, dtype=torch.int32, device=dev) if with_stats else None
        vals = self._empty_vals(n) if with_values else None
        _lib.check(_lib.lib().ch_find(self._dt.handle, k.data_ptr(), n, slots.data_ptr(),
                                      att.data_ptr() if att is not None else None,
                                      win.data_ptr() if win is not None else None,
                                      vals.data_ptr() if vals is not None else None,
                                      self._stream(stream)), "find")
        return slots, att, win, vals

    # -- host-buffer bulk API (pipelined H2D / kernels / D2H) ---------------------
    def insert_host(self, keys, values, chunk: int | None = None,
                    status_out: torch.Tensor | None = None, sync: bool = True) -> torch.Tensor:
        """Bulk insert from (pinned) host tensors; returns pinned host status codes.
        Copies and kernels of consecutive chunks overlap (_io.pipelined).  ``sync=False``
        returns at once: the statuses are valid after the device's current stream
        synchronises (e.g. at the end of a following retrieve_host), and that call's
        copies overlap this one's remaining kernels."""
        keys = _host_tensor(keys, self.key_bits)
        values = _host_tensor(values, self.value_bits)
        status = status_out if status_out is not None else \
            torch.empty(keys.numel(), dtype=torch.uint8, pin_memory=True)
        _io.pipelined(self.device, [keys, values], [status],
                      lambda d, s: [self.insert_device(d[0], d[1], stream=s)], chunk or self._host_chunk(),
                      self._staging())
        if sync:
            torch.cuda.current_stream(self.device).synchronize()
        return status

    def retrieve_host(self, keys, chunk: int | None = None, values_out: torch.Tensor | None = None,
                      found_out: torch.Tensor | None = None, sync: bool = True) -> tuple[torch.Tensor, torch.Tensor]:
        """Bulk retrieve for (pinned) host keys; returns pinned host (values, found)."""
        keys = _host_tensor(keys, self.key_bits)
        n = keys.numel()
        vals = values_out if values_out is not None else \
            torch.empty(n, dtype=_io.torch_dtype(self.value_bits), pin_memory=True)
        found = found_out if found_out is not None else torch.empty(n, dtype=torch.uint8, pin_memory=True)
        _io.pipelined(self.device, [keys], [vals, found],
                      lambda d, s: list(self.retrieve_device(d[0], stream=s)), chunk or self._host_chunk(),
                      self._staging())
        if sync:
            torch.cuda.current_stream(self.device).synchronize()
        return vals, found

    def _staging(self) -> "_io.Staging":
        st = getattr(self, "_stage", None)
        if st is None:
            st = self._stage = _io.Staging()
        return st

    def _host_chunk(self) -> int:
        # c/24 keys per chunk: short pipeline fill / drain, and each chunk still covers the
        # table densely enough for region-ordered execution (tools/e2e_sweep.py: c/8 77.6 ms,
        # c/12 76.2 ms, c/24 74.0 ms per insert_host + retrieve_host of 2^28 keys)
        return max(1 << 20, -(-self.capacity // 24))

    # -- element operations (single_table.py:273-351) ---------------------------
    def insert(self, key: int, value: int) -> InsertStatus:
        return self.insert_bulk([(key, value)])[0]

    def find_or_claim(self, key: int) -> tuple[InsertStatus, int]:
        k = self._keys([key])
        st = self._u8(1)
        slots = torch.empty(1, dtype=torch.int64, device=f"cuda:{self.device}")
        _lib.check(_lib.lib().ch_find_or_claim(self._dt.handle, k.data_ptr(), 1, st.data_ptr(),
                                               slots.data_ptr(), self._stream()), "find_or_claim")
        self._dt.touch()
        return STATUS_BY_CODE[int(st.item())], int(slots.item())

    def retrieve(self, key: int) -> Optional[int]:
        return self.retrieve_bulk([key])[0]

    def retrieve_with_stats(self, key: int) -> tuple[Optional[int], ProbeStats]:
        if self._is_sentinel(key):
            return None, ProbeStats(0, 0)
        slots, att, win, vals = self.find_device([key], with_stats=True, with_values=True)
        slot = int(slots.item())
        stats = ProbeStats(int(att.item()), int(win.item()))
        if slot < 0:
            return None, stats
        return int(_io.from_device(vals, self.value_bits)[0]), stats

    def slot_of(self, key: int) -> int:
        if self._is_sentinel(key):
            return -1
        return int(self.find_device([key])[0].item())

    def erase(self, key: int) -> bool:
        if self._is_sentinel(key):
            return False
        return bool(self.erase_device([key]).item())

    # -- bulk operations (single_table.py:355-408) ------------------------------
    def insert_bulk(self, pairs: Sequence[tuple[int, int]], workers: int | None = None) -> list[InsertStatus]:
        keys, vals = _io.split_pairs(pairs)
        if not keys:
            return []
        st = self.insert_device(keys, vals)
        return statuses_from_codes(st.cpu().numpy())

    def retrieve_bulk(self, keys: Sequence[int], workers: int | None = None) -> list[Optional[int]]:
        keys = list(keys)
        if not keys:
            return []
        vals, found = self.retrieve_device(keys)
        v = _io.from_device(vals, self.value_bits).tolist()
        f = found.cpu().numpy().tolist()
        return [x if hit else None for x, hit in zip(v, f)]

    # -- callbacks (single_table.py:412-429) ------------------------------------
    def for_each(self, keys: Iterable[int], callback: Callable[[int, int, int], None]) -> None:
        keys = [k for k in keys if not self._is_sentinel(k)]
        if not keys:
            return
        slots, _, _, vals = self.find_device(keys, with_values=True)
        s = slots.cpu().numpy().tolist()
        v = _io.from_device(vals, self.value_bits).tolist()
        for k, slot, val in zip(keys, s, v):
            if slot >= 0:
                callback(k, val, slot)

    def for_each_device(self, keys, fn: Callable | None = None, stream=None):
        """The present queries as CUDA tensors (keys, values, slots), in query order; with
        ``fn``, fn(keys, values, slots) runs on them on the device."""
        k = self._keys(keys)
        slots, _, _, vals = self.find_device(k, with_values=True, stream=stream)
        hit = slots >= 0
        out = (k[hit], vals[hit], slots[hit])
        return fn(*out) if fn is not None else out

    def for_all(self, callback: Callable[[int, int, int], None]) -> None:
        """callback(key, value, slot) per live cell in slot order (single_table.py:425-429);
        the cells are enumerated on the device (ch_for_all), only the live ones cross."""
        keys, vals, slots = self.for_all_device()
        kb, vb = self.key_bits, self.value_bits
        for k, v, i in zip(_io.from_device(keys, kb).tolist(), _io.from_device(vals, vb).tolist(),
                           slots.cpu().tolist()):
            callback(k, v, i)
