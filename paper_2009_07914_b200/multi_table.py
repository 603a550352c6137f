"""Multi-value hash table on B200 (mirrors coophash.multi_table).

  insert / insert_bulk   K4 ch_multi_insert   (multi_table.py:107-152, 207-226)
  count / count_bulk     K5 ch_multi_count    (:154-160, 228-254) -- counts + device prefix sum
  retrieve_bulk          K5 then K6 ch_multi_retrieve (:256-295): two passes, values of query i
                         at values[offsets[i]:offsets[i+1]] in probe order
"""
from __future__ import annotations

from itertools import accumulate
from typing import Callable, Iterable, Sequence

import numpy as np
import torch

from . import _io, _lib
from .layout import LayoutKind, Sentinels
from .probing import CapacityPlan, ProbingScheme
from .single_table import InsertStatus, _TableBase, statuses_from_codes


def exclusive_prefix_sum(counts):
    """offsets[0] = 0, offsets[i+1] = offsets[i] + counts[i] (multi_table.py:28-30).

    A CUDA uint32/int32 tensor is scanned on the device (ch_exclusive_scan_u32)
    into an int64 tensor; sequences return a list like the reference.
    """
    if isinstance(counts, torch.Tensor) and counts.is_cuda:
        c = counts.contiguous()
        if c.element_size() != 4:
            c = c.to(torch.int32)
        out = torch.empty(c.numel() + 1, dtype=torch.int64, device=c.device)
        _lib.check(_lib.lib().ch_exclusive_scan_u32(c.data_ptr(), c.numel(), out.data_ptr(), c.device.index,
                                                    torch.cuda.current_stream(c.device).cuda_stream), "scan")
        return out
    return list(accumulate(counts, initial=0))


class MultiValueHashTable(_TableBase):
    """Concurrent open-addressing table storing every (key, value) pair (HBM-resident)."""

    _kind = _lib.CH_MULTI

    def __init__(self, min_capacity: int, *, layout: LayoutKind | str = LayoutKind.SOA,
                 key_bits: int = 64, value_bits: int = 64, sentinels: Sentinels | None = None,
                 group_width: int = 32, scheme: ProbingScheme = ProbingScheme.COOPERATIVE,
                 max_outer_attempts: int | None = None, workers: int = 1,
                 plan: CapacityPlan | None = None, device=None):
        self._setup(min_capacity, layout=layout, key_bits=key_bits, value_bits=value_bits,
                    sentinels=sentinels, group_width=group_width, scheme=scheme,
                    max_outer_attempts=max_outer_attempts, workers=workers, plan=plan, device=device)

    def storage_density(self) -> float:
        # one slot per value: density coincides with the load factor (multi_table.py:71-74)
        return self.load_factor()

    # -- device-native API ----------------------------------------------------
    def insert_device(self, keys, values, stream=None) -> torch.Tensor:
        k, v = self._keys(keys), self._vals(values)
        if k.numel() != v.numel():
            raise ValueError("keys and values differ in length")
        n = k.numel()
        st = self._u8(n)
        _lib.check(_lib.lib().ch_multi_insert(self._dt.handle, k.data_ptr(), v.data_ptr(), n, st.data_ptr(),
                                              self._stream(stream)), "multi insert")
        self._dt.touch()
        return st

    def set_grouping(self, on: bool) -> None:
        """Bulk inserts of >= 4096 pairs group the batch by key first and walk each distinct
        key's sequence once (csrc/mgroup.cu); off = the reference's pair-by-pair order."""
        _lib.check(_lib.lib().ch_set_multi_grouping(self._dt.handle, int(bool(on))), "set_grouping")

    def count_device(self, keys, stream=None) -> tuple[torch.Tensor, torch.Tensor]:
        """Counting pass + device exclusive scan: (counts int32, offsets int64[n+1])."""
        k = self._keys(keys)
        n = k.numel()
        dev = f"cuda:{self.device}"
        counts = torch.empty(n, dtype=torch.int32, device=dev)
        offsets = torch.empty(n + 1, dtype=torch.int64, device=dev)
        _lib.check(_lib.lib().ch_multi_count(self._dt.handle, k.data_ptr(), n, counts.data_ptr(),
                                             offsets.data_ptr(), self._stream(stream)), "multi count")
        return counts, offsets

    def retrieve_device(self, keys, stream=None) -> tuple[torch.Tensor, torch.Tensor]:
        """Two-pass bulk retrieval: (offsets int64[n+1], values)."""
        k = self._keys(keys)
        n = k.numel()
        _, offsets = self.count_device(k, stream)
        total = int(offsets[n].item()) if n else 0  # sizes the output (one D2H read)
        vals = torch.zeros(total, dtype=_io.torch_dtype(self.value_bits), device=f"cuda:{self.device}")
        if n and total:
            _lib.check(_lib.lib().ch_multi_retrieve(self._dt.handle, k.data_ptr(), n, offsets.data_ptr(),
                                                    vals.data_ptr(), self._stream(stream)), "multi retrieve")
        elif n:
            # the reference still walks the second pass (ops += n, multi_table.py:290)
            _lib.check(_lib.lib().ch_multi_retrieve(self._dt.handle, k.data_ptr(), n, offsets.data_ptr(),
                                                    None, self._stream(stream)), "multi retrieve")
        return offsets, vals

    # -- element operations -----------------------------------------------------
    def insert(self, key: int, value: int) -> InsertStatus:
        return self.insert_bulk([(key, value)])[0]

    def count(self, key: int) -> int:
        if self._is_sentinel(key):
            return 0
        return self.count_bulk([key])[0]

    def retrieve(self, key: int) -> list[int]:
        if self._is_sentinel(key):
            return []
        return self.retrieve_bulk([key])[1]

    # -- bulk operations ----------------------------------------------------------
    def insert_bulk(self, pairs: Sequence[tuple[int, int]], workers: int | None = None) -> list[InsertStatus]:
        keys, vals = _io.split_pairs(pairs)
        if not keys:
            return []
        return statuses_from_codes(self.insert_device(keys, vals).cpu().numpy())

    def count_bulk(self, keys: Sequence[int], workers: int | None = None) -> list[int]:
        keys = list(keys)
        if not keys:
            return []
        counts, _ = self.count_device(keys)
        return counts.cpu().numpy().astype(np.int64).tolist()

    def retrieve_bulk(self, keys: Sequence[int], workers: int | None = None) -> tuple[list[int], list[int]]:
        keys = list(keys)
        if not keys:
            return [0], []
        offsets, vals = self.retrieve_device(keys)
        return offsets.cpu().numpy().tolist(), _io.from_device(vals, self.value_bits).tolist()

    # -- callbacks (multi_table.py:299-339) ------------------------------------------
    def retrieve_slots_device(self, keys, stream=None):
        """Two-pass retrieval that also returns each value's slot (ch_multi_retrieve_slots):
        (offsets int64[n+1], values, slots int64) on the device, values in probe order."""
        k = self._keys(keys)
        n = k.numel()
        _, offsets = self.count_device(k, stream)
        total = int(offsets[n].item()) if n else 0
        dev = f"cuda:{self.device}"
        vals = torch.zeros(total, dtype=_io.torch_dtype(self.value_bits), device=dev)
        slots = torch.full((total,), -1, dtype=torch.int64, device=dev)
        if n and total:
            _lib.check(_lib.lib().ch_multi_retrieve_slots(self._dt.handle, k.data_ptr(), n, offsets.data_ptr(),
                                                          vals.data_ptr(), slots.data_ptr(), self._stream(stream)),
                       "multi retrieve slots")
        return offsets, vals, slots

    def for_each_device(self, keys, fn: Callable | None = None, stream=None):
        """Every match of the queries as CUDA tensors (keys, values, slots), query-major and in
        probe order within a query; with ``fn``, fn(keys, values, slots) on the device."""
        k = self._keys(keys)
        offsets, vals, slots = self.retrieve_slots_device(k, stream)
        reps = torch.repeat_interleave(k, (offsets[1:] - offsets[:-1]))
        return fn(reps, vals, slots) if fn is not None else (reps, vals, slots)

    def for_each(self, keys: Iterable[int], callback: Callable[[int, int, int], None]) -> None:
        """callback(key, value, slot) per match (multi_table.py:299-328); matches and their
        slots come from the device walk (ch_multi_retrieve_slots)."""
        keys = [k for k in keys if not self._is_sentinel(k)]
        if not keys:
            return
        ks, vals, slots = self.for_each_device(keys)
        for k, v, s in zip(_io.from_device(ks, self.key_bits).tolist(), _io.from_device(vals, self.value_bits).tolist(),
                           slots.cpu().tolist()):
            callback(k, v, s)

    def for_all(self, callback: Callable[[int, int, int], None]) -> None:
        """callback(key, value, slot) per stored pair in slot order (multi_table.py:330-339),
        enumerated on the device (ch_for_all)."""
        keys, vals, slots = self.for_all_device()
        for k, v, i in zip(_io.from_device(keys, self.key_bits).tolist(),
                           _io.from_device(vals, self.value_bits).tolist(), slots.cpu().tolist()):
            callback(k, v, i)
