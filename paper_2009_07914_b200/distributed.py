"""Hash-partitioned tables (mirrors coophash.distributed) -- K10/C1/K11.

Placement is bit-exact with the reference: a key lives on shard
(mix64(key) >> 32) mod S (distributed.py:44-45).

Two deployments share the device kernels:

* ``DistributedTable(num_shards, shard_factory, mode)`` -- the reference's
  in-process facade (distributed.py:84-230).  Shards are B200 tables (on one
  GPU or one per GPU, as the factory decides).  Route + stable multi-split run
  as one device pass (ch_multi_split); the "exchange" is a view of the split
  output (plus a peer copy when a shard lives on another GPU); results return
  by inverse-permutation scatter (ch_scatter) and, for multi-value shards, a
  segmented copy (ch_segment_copy).

* ``ShardedTable(local_table, group)`` -- one process per GPU (torchrun).
  Each rank owns one shard; a bulk call splits its local batch on the device,
  exchanges segment counts and payloads with NCCL all_to_all over NVLink, runs
  the local kernel, and all_to_all's the results back (C1).
"""
from __future__ import annotations

import threading
from dataclasses import dataclass
from enum import Enum
from typing import Callable, Optional, Sequence

import numpy as np
import torch

from . import _io, _lib
from .multi_table import exclusive_prefix_sum
from .probing import mix64
from .single_table import InsertStatus, STATUS_BY_CODE, statuses_from_codes


class ShardMode(Enum):
    DISTRIBUTED = "distributed"
    INDEPENDENT = "independent"


@dataclass(frozen=True)
class ShardRouter:
    num_shards: int

    def __post_init__(self) -> None:
        if self.num_shards < 1:
            raise ValueError("need at least one shard")

    def route(self, key: int) -> int:
        return (mix64(key) >> 32) % self.num_shards


@dataclass(frozen=True)
class PartitionPlan:
    permutation: list[int]
    offsets: list[int]

    def segment(self, shard: int) -> list[int]:
        return self.permutation[self.offsets[shard]:self.offsets[shard + 1]]


def _cuda_device(device=None) -> int:
    return _lib.require_cuda(device)


def split_device(keys: torch.Tensor, num_shards: int, values: torch.Tensor | None = None, stream=None):
    """Route + stable multi-split on the device (ch_multi_split).

    Returns (perm int64[n], offsets int64[S+1], keys_out, values_out): keys_out[j]
    = keys[perm[j]]; segment s is [offsets[s], offsets[s+1]).
    """
    dev = keys.device.index
    n = keys.numel()
    perm = torch.empty(n, dtype=torch.int64, device=keys.device)
    offsets = torch.empty(num_shards + 1, dtype=torch.int64, device=keys.device)
    kout = torch.empty_like(keys)
    vout = torch.empty_like(values) if values is not None else None
    _lib.check(_lib.lib().ch_multi_split(
        keys.data_ptr(), keys.element_size(), values.data_ptr() if values is not None else None,
        values.element_size() if values is not None else 4, n, num_shards, perm.data_ptr(), offsets.data_ptr(),
        kout.data_ptr(), vout.data_ptr() if vout is not None else None, dev,
        _io.stream_of(dev, stream)), "multi_split")
    return perm, offsets, kout, vout


def split_device32(keys: torch.Tensor, num_shards: int, values: torch.Tensor | None = None, stream=None):
    """split_device with a u32 permutation (ch_multi_split32): batches < 2^32 keys.

    Returns (perm int32[n] holding u32 source indices, offsets int64[S+1], keys_out, values_out)."""
    dev = keys.device.index
    n = keys.numel()
    perm = torch.empty(n, dtype=torch.int32, device=keys.device)
    offsets = torch.empty(num_shards + 1, dtype=torch.int64, device=keys.device)
    kout = torch.empty_like(keys)
    vout = torch.empty_like(values) if values is not None else None
    _lib.check(_lib.lib().ch_multi_split32(
        keys.data_ptr(), keys.element_size(), values.data_ptr() if values is not None else None,
        values.element_size() if values is not None else 4, n, num_shards, perm.data_ptr(), offsets.data_ptr(),
        kout.data_ptr(), vout.data_ptr() if vout is not None else None, dev,
        _io.stream_of(dev, stream)), "multi_split32")
    return perm, offsets, kout, vout


def route_split_device32(keys: torch.Tensor, num_shards: int, values: torch.Tensor | None = None, stream=None):
    """Route + stable split returning the inverse map (ch_route_split32): pos[i] = split
    position of element i.  Results come back with gather_device32(results, pos)."""
    dev = keys.device.index
    n = keys.numel()
    pos = torch.empty(n, dtype=torch.int32, device=keys.device)
    offsets = torch.empty(num_shards + 1, dtype=torch.int64, device=keys.device)
    kout = torch.empty_like(keys)
    vout = torch.empty_like(values) if values is not None else None
    _lib.check(_lib.lib().ch_route_split32(
        keys.data_ptr(), keys.element_size(), values.data_ptr() if values is not None else None,
        values.element_size() if values is not None else 4, n, num_shards, pos.data_ptr(), offsets.data_ptr(),
        kout.data_ptr(), vout.data_ptr() if vout is not None else None, dev,
        _io.stream_of(dev, stream)), "route_split32")
    return pos, offsets, kout, vout


def route_part_device32(keys: torch.Tensor, num_shards: int, values: torch.Tensor | None = None, stream=None,
                        slack: float = 1.05):
    """One-pass route partition (ch_route_part32) into fixed-capacity segments: segment d is
    [d cap, d cap + counts[d]) of the outputs, pos[i] the position of element i.  Returns
    (pos, counts (device u64), flag (device int: a segment passed cap), cap, kout, vout).
    32-bit keys / values, num_shards <= 64."""
    dev = keys.device.index
    n = keys.numel()
    cap = int(n / num_shards * slack) + 4096
    pos = torch.empty(n, dtype=torch.int32, device=keys.device)
    counts = torch.empty(num_shards, dtype=torch.int64, device=keys.device)
    flag = torch.empty(1, dtype=torch.int32, device=keys.device)
    kout = torch.empty(num_shards * cap, dtype=keys.dtype, device=keys.device)
    vout = torch.empty(num_shards * cap, dtype=values.dtype, device=keys.device) if values is not None else None
    _lib.check(_lib.lib().ch_route_part32(
        keys.data_ptr(), values.data_ptr() if values is not None else None, n, num_shards, cap, pos.data_ptr(),
        counts.data_ptr(), kout.data_ptr(), vout.data_ptr() if vout is not None else None, flag.data_ptr(), dev,
        _io.stream_of(dev, stream)), "route_part32")
    return pos, counts, flag, cap, kout, vout


def gather_device32(src: torch.Tensor, pos: torch.Tensor, out: torch.Tensor, stream=None) -> torch.Tensor:
    """out[i] = src[pos[i]] (ch_gather32)."""
    dev = src.device.index
    _lib.check(_lib.lib().ch_gather32(src.data_ptr(), src.element_size(), pos.data_ptr(), out.numel(),
                                      out.data_ptr(), dev, _io.stream_of(dev, stream)), "gather32")
    return out


def scatter_device32(src: torch.Tensor, perm: torch.Tensor, out: torch.Tensor, stream=None) -> torch.Tensor:
    """out[perm[i]] = src[i] with a u32 permutation (ch_scatter32)."""
    dev = src.device.index
    _lib.check(_lib.lib().ch_scatter32(src.data_ptr(), src.element_size(), perm.data_ptr(), src.numel(),
                                       out.data_ptr(), dev, _io.stream_of(dev, stream)), "scatter32")
    return out


def scatter_device(src: torch.Tensor, perm: torch.Tensor, out: torch.Tensor, stream=None) -> torch.Tensor:
    """out[perm[i]] = src[i] (ch_scatter)."""
    dev = src.device.index
    _lib.check(_lib.lib().ch_scatter(src.data_ptr(), src.element_size(), perm.data_ptr(), src.numel(),
                                     out.data_ptr(), dev, _io.stream_of(dev, stream)), "scatter")
    return out


def multi_split(keys: Sequence, router) -> PartitionPlan:
    """Stable partition of a batch by destination shard (distributed.py:59-69).

    ShardRouter routing runs fused on the device; other routers (any object with
    ``route`` and ``num_shards``) are evaluated per key in Python -- their code
    is arbitrary -- and the stable partition itself still runs on the device.
    """
    keys = list(keys)
    n = len(keys)
    dev = _cuda_device()
    S = router.num_shards
    if isinstance(router, ShardRouter) and all(isinstance(k, (int, np.integer)) for k in keys):
        k = _io.to_device(keys, 64, dev)
        perm, offsets, _, _ = split_device(k, S)
    else:
        dest = torch.tensor([router.route(k) for k in keys], dtype=torch.int32).to(f"cuda:{dev}")
        perm = torch.empty(n, dtype=torch.int64, device=f"cuda:{dev}")
        offsets = torch.empty(S + 1, dtype=torch.int64, device=f"cuda:{dev}")
        _lib.check(_lib.lib().ch_partition(dest.data_ptr(), n, S, perm.data_ptr(), offsets.data_ptr(), dev,
                                           _io.stream_of(dev)), "partition")
    return PartitionPlan(permutation=perm.cpu().tolist(), offsets=offsets.cpu().tolist())


def exchange(outboxes: Sequence[Sequence[Sequence]]) -> list[list]:
    """All-to-all on host sequences: inbox[t] = concat_s outboxes[s][t] (distributed.py:72-81)."""
    num = len(outboxes)
    inboxes: list[list] = [[] for _ in range(num)]
    for s in range(num):
        if len(outboxes[s]) != num:
            raise ValueError("every outbox must address every shard")
        for t in range(num):
            inboxes[t].extend(outboxes[s][t])
    return inboxes


def _is_multi(table) -> bool:
    return hasattr(table, "count_bulk")


class NativeDist:
    """ch_dist_* (include/coophash_b200.h): the distributed single-value table in the C ABI.

    Wraps existing single-value shard tables (one per device: NCCL grouped send/recv over
    NVLink; shards sharing a device: copy engines).  ``insert`` / ``retrieve`` take one batch
    per source shard (``None`` = no keys from that source) and return per-source results,
    each on its source's device (distributed.py:131-178)."""

    TRANSPORTS = {"auto": _lib.CH_DIST_AUTO, "nccl": _lib.CH_DIST_NCCL, "copy": _lib.CH_DIST_COPY}

    def __init__(self, shards: Sequence, transport: str = "auto"):
        import ctypes as C
        self.shards = list(shards)
        S = len(self.shards)
        arr = (C.c_void_p * S)(*[t._dt.handle for t in self.shards])
        h = C.c_void_p()
        _lib.check(_lib.lib().ch_dist_create(C.byref(h), arr, S, self.TRANSPORTS[transport]), "dist_create")
        self.handle = h
        ns, tr = C.c_int(), C.c_int()
        _lib.check(_lib.lib().ch_dist_info(h, C.byref(ns), C.byref(tr)), "dist_info")
        self.transport = {v: k for k, v in self.TRANSPORTS.items()}[tr.value]

    def close(self) -> None:
        if getattr(self, "handle", None):
            _lib.lib().ch_dist_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _ptrs(self, ts):
        import ctypes as C
        return (C.c_void_p * len(ts))(*[t.data_ptr() if t is not None and t.numel() else None for t in ts])

    def _prep(self, batches, bits):
        S = len(self.shards)
        if len(batches) != S:
            raise ValueError("one batch per source shard")
        out = []
        for s, b in enumerate(batches):
            out.append(None if b is None else _io.to_device(b, bits, self.shards[s].device))
        return out

    def insert(self, keys: Sequence, values: Sequence) -> list:
        import ctypes as C
        sh = self.shards[0]
        ks = self._prep(keys, sh.key_bits)
        vs = self._prep(values, sh.value_bits)
        n = [0 if k is None else k.numel() for k in ks]
        for k, v in zip(ks, vs):
            if (k is None) != (v is None) or (k is not None and k.numel() != v.numel()):
                raise ValueError("keys and values differ in length")
        st = [torch.empty(n[s], dtype=torch.uint8, device=f"cuda:{t.device}") for s, t in enumerate(self.shards)]
        streams = (C.c_void_p * len(n))(*[_io.stream_of(t.device) for t in self.shards])
        _lib.check(_lib.lib().ch_dist_insert(self.handle, self._ptrs(ks), self._ptrs(vs),
                                             (C.c_uint64 * len(n))(*n), self._ptrs(st), streams), "dist_insert")
        for t in self.shards:
            t._dt.touch()
        return st

    def retrieve(self, keys: Sequence) -> list:
        import ctypes as C
        sh = self.shards[0]
        ks = self._prep(keys, sh.key_bits)
        n = [0 if k is None else k.numel() for k in ks]
        vals = [torch.empty(n[s], dtype=_io.torch_dtype(sh.value_bits), device=f"cuda:{t.device}")
                for s, t in enumerate(self.shards)]
        found = [torch.empty(n[s], dtype=torch.uint8, device=f"cuda:{t.device}") for s, t in enumerate(self.shards)]
        streams = (C.c_void_p * len(n))(*[_io.stream_of(t.device) for t in self.shards])
        _lib.check(_lib.lib().ch_dist_retrieve(self.handle, self._ptrs(ks), (C.c_uint64 * len(n))(*n),
                                               self._ptrs(vals), self._ptrs(found), streams), "dist_retrieve")
        return list(zip(vals, found))


class DistributedTable:
    """Bulk facade over per-shard B200 tables (single-, multi- or bucket-value)."""

    def __init__(self, num_shards: int, shard_factory: Callable[[int], object],
                 mode: ShardMode = ShardMode.DISTRIBUTED):
        self.router = ShardRouter(num_shards)
        self.mode = mode
        self.shards = [shard_factory(s) for s in range(num_shards)]
        self._multi = _is_multi(self.shards[0])
        self._bulk_lock = threading.Lock()
        self.device = self.shards[0].device
        # single-value shards in distributed mode run through the C ABI's distributed table
        # (ch_dist_*: split -> exchange -> local -> back -> scatter, all native)
        self._native = None
        if mode == ShardMode.DISTRIBUTED and not self._multi and \
                all(type(t).__name__ == "SingleValueHashTable" for t in self.shards):
            self._native = NativeDist(self.shards)

    @property
    def num_shards(self) -> int:
        return self.router.num_shards

    def close(self) -> None:
        if self._native is not None:
            self._native.close()
            self._native = None

    def __enter__(self) -> "DistributedTable":
        return self

    def __exit__(self, *exc) -> None:
        self.close()

    # -- plumbing ------------------------------------------------------------------------
    def _to_shard(self, t: torch.Tensor, s: int) -> torch.Tensor:
        dev = self.shards[s].device
        return t if t.device.index == dev else t.to(f"cuda:{dev}")

    def _segments(self, keys: torch.Tensor, values: torch.Tensor | None):
        S = self.num_shards
        if self.mode == ShardMode.DISTRIBUTED:
            perm, offsets, kout, vout = split_device(keys, S, values)
            off = offsets.cpu().tolist()
            segs = [(kout[off[s]:off[s + 1]], vout[off[s]:off[s + 1]] if vout is not None else None)
                    for s in range(S)]
            return perm, off, segs
        # independent mode: round-robin scatter of the batch (distributed.py:137-140)
        n = keys.numel()
        idx = torch.arange(n, device=keys.device, dtype=torch.int64)
        perm = torch.cat([idx[s::S] for s in range(S)]) if n else idx
        sizes = [len(range(s, n, S)) for s in range(S)]
        off = [0]
        for z in sizes:
            off.append(off[-1] + z)
        segs = [(keys[s::S].contiguous(), values[s::S].contiguous() if values is not None else None)
                for s in range(S)]
        return perm, off, segs

    # -- insertion (distributed.py:131-147) --------------------------------------------------
    def insert_device(self, keys, values) -> torch.Tensor:
        with self._bulk_lock:
            sh = self.shards[0]
            k = sh._keys(keys)
            v = sh._vals(values)
            n = k.numel()
            if self._native is not None and self.mode == ShardMode.DISTRIBUTED:
                srcs = [k] + [None] * (self.num_shards - 1)
                vsrc = [v] + [None] * (self.num_shards - 1)
                return self._native.insert(srcs, vsrc)[0]
            perm, off, segs = self._segments(k, v)
            parts = []
            for s, (ks, vs) in enumerate(segs):
                st = self.shards[s].insert_device(self._to_shard(ks, s), self._to_shard(vs, s))
                parts.append(self._to_shard(st, 0) if st.device.index != k.device.index else st)
            cat = torch.cat(parts) if parts else torch.empty(0, dtype=torch.uint8, device=k.device)
            out = torch.empty(n, dtype=torch.uint8, device=k.device)
            return scatter_device(cat, perm, out) if n else out

    def insert_bulk(self, pairs: Sequence[tuple[int, int]]) -> list[InsertStatus]:
        keys, vals = _io.split_pairs(pairs)
        if not keys:
            return []
        return statuses_from_codes(self.insert_device(keys, vals).cpu().numpy())

    # -- retrieval (distributed.py:151-203) -----------------------------------------------------
    def retrieve_bulk(self, keys: Sequence[int]):
        with self._bulk_lock:
            keys = list(keys)
            if not keys:
                return ([0], []) if self._multi else []
            sh = self.shards[0]
            k = sh._keys(keys)
            if self.mode == ShardMode.DISTRIBUTED:
                return self._retrieve_distributed(k)
            return self._retrieve_independent(k)

    def retrieve_device(self, keys):
        """Bulk retrieval over CUDA tensors: (values, found) for single-value shards,
        (offsets int64[n+1], flat values) for multi-value / bucket shards, on the
        device of shard 0 (distributed.py:151-203)."""
        with self._bulk_lock:
            k = self.shards[0]._keys(keys)
            if self.mode == ShardMode.DISTRIBUTED:
                return self._retrieve_distributed_device(k)
            return self._retrieve_independent_device(k)

    def _to_lists(self, res):
        sh = self.shards[0]
        if not self._multi:
            vals, found = res
            v = _io.from_device(vals, sh.value_bits).tolist()
            f = found.cpu().numpy().tolist()
            return [x if hit else None for x, hit in zip(v, f)]
        offsets, flat = res
        return offsets.cpu().tolist(), _io.from_device(flat, sh.value_bits).tolist()

    def _retrieve_distributed(self, k: torch.Tensor):
        return self._to_lists(self._retrieve_distributed_device(k))

    def _retrieve_independent(self, k: torch.Tensor):
        return self._to_lists(self._retrieve_independent_device(k))

    def _retrieve_distributed_device(self, k: torch.Tensor):
        n = k.numel()
        sh = self.shards[0]
        if self._native is not None:
            return self._native.retrieve([k] + [None] * (self.num_shards - 1))[0]
        perm, off, segs = self._segments(k, None)
        if not self._multi:
            vparts, fparts = [], []
            for s, (ks, _) in enumerate(segs):
                v, f = self.shards[s].retrieve_device(self._to_shard(ks, s))
                vparts.append(self._to_shard(v, 0))
                fparts.append(self._to_shard(f, 0))
            vals = scatter_device(torch.cat(vparts), perm, sh._empty_vals(n))
            found = scatter_device(torch.cat(fparts), perm, sh._u8(n))
            return vals, found
        # multi-value: per-shard (offsets, flat) -> global offsets in query order -> segmented copy
        cparts, oparts, fparts = [], [], []
        base = 0
        for s, (ks, _) in enumerate(segs):
            o, f = self.shards[s].retrieve_device(self._to_shard(ks, s))
            o = self._to_shard(o, 0)
            cparts.append((o[1:] - o[:-1]).to(torch.int32))
            oparts.append(o[:-1] + base)
            fparts.append(self._to_shard(f, 0))
            base += f.numel()
        counts = scatter_device(torch.cat(cparts), perm, torch.empty(n, dtype=torch.int32, device=k.device))
        dst_off = exclusive_prefix_sum(counts)
        flat_src = torch.cat(fparts)
        flat = torch.zeros(int(dst_off[n].item()), dtype=flat_src.dtype, device=k.device)
        src_off = torch.cat(oparts)
        if flat.numel():
            _lib.check(_lib.lib().ch_segment_copy(flat_src.data_ptr(), flat_src.element_size(), src_off.data_ptr(),
                                                  perm.data_ptr(), n, dst_off.data_ptr(), flat.data_ptr(),
                                                  k.device.index, _io.stream_of(k.device.index)), "segment copy")
        return dst_off, flat

    def _retrieve_independent_device(self, k: torch.Tensor):
        # broadcast the queries; lowest shard id wins for single-value, concatenation in shard
        # order for multi-value (distributed.py:180-195)
        n = k.numel()
        sh = self.shards[0]
        if not self._multi:
            vals = sh._empty_vals(n).zero_()
            found = torch.zeros(n, dtype=torch.bool, device=k.device)
            for s in range(self.num_shards):
                v, f = self.shards[s].retrieve_device(self._to_shard(k, s))
                v, f = self._to_shard(v, 0), self._to_shard(f, 0).bool()
                take = f & ~found
                vals = torch.where(take, v, vals)
                found |= f
            return vals, found.to(torch.uint8)
        res = [self.shards[s].retrieve_device(self._to_shard(k, s)) for s in range(self.num_shards)]
        res = [(self._to_shard(o, 0), self._to_shard(f, 0)) for o, f in res]
        counts = [(o[1:] - o[:-1]) for o, _ in res]
        total_counts = torch.stack(counts).sum(0) if counts else torch.zeros(n, dtype=torch.int64, device=k.device)
        offsets = exclusive_prefix_sum(total_counts.to(torch.int32))
        flat = torch.zeros(int(offsets[n].item()), dtype=res[0][1].dtype, device=k.device)
        base = offsets[:-1].clone()
        for (o, f), c in zip(res, counts):   # shard s's segment of query i follows shards < s
            if f.numel():
                seg_start = torch.repeat_interleave(base - o[:-1], c)
                flat[seg_start + torch.arange(f.numel(), device=k.device)] = f
            base += c
        return offsets, flat

    def count_bulk(self, keys: Sequence[int]) -> list[int]:
        if not self._multi:
            raise TypeError("count_bulk needs multi-value shard tables")
        with self._bulk_lock:
            keys = list(keys)
            if not keys:
                return []
            sh = self.shards[0]
            k = sh._keys(keys)
            n = k.numel()
            if self.mode == ShardMode.DISTRIBUTED:
                perm, off, segs = self._segments(k, None)
                parts = [self._to_shard(self.shards[s].count_device(self._to_shard(ks, s))[0], 0)
                         for s, (ks, _) in enumerate(segs)]
                counts = scatter_device(torch.cat(parts), perm,
                                        torch.empty(n, dtype=torch.int32, device=k.device))
            else:
                counts = torch.zeros(n, dtype=torch.int64, device=k.device)
                for s in range(self.num_shards):
                    counts += self._to_shard(self.shards[s].count_device(self._to_shard(k, s))[0], 0)
            return counts.cpu().numpy().astype(np.int64).tolist()


# ------------------------------------------------------------------ one process per GPU

def all_to_all_segments(send: torch.Tensor, send_counts: list[int], group=None):
    """Exchange variable-length segments with every rank (NCCL all_to_all over NVLink;
    gloo on CPU).  Returns (recv, recv_counts)."""
    import torch.distributed as dist
    world = dist.get_world_size(group)
    home = send.device
    if _host_staged(send, group):
        send = send.cpu()
    sc = torch.tensor(send_counts, dtype=torch.int64, device=send.device)
    rc = torch.empty(world, dtype=torch.int64, device=send.device)
    dist.all_to_all_single(rc, sc, group=group)
    recv_counts = rc.cpu().tolist()
    recv = torch.empty(sum(recv_counts), dtype=send.dtype, device=send.device)
    dist.all_to_all_single(recv, send, output_split_sizes=recv_counts, input_split_sizes=list(send_counts),
                           group=group)
    return recv.to(home), recv_counts


def _host_staged(t: torch.Tensor, group) -> bool:
    """gloo has no device all_to_all: device tensors cross it through host memory.
    Used by the world-size-2 tests that run two ranks on one GPU; NCCL exchanges
    device memory directly."""
    import torch.distributed as dist
    return t.is_cuda and dist.get_backend(group) == "gloo"


def all_to_all_back(send: torch.Tensor, counts_in: list[int], counts_out: list[int], group=None) -> torch.Tensor:
    """Reverse exchange with known split sizes (results travel back to the requesters)."""
    import torch.distributed as dist
    home = send.device
    if _host_staged(send, group):
        send = send.cpu()
    recv = torch.empty(sum(counts_out), dtype=send.dtype, device=send.device)
    dist.all_to_all_single(recv, send, output_split_sizes=list(counts_out), input_split_sizes=list(counts_in),
                           group=group)
    return recv.to(home)


def exchange_segments(sends: Sequence[torch.Tensor], send_counts: list[int], recv_counts: list[int],
                      group=None, send_starts: list[int] | None = None, recv_starts: list[int] | None = None,
                      recv_len: int | None = None) -> list[torch.Tensor]:
    """Variable-length all-to-all of several parallel arrays in ONE grouped exchange.

    ``sends[j]`` holds segments for ranks 0..W-1 back to back (``send_counts``); the
    result ``recvs[j]`` holds what every rank sent this rank, in rank order
    (``recv_counts``).  NCCL: one ``batch_isend_irecv`` group (ncclGroupStart, a
    send + recv per peer and array, ncclGroupEnd) over NVLink; the rank's own segment
    is a device copy.  gloo (CPU tests): the same through host memory."""
    import torch.distributed as dist
    rank = dist.get_rank(group)
    world = dist.get_world_size(group)
    staged = any(_host_staged(t, group) for t in sends)
    home = sends[0].device if sends else None
    src = [t.cpu() if staged else t for t in sends]
    recvs = [torch.empty(recv_len if recv_len is not None else sum(recv_counts), dtype=t.dtype, device=t.device)
             for t in src]
    # segment p: [so[p], so[p] + send_counts[p]) / [ro[p], ro[p] + recv_counts[p]); back to back
    # unless explicit starts are given (fixed-capacity segments of ch_route_part32)
    so = list(send_starts) if send_starts is not None else [sum(send_counts[:p]) for p in range(world)]
    ro = list(recv_starts) if recv_starts is not None else [sum(recv_counts[:p]) for p in range(world)]
    so.append(0)
    ro.append(0)
    sc = list(send_counts)
    rcn = list(recv_counts)
    ops = []
    for j, t in enumerate(src):
        for peer in range(world):
            gpeer = dist.get_global_rank(group, peer) if group is not None else peer
            s_lo, s_hi = so[peer], so[peer] + sc[peer]
            r_lo, r_hi = ro[peer], ro[peer] + rcn[peer]
            if peer == rank:
                if sc[peer]:
                    recvs[j][r_lo:r_hi].copy_(t[s_lo:s_hi])
                continue
            if sc[peer]:
                ops.append(dist.P2POp(dist.isend, t[s_lo:s_hi], gpeer, group))
            if rcn[peer]:
                ops.append(dist.P2POp(dist.irecv, recvs[j][r_lo:r_hi], gpeer, group))
    if ops:
        for w in dist.batch_isend_irecv(ops):
            w.wait()
    return [r.to(home) for r in recvs] if staged else recvs


class ShardedTable:
    """Rank-local shard of a hash-partitioned single-value table (torchrun, NCCL).

    insert_device / retrieve_device are collective: every rank calls them with its own
    batch (distributed.py:131-178, one process per GPU).  Pipeline per call:

      split      one-pass route partition into fixed-capacity segments, u32 position per source
                 element (ch_route_part32; the stable ch_route_split32 for 64-bit keys / values,
                 > 64 ranks or a skewed batch that overflows a segment)
      counts     one all_to_all of the S segment sizes + the overflow flag (the only host sync)
      exchange   keys (+ values) in ONE grouped send/recv (exchange_segments, NVLink)
      local      the shard's own insert / retrieve (staged regions for full-size batches)
      back       statuses / (values, found) in one grouped exchange
      back-map   coalesced gather through that map into the caller's order (K11, ch_gather32)
    """

    def __init__(self, local_table, group=None):
        import torch.distributed as dist
        self.table = local_table
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self.router = ShardRouter(self.world)
        self.last_phase_ms: dict[str, float] = {}

    def _counts(self, offsets: torch.Tensor) -> tuple[list[int], list[int]]:
        import torch.distributed as dist
        sc = (offsets[1:] - offsets[:-1]).to(torch.int64)
        rc = torch.empty_like(sc)
        if _host_staged(sc, self.group):
            sc_h, rc_h = sc.cpu(), torch.empty(self.world, dtype=torch.int64)
            dist.all_to_all_single(rc_h, sc_h, group=self.group)
            return sc_h.tolist(), rc_h.tolist()
        dist.all_to_all_single(rc, sc, group=self.group)
        both = torch.cat([sc, rc]).cpu().tolist()   # one device -> host read per call
        return both[:self.world], both[self.world:]

    def _split(self, k: torch.Tensor, v: torch.Tensor | None):
        """Route + split: the one-pass partition into fixed-capacity segments (ch_route_part32)
        for 32-bit keys / values and <= 64 ranks, the stable split (ch_route_split32)
        otherwise or when a segment overflowed (skewed batch).  Returns (pos, kout, vout,
        send counts, recv counts, send starts)."""
        import torch.distributed as dist
        if k.element_size() == 4 and (v is None or v.element_size() == 4) and self.world <= 64 and k.numel():
            pos, cnt, flag, cap, kout, vout = route_part_device32(k, self.world, v)
            rc = torch.empty_like(cnt)
            if _host_staged(cnt, self.group):
                sc_h, rc_h = cnt.cpu(), torch.empty(self.world, dtype=torch.int64)
                dist.all_to_all_single(rc_h, sc_h, group=self.group)
                both = torch.cat([sc_h, rc_h, flag.cpu().to(torch.int64)]).tolist()
            else:
                dist.all_to_all_single(rc, cnt, group=self.group)
                both = torch.cat([cnt, rc, flag.to(torch.int64)]).cpu().tolist()  # one device -> host read
            ovf = torch.tensor([both[-1]], dtype=torch.int64)
            if not _host_staged(cnt, self.group):
                ovf = ovf.to(k.device)
            dist.all_reduce(ovf, group=self.group)  # every rank takes the same path
            if int(ovf.item()) == 0:
                return pos, kout, vout, both[:self.world], both[self.world:2 * self.world], \
                    [p * cap for p in range(self.world)]
        pos, offsets, kout, vout = route_split_device32(k, self.world, v)
        send, recv = self._counts(offsets)
        return pos, kout, vout, send, recv, None

    def insert_device(self, keys: torch.Tensor, values: torch.Tensor) -> torch.Tensor:
        k = self.table._keys(keys)
        v = self.table._vals(values)
        if k.numel() != v.numel():
            raise ValueError("keys and values differ in length")
        pos, kout, vout, send, recv, starts = self._split(k, v)
        rk, rv = exchange_segments([kout, vout], send, recv, self.group, send_starts=starts)
        st = self.table.insert_device(rk, rv)
        (back,) = exchange_segments([st], recv, send, self.group, recv_starts=starts,
                                    recv_len=kout.numel() if starts is not None else None)
        out = torch.empty(k.numel(), dtype=torch.uint8, device=k.device)
        return gather_device32(back, pos, out) if k.numel() else out

    def retrieve_device(self, keys: torch.Tensor):
        k = self.table._keys(keys)
        pos, kout, _, send, recv, starts = self._split(k, None)
        (rk,) = exchange_segments([kout], send, recv, self.group, send_starts=starts)
        v, f = self.table.retrieve_device(rk)
        vb, fb = exchange_segments([v, f], recv, send, self.group, recv_starts=starts,
                                   recv_len=kout.numel() if starts is not None else None)
        n = k.numel()
        vals = torch.empty(n, dtype=v.dtype, device=k.device)
        found = torch.empty(n, dtype=torch.uint8, device=k.device)
        if n:
            gather_device32(vb, pos, vals)
            gather_device32(fb, pos, found)
        return vals, found
