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

    @property
    def num_shards(self) -> int:
        return self.router.num_shards

    def close(self) -> None:
        pass

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

    def _retrieve_distributed(self, k: torch.Tensor):
        n = k.numel()
        perm, off, segs = self._segments(k, None)
        sh = self.shards[0]
        if not self._multi:
            vparts, fparts = [], []
            for s, (ks, _) in enumerate(segs):
                v, f = self.shards[s].retrieve_device(self._to_shard(ks, s))
                vparts.append(self._to_shard(v, 0))
                fparts.append(self._to_shard(f, 0))
            vals = scatter_device(torch.cat(vparts), perm, sh._empty_vals(n))
            found = scatter_device(torch.cat(fparts), perm, sh._u8(n))
            v = _io.from_device(vals, sh.value_bits).tolist()
            f = found.cpu().numpy().tolist()
            return [x if hit else None for x, hit in zip(v, f)]
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
        return dst_off.cpu().tolist(), _io.from_device(flat, sh.value_bits).tolist()

    def _retrieve_independent(self, k: torch.Tensor):
        # broadcast the queries; lowest shard id wins for single-value, concatenation for
        # multi-value (distributed.py:180-195)
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
            v = _io.from_device(vals, sh.value_bits).tolist()
            f = found.cpu().numpy().tolist()
            return [x if hit else None for x, hit in zip(v, f)]
        per_key: list[list[int]] = [[] for _ in range(n)]
        for s in range(self.num_shards):
            o, f = self.shards[s].retrieve_device(self._to_shard(k, s))
            o = o.cpu().tolist()
            f = _io.from_device(f, sh.value_bits).tolist()
            for i in range(n):
                per_key[i].extend(f[o[i]:o[i + 1]])
        offsets = exclusive_prefix_sum([len(p) for p in per_key])
        return offsets, [v for p in per_key for v in p]

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


class ShardedTable:
    """Rank-local shard of a hash-partitioned single-value table (torchrun, NCCL).

    insert_device / retrieve_device are collective: every rank calls them with
    its own batch.  Pipeline per call: split (K10) -> all_to_all (C1) -> local
    K1/K2 -> all_to_all back (C1) -> inverse-permutation scatter (K11).
    """

    def __init__(self, local_table, group=None):
        import torch.distributed as dist
        self.table = local_table
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self.router = ShardRouter(self.world)

    def insert_device(self, keys: torch.Tensor, values: torch.Tensor) -> torch.Tensor:
        perm, offsets, kout, vout = split_device(keys, self.world, values)
        counts = (offsets[1:] - offsets[:-1]).cpu().tolist()
        rk, rcounts = all_to_all_segments(kout, counts, self.group)
        rv, _ = all_to_all_segments(vout, counts, self.group)
        st = self.table.insert_device(rk, rv)
        back = all_to_all_back(st, rcounts, counts, self.group)
        out = torch.empty(keys.numel(), dtype=torch.uint8, device=keys.device)
        return scatter_device(back, perm, out) if keys.numel() else out

    def retrieve_device(self, keys: torch.Tensor):
        perm, offsets, kout, _ = split_device(keys, self.world)
        counts = (offsets[1:] - offsets[:-1]).cpu().tolist()
        rk, rcounts = all_to_all_segments(kout, counts, self.group)
        v, f = self.table.retrieve_device(rk)
        vb = all_to_all_back(v, rcounts, counts, self.group)
        fb = all_to_all_back(f, rcounts, counts, self.group)
        n = keys.numel()
        vals = torch.empty(n, dtype=v.dtype, device=keys.device)
        found = torch.empty(n, dtype=torch.uint8, device=keys.device)
        if n:
            scatter_device(vb, perm, vals)
            scatter_device(fb, perm, found)
        return vals, found
