"""GPU parity: device functors -- for_all / for_each enumerated on the device (ch_for_all,
ch_multi_retrieve_slots, ch_reduce_live) against the host view of the same cells
(reference single_table.py:412-429, multi_table.py:299-339)."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

from paper_2009_07914_b200 import (BucketListHashTable, MultiValueHashTable,  # noqa: E402
                                   SingleValueHashTable)

LAYOUTS = [("soa", 32, 32), ("soa", 64, 64), ("aos", 32, 64), ("aos", 64, 32), ("packed", 32, 32)]


def _host_live(t):
    keys, vals = t._dt.read_slots(64 if isinstance(t, BucketListHashTable) else None)
    e, tb = t.sentinels.empty_key, t.sentinels.tombstone_key
    live = np.nonzero((keys != keys.dtype.type(e)) & (keys != keys.dtype.type(tb)))[0]
    return live, keys[live].astype(np.uint64), vals[live].astype(np.uint64)


def _u(t):
    a = t.cpu().numpy()
    return (a.view(np.uint32) if a.dtype.itemsize == 4 else a.view(np.uint64)).astype(np.uint64)


@pytest.mark.parametrize("layout,kb,vb", LAYOUTS)
def test_for_all_device_equals_slot_view(layout, kb, vb):
    rng = np.random.default_rng(3)
    n = 20_000
    keys = rng.permutation(np.unique(rng.integers(1, 1 << (kb - 1), size=2 * n, dtype=np.uint64)))[:n]
    vals = rng.integers(0, 1 << (vb - 1), size=n, dtype=np.uint64)
    t = SingleValueHashTable(int(n / 0.8), layout=layout, key_bits=kb, value_bits=vb, group_width=8)
    t.insert_bulk(list(zip(keys.tolist(), vals.tolist())))
    t.erase_device(keys[: n // 10].tolist())        # tombstones are not live
    k, v, s = t.for_all_device()
    live, hk, hv = _host_live(t)
    assert np.array_equal(s.cpu().numpy(), live)   # slot order
    assert np.array_equal(_u(k), hk) and np.array_equal(_u(v), hv)
    assert len(live) == t.occupied == n - n // 10
    assert t.for_all_device(lambda kk, vv, ss: int(ss.numel())) == t.occupied   # a device functor
    red = t.reduce_live()
    assert red["count"] == len(live)
    assert red["value_sum"] == int(hv.sum(dtype=np.uint64))
    assert red["key_xor"] == int(np.bitwise_xor.reduce(hk))
    assert red["min_value"] == int(hv.min()) and red["max_value"] == int(hv.max())
    seen = []
    t.for_all(lambda kk, vv, ii: seen.append((kk, vv, ii)))
    assert seen == list(zip(hk.tolist(), hv.tolist(), live.tolist()))


def test_for_all_empty_table():
    t = SingleValueHashTable(1000, layout="packed", key_bits=32, value_bits=32)
    k, v, s = t.for_all_device()
    assert k.numel() == 0
    assert t.reduce_live() == {"count": 0, "value_sum": 0, "key_xor": 0, "min_value": None, "max_value": None}


def test_for_each_device_single():
    t = SingleValueHashTable(4096, layout="soa", key_bits=32, value_bits=32)
    t.insert_bulk([(k, 10 * k) for k in range(1, 1001)])
    q = [5, 2000, 7, 999, 3000]
    k, v, s = t.for_each_device(q)
    assert k.cpu().tolist() == [5, 7, 999] and v.cpu().tolist() == [50, 70, 9990]
    assert s.cpu().tolist() == [t.slot_of(5), t.slot_of(7), t.slot_of(999)]


@pytest.mark.parametrize("layout", ["soa", "packed"])
def test_multi_for_each_slots(layout):
    rng = np.random.default_rng(11)
    n = 30_000
    keys = rng.integers(1, 2000, size=n, dtype=np.uint64)
    vals = np.arange(1, n + 1, dtype=np.uint64)
    t = MultiValueHashTable(int(n / 0.8), layout=layout, key_bits=32, value_bits=32, group_width=8)
    t.insert_bulk(list(zip(keys.tolist(), vals.tolist())))
    q = list(range(1, 2100))
    ks, vs, ss = t.for_each_device(q)
    hkeys, hvals = t._dt.read_slots()
    s = ss.cpu().numpy()
    assert (s >= 0).all()
    assert np.array_equal(hkeys[s].astype(np.uint64), _u(ks))      # each slot holds its key ...
    assert np.array_equal(hvals[s].astype(np.uint64), _u(vs))      # ... and the reported value
    assert len(np.unique(s)) == n                                   # every stored pair exactly once
    off, flat = t.retrieve_bulk(q)
    assert sorted(flat) == sorted(_u(vs).tolist())
    calls = []
    t.for_each([7, 8], lambda k, v, i: calls.append((k, v, i)))
    assert sorted(v for _, v, _ in calls) == sorted(vals[np.isin(keys, [7, 8])].tolist())
    assert all(int(hkeys[i]) == k for k, _, i in calls)
    k2, v2, s2 = t.for_all_device()
    assert k2.numel() == n and len(np.unique(s2.cpu().numpy())) == n


def test_for_all_large_packed():
    n = 1 << 24
    keys = torch.randperm(1 << 30, device="cuda")[:n].to(torch.int32) + 1
    t = SingleValueHashTable(int(n / 0.9), layout="packed", key_bits=32, value_bits=32, group_width=8)
    t.insert_device(keys, keys * 2)
    k, v, s = t.for_all_device()
    assert k.numel() == n
    assert torch.equal(torch.sort(k)[0], torch.sort(keys)[0])
    assert bool((v == k * 2).all()) and bool((s[1:] > s[:-1]).all())


def test_bucket_for_all_device_enumerates_key_store():
    t = BucketListHashTable(256, 4096, key_bits=32, value_bits=32)
    t.insert_bulk([(k % 50 + 1, k) for k in range(1000)])
    k, h, s = t.for_all_device()
    assert sorted(k.cpu().tolist()) == list(range(1, 51))
    from paper_2009_07914_b200 import unpack_handle
    counts = [unpack_handle(int(x) & ((1 << 64) - 1))[1] for x in h.cpu().tolist()]
    assert sum(counts) == 1000
