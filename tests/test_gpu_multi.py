"""GPU parity: multi-value tables (K4-K6) against the reference goldens and the oracle."""
import random
from collections import Counter

import numpy as np
import pytest
import torch

import oracle as orc
from gold import ints, load

pytestmark = pytest.mark.gpu

from paper_2009_07914_b200 import (InsertStatus, MultiValueHashTable,  # noqa: E402
                                   SingleValueHashTable, exclusive_prefix_sum)

INSERTED = InsertStatus.INSERTED


def table_from(sc):
    return MultiValueHashTable(sc["min_capacity"], layout=sc["layout"], key_bits=sc["key_bits"],
                               value_bits=32 if sc["layout"] == "packed" else 64, group_width=sc["group_width"])


@pytest.mark.parametrize("idx", range(5))
def test_sequential_replay_is_slot_exact(idx):
    sc = load("multi.json")["scenarios"][idx]
    t = table_from(sc)
    keys, vals = ints(sc["keys"]), ints(sc["vals"])
    assert [t.insert(k, v).value for k, v in zip(keys, vals)] == sc["status"]
    q = ints(sc["queries"])
    assert t.count_bulk(q) == sc["counts"]
    offsets, flat = t.retrieve_bulk(q)
    assert offsets == sc["offsets"]
    assert flat == ints(sc["flat"])  # probe order, exactly
    assert [t.slots.load_key(i) for i in range(t.capacity)] == ints(sc["final_keys"])
    assert [t.slots.load_value(i) for i in range(t.capacity)] == ints(sc["final_vals"])
    c = t.probe_counters()
    assert (t.occupied, c.ops, c.attempts, c.windows_visited) == \
        (sc["occupied"], sc["counters"]["ops"], sc["counters"]["attempts"], sc["counters"]["windows"])


@pytest.mark.parametrize("idx", range(5))
def test_bulk_replay_multiset_parity(idx):
    sc = load("multi.json")["scenarios"][idx]
    t = table_from(sc)
    keys, vals = ints(sc["keys"]), ints(sc["vals"])
    assert all(s == INSERTED for s in t.insert_bulk(list(zip(keys, vals))))
    q = ints(sc["queries"])
    assert t.count_bulk(q) == sc["counts"]            # counts exact
    offsets, flat = t.retrieve_bulk(q)
    assert offsets == sc["offsets"]                   # offsets exact
    ref = ints(sc["flat"])
    for i in range(len(q)):                           # values: sorted multisets per key
        assert sorted(flat[offsets[i]:offsets[i + 1]]) == sorted(ref[offsets[i]:offsets[i + 1]])


@pytest.mark.parametrize("r,g,layout", [(1, 8, "packed"), (16, 4, "soa"), (16, 8, "packed"), (64, 8, "packed"),
                                        (256, 32, "aos"), (256, 8, "packed"), (4096, 16, "soa")])
def test_large_multiset_vs_oracle(r, g, layout):
    n = 1 << 17
    rng = np.random.default_rng(r * 31 + g)
    keys = rng.integers(1, n // r + 1, size=n, dtype=np.uint64) if r > 1 else \
        rng.permutation(np.arange(1, n + 1, dtype=np.uint64))
    vals = np.arange(1, n + 1, dtype=np.uint64)
    kb = 32
    vb = 32 if layout == "packed" else 64
    t = MultiValueHashTable(int(np.ceil(n / 0.8)), layout=layout, key_bits=kb, value_bits=vb, group_width=g)
    st = t.insert_device(keys, vals).cpu().numpy()
    assert (st == 0).all()
    q = np.arange(1, n + 1, dtype=np.uint64)
    offsets, flat = t.retrieve_device(q)
    offsets = offsets.cpu().numpy()
    flat = flat.cpu().numpy().view(np.uint32 if vb == 32 else np.uint64).astype(np.uint64)
    ref = orc.OracleMulti(int(np.ceil(n / 0.8)), group_width=g, key_bits=kb, packed=layout == "packed")
    ref.insert_bulk(keys, vals)
    roff, rflat = ref.retrieve_bulk(q)
    assert (offsets == roff).all() and offsets[-1] == n
    # per-key sorted multisets: sort within segments via (segment id, value)
    seg = np.repeat(np.arange(n), np.diff(offsets))
    a = np.lexsort((flat, seg))
    b = np.lexsort((rflat, seg))
    assert (flat[a] == rflat[b]).all()


def test_prefix_sum_device_and_host():       # test_multi_table.py:55-66
    assert exclusive_prefix_sum([]) == [0]
    assert exclusive_prefix_sum([2, 0, 3]) == [0, 2, 2, 5]
    rng = np.random.default_rng(79)
    for n in (1, 4095, 4096, 4097, 1 << 20, (1 << 24) + 17):
        counts = rng.integers(0, 10, size=n, dtype=np.int32)
        dev = exclusive_prefix_sum(torch.from_numpy(counts).cuda()).cpu().numpy()
        ref = np.concatenate([[0], np.cumsum(counts, dtype=np.int64)])
        assert (dev == ref).all(), n


def test_reference_semantics():              # test_multi_table.py:19-52,90-96,165-178
    t = MultiValueHashTable(1000)
    assert t.insert(8, 1) == INSERTED and t.insert(8, 2) == INSERTED
    assert t.count(8) == 2 and sorted(t.retrieve(8)) == [1, 2]
    for _ in range(10):
        assert t.insert(3, 3) == INSERTED
    assert t.count(3) == 10
    t2 = MultiValueHashTable(1000)
    t2.insert(1, 10)
    assert t2.retrieve_bulk([999, 1, 998]) == ([0, 0, 1, 1], [10])
    assert t2.retrieve_bulk([]) == ([0], [])
    full = MultiValueHashTable(32)
    for i in range(64):
        assert full.insert(1, i) == INSERTED
    assert full.insert(1, 64) == InsertStatus.TABLE_FULL and full.insert(2, 0) == InsertStatus.TABLE_FULL
    e = t.slots.sentinels.empty_key
    assert t.insert(e, 0) == InsertStatus.INVALID_KEY and t.count(e) == 0 and t.retrieve(e) == []


def test_distinct_keys_match_single_value():  # test_multi_table.py:29-39
    rng = random.Random(71)
    keys = rng.sample(range(1, 1 << 30), 2000)
    multi, single = MultiValueHashTable(4000), SingleValueHashTable(4000)
    for k in keys:
        assert multi.insert(k, k) == single.insert(k, k) == INSERTED
    assert ({k: v for _, k, v in multi.slots.iter_items()} == {k: v for _, k, v in single.slots.iter_items()})


def test_same_key_storm_all_land():          # test_multi_table.py:145-162
    t = MultiValueHashTable(1 << 14, key_bits=32, value_bits=32, layout="packed")
    n = 10_000
    st = t.insert_device(torch.full((n,), 55, dtype=torch.int32, device="cuda"),
                         torch.arange(n, dtype=torch.int32, device="cuda")).cpu().numpy()
    assert (st == 0).all()
    assert t.count(55) == n and sorted(t.retrieve(55)) == list(range(n))


def test_high_multiplicity_completes():      # test_multi_table.py:113-122
    n, r = 1 << 14, 4096
    rng = random.Random(91)
    keys = [rng.randrange(1, n // r + 1) for _ in range(n)]
    t = MultiValueHashTable(int(n / 0.8))
    assert all(s == INSERTED for s in t.insert_bulk(list(zip(keys, range(n)))))
    assert sum(t.count(k) for k in range(1, n // r + 1)) == n
    assert Counter(keys) == Counter({k: t.count(k) for k in range(1, n // r + 1)})


def test_for_each_matches_retrieve_bulk():  # test_multi_table.py:99-110
    t = MultiValueHashTable(2000)
    rng = random.Random(89)
    t.insert_bulk([(rng.randrange(1, 40), i) for i in range(500)])
    queries = list(range(1, 50))
    calls = []
    t.for_each(queries, lambda k, v, i: calls.append((k, v)))
    offsets, flat = t.retrieve_bulk(queries)
    via = [(q, v) for i, q in enumerate(queries) for v in flat[offsets[i]:offsets[i + 1]]]
    assert Counter(calls) == Counter(via)


@pytest.mark.parametrize("layout", ["packed", "soa"])
def test_grouped_insert_zipf_matches_pairwise(layout):
    """Grouped bulk insert (csrc/mgroup.cu: sort by key, one warp per distinct key, hot keys
    first, several windows per step) vs the reference's pair-by-pair order: identical counts
    and per-key value multisets on Zipf keys with groups of thousands of copies."""
    n = 1 << 18
    rng = np.random.default_rng(2009)
    ranks = np.arange(1, 4097, dtype=np.float64)
    p = ranks ** -0.9
    keys = (rng.choice(4096, size=n, p=p / p.sum()) + 1).astype(np.uint64) * 2654435761 % (1 << 31) + 1
    vals = np.arange(1, n + 1, dtype=np.uint64)
    vb = 32 if layout == "packed" else 64
    q = np.unique(keys)
    res = []
    for grouped in (True, False):
        t = MultiValueHashTable(int(np.ceil(n / 0.8)), layout=layout, key_bits=32, value_bits=vb, group_width=8)
        t.set_grouping(grouped)
        st = t.insert_device(keys, vals).cpu().numpy()
        assert (st == 0).all() and t.occupied == n
        offsets, flat = t.retrieve_device(q)
        offsets = offsets.cpu().numpy()
        flat = flat.cpu().numpy().view(np.uint32 if vb == 32 else np.uint64).astype(np.uint64)
        counts = np.diff(offsets)
        true = np.array([np.count_nonzero(keys == k) for k in q[:64]])
        assert (counts[:64] == true).all()
        seg = np.repeat(np.arange(q.size), counts)
        o = np.lexsort((flat, seg))
        res.append((offsets, flat[o]))
    assert (res[0][0] == res[1][0]).all() and (res[0][1] == res[1][1]).all()
    assert res[0][0][-1] == n


def test_hot_chain_cta_walker():
    """A key with tens of thousands of copies walks far more than HUGE_W windows: the warp walker
    hands it to the CTA walker (csrc/multi.cu k_multi_walk_cta, 128 windows per step).  Its count
    is exact and its values come back in probe order (the grouped insert placed copies 1..m in
    sequence order), next to ordinary keys."""
    rng = np.random.default_rng(77)
    m_hot = 60_000
    hot = np.uint64(123456789)
    bg = rng.integers(1, (1 << 31) - 3, size=1 << 20, dtype=np.uint64)
    bg = bg[bg != hot]
    keys = np.concatenate([np.full(m_hot, hot, dtype=np.uint64), bg])
    vals = np.concatenate([np.arange(1, m_hot + 1, dtype=np.uint64), rng.integers(0, 1 << 32, size=bg.size,
                                                                                   dtype=np.uint64)])
    t = MultiValueHashTable(int(np.ceil(keys.size / 0.8)), layout="packed", key_bits=32, value_bits=32,
                            group_width=8)
    st = t.insert_device(keys, vals).cpu().numpy()
    assert (st == 0).all() and t.occupied == keys.size
    q = np.concatenate([np.array([hot], dtype=np.uint64), bg[:5000]])
    offsets, flat = t.retrieve_device(q)
    offsets = offsets.cpu().numpy()
    flat = flat.cpu().numpy().view(np.uint32).astype(np.uint64)
    assert offsets[1] - offsets[0] == m_hot
    assert (flat[: m_hot] == np.arange(1, m_hot + 1, dtype=np.uint64)).all()  # probe order
    counts = np.diff(offsets)[1:]
    u, c = np.unique(bg, return_counts=True)
    want = dict(zip(u.tolist(), c.tolist()))
    assert all(int(counts[i]) == want[int(k)] for i, k in enumerate(bg[:5000]))
    cnt, _ = t.count_device(q)
    assert int(cnt.cpu().numpy()[0]) == m_hot


def _walk_retrieve(t, k, offsets):
    """ch_multi_retrieve over a copy of the keys (another buffer: no stash, a full second walk)."""
    from paper_2009_07914_b200 import _io, _lib
    kc = k.clone()
    total = int(offsets[-1].item())
    vals = torch.zeros(total, dtype=_io.torch_dtype(t.value_bits), device=k.device)
    _lib.check(_lib.lib().ch_multi_retrieve(t._dt.handle, kc.data_ptr(), kc.numel(), offsets.data_ptr(),
                                            vals.data_ptr(), t._stream(None)), "multi retrieve")
    return vals


@pytest.mark.parametrize("layout,kb,vb", [("packed", 32, 32), ("soa", 64, 64)])
def test_retrieve_from_count_stash_is_exact(layout, kb, vb):
    """The retrieve pass copies the count pass's stash for short chains: values in probe order,
    offsets and probe counters identical to walking the sequences again."""
    n = 1 << 16
    rng = np.random.default_rng(7)
    ranks = np.minimum(rng.zipf(1.3, size=n), 1 << 14).astype(np.uint64)  # multiplicities 1 .. thousands
    keys = ranks * np.uint64(2654435761) % np.uint64(1 << 31) + np.uint64(1)
    vals = np.arange(1, n + 1, dtype=np.uint64) * np.uint64(3 if vb == 64 else 1)
    t = MultiValueHashTable(int(np.ceil(n / 0.8)), layout=layout, key_bits=kb, value_bits=vb, group_width=8)
    assert (t.insert_device(keys, vals).cpu().numpy() == 0).all()
    kt = torch.int32 if kb == 32 else torch.int64
    q = torch.from_numpy(np.unique(keys).astype(np.int64)).to(kt).cuda()
    q = torch.cat([q, torch.tensor([12345, 0x7FFFFFF0], dtype=kt, device="cuda")])  # absent keys
    c0 = t.probe_counters()
    offsets, flat = t.retrieve_device(q)                      # count (stash) + retrieve (copy)
    c1 = t.probe_counters()
    _, offsets2 = t.count_device(q)
    flat2 = _walk_retrieve(t, q, offsets2)                    # count + full second walk
    c2 = t.probe_counters()
    assert torch.equal(offsets, offsets2) and int(offsets[-1]) == n
    assert torch.equal(flat, flat2)                           # probe order, exactly
    assert (c1.ops - c0.ops, c1.attempts - c0.attempts, c1.windows_visited - c0.windows_visited) == \
        (c2.ops - c1.ops, c2.attempts - c1.attempts, c2.windows_visited - c1.windows_visited)


def test_count_stash_checks_keys_and_invalidates():
    """A key changed in place between the passes is walked (the stash entry's key differs); any
    other operation on the table between the passes drops the stash."""
    from paper_2009_07914_b200 import _io, _lib
    n = 1 << 14
    keys = np.repeat(np.arange(1, n // 4 + 1, dtype=np.uint64), 4)
    vals = np.arange(1, n + 1, dtype=np.uint64)
    t = MultiValueHashTable(int(np.ceil(n / 0.8)), layout="packed", key_bits=32, value_bits=32, group_width=8)
    t.insert_device(keys, vals)
    q = torch.arange(1, n // 4 + 1, dtype=torch.int32, device="cuda")
    _, offsets = t.count_device(q)
    q[3] = 9                                                  # same count (4), other values
    vals_out = torch.zeros(int(offsets[-1]), dtype=torch.int32, device="cuda")
    _lib.check(_lib.lib().ch_multi_retrieve(t._dt.handle, q.data_ptr(), q.numel(), offsets.data_ptr(),
                                            vals_out.data_ptr(), t._stream(None)), "multi retrieve")
    assert torch.equal(vals_out, _walk_retrieve(t, q, offsets))
    seg = vals_out[offsets[3]:offsets[4]].cpu().numpy()
    assert sorted(seg.tolist()) == list(range(33, 37))        # key 9's values, not key 4's
    # count, then an insert, then retrieve: the stash is gone, the new copy is found
    q2 = torch.arange(1, n // 4 + 1, dtype=torch.int32, device="cuda")
    _, off2 = t.count_device(q2)
    t.insert_device(np.array([1], dtype=np.uint64), np.array([999999], dtype=np.uint64))
    _, off3 = t.count_device(q2)
    v3 = torch.zeros(int(off3[-1]), dtype=torch.int32, device="cuda")
    _lib.check(_lib.lib().ch_multi_retrieve(t._dt.handle, q2.data_ptr(), q2.numel(), off3.data_ptr(),
                                            v3.data_ptr(), t._stream(None)), "multi retrieve")
    assert int(off3[-1]) == int(off2[-1]) + 1 and 999999 in v3[:5].cpu().tolist()
    assert _io is not None


@pytest.mark.parametrize("layout,kb,vb", [("packed", 32, 32), ("soa", 64, 64), ("aos", 32, 64)])
def test_grouped_insert_keeps_batch_order_per_key(layout, kb, vb):
    """The grouping sort (csrc/rsort.cu) is stable, so a key's copies are claimed in batch order
    and come back from retrieve (probe order) exactly in batch order -- what the reference's
    pair-by-pair inserts give (multi_table.py:113-152).  32- and 64-bit keys (4 / 8 sort passes)."""
    n = 1 << 17
    rng = np.random.default_rng(kb + vb)
    ranks = np.arange(1, 2049, dtype=np.float64)
    p = ranks ** -0.8
    base = (rng.choice(2048, size=n, p=p / p.sum()) + 1).astype(np.uint64)
    keys = base * np.uint64(0x9E3779B97F4A7C15 if kb == 64 else 2654435761) % np.uint64((1 << (kb - 1)) - 1) + 1
    vals = rng.integers(0, 1 << (vb - 1), size=n, dtype=np.uint64)
    t = MultiValueHashTable(int(np.ceil(n / 0.8)), layout=layout, key_bits=kb, value_bits=vb, group_width=8)
    assert (t.insert_device(keys, vals).cpu().numpy() == 0).all()
    q = np.unique(keys)
    offsets, flat = t.retrieve_device(q)
    offsets = offsets.cpu().numpy()
    flat = flat.cpu().numpy().view(np.uint32 if vb == 32 else np.uint64).astype(np.uint64)
    order = np.argsort(keys, kind="stable")                 # batch order within each key
    sk = keys[order]
    starts = np.searchsorted(sk, q)
    assert (np.diff(offsets) == np.diff(np.append(starts, n))).all()
    assert (flat == vals[order]).all()                      # q ascending = sk's key order
