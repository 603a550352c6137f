"""GPU parity: bucket-list tables (K7-K9) against the reference goldens and the oracle."""
import random
from collections import Counter

import numpy as np
import pytest

import oracle as orc
from gold import ints, load

pytestmark = pytest.mark.gpu

from paper_2009_07914_b200 import (BucketListHashTable, GrowthPolicy, HandleState,  # noqa: E402
                                   InsertStatus, unpack_handle)

INSERTED = InsertStatus.INSERTED


def table_from(sc):
    return BucketListHashTable(sc["min_keys"], sc["pool"], growth=GrowthPolicy(sc["s0"], sc["factor"]),
                               group_width=sc["group_width"])


@pytest.mark.parametrize("idx", range(6))
def test_sequential_replay_is_arena_exact(idx):
    """One value per batch == the reference's sequential appends: arena, handles,
    chains and head-first retrieval order all match exactly, including pool exhaustion."""
    sc = load("bucket.json")["scenarios"][idx]
    t = table_from(sc)
    keys, vals = ints(sc["keys"]), ints(sc["vals"])
    assert [t.insert(k, v).value for k, v in zip(keys, vals)] == sc["status"]
    q = ints(sc["queries"])
    assert t.count_bulk(q) == sc["counts"]
    offsets, flat = t.retrieve_bulk(q)
    assert offsets == sc["offsets"] and flat == ints(sc["flat"])
    for k, chain in sc["chains"].items():
        assert t.chain_sizes(int(k)) == chain
    assert t.pool.allocated == sc["allocated"]
    assert t.pool.arena[: sc["allocated"]] == ints(sc["arena"])
    assert (t.occupied_keys, t.total_values) == (sc["occupied_keys"], sc["total_values"])
    ks = t.key_store
    assert [ks.slots.load_key(i) for i in range(ks.capacity)] == ints(sc["final_keys"])
    assert [ks.slots.load_value(i) for i in range(ks.capacity)] == ints(sc["final_handles"])
    assert t.storage_density() == pytest.approx(sc["storage_density"], rel=0, abs=0)


@pytest.mark.parametrize("idx", [0, 1, 2, 3, 5])
def test_bulk_replay_multiset_parity(idx):
    sc = load("bucket.json")["scenarios"][idx]
    t = table_from(sc)
    keys, vals = ints(sc["keys"]), ints(sc["vals"])
    assert [s.value for s in t.insert_bulk(list(zip(keys, vals)))] == sc["status"]  # pool suffices
    q = ints(sc["queries"])
    assert t.count_bulk(q) == sc["counts"]
    offsets, flat = t.retrieve_bulk(q)
    assert offsets == sc["offsets"]
    ref = ints(sc["flat"])
    for i in range(len(q)):
        assert sorted(flat[offsets[i]:offsets[i + 1]]) == sorted(ref[offsets[i]:offsets[i + 1]])
    # allocation depends only on the final counts (test_bucket_list.py:174-187)
    assert t.pool.allocated == sc["allocated"]
    for k, chain in sc["chains"].items():
        assert t.chain_sizes(int(k)) == chain


def test_bulk_exhaustion_totals():
    sc = load("bucket.json")["scenarios"][4]  # "exhaust": pool of 300 cells
    t = table_from(sc)
    keys, vals = ints(sc["keys"]), ints(sc["vals"])
    st = t.insert_bulk(list(zip(keys, vals)))
    ins = sum(s == INSERTED for s in st)
    oom = sum(s == InsertStatus.OUT_OF_MEMORY for s in st)
    assert ins + oom == len(keys)
    assert t.total_values == ins and t.pool.allocated <= sc["pool"]
    counts = t.count_bulk(range(0, 25))
    assert sum(counts) == ins
    # values that made it are retrievable and belong to their key
    ref = {}
    for k, v in zip(keys, vals):
        ref.setdefault(k, []).append(v)
    offsets, flat = t.retrieve_bulk(list(range(0, 25)))
    for i, k in enumerate(range(0, 25)):
        seg = flat[offsets[i]:offsets[i + 1]]
        assert not (Counter(seg) - Counter(ref.get(k, [])))


@pytest.mark.parametrize("s0,lam", [(1, "1.1"), (24, "1.0"), (1, "2")])
def test_large_power_law_vs_oracle(s0, lam):
    rng = np.random.default_rng(5)
    m = np.arange(1, 1001)
    p = m ** -1.5
    p /= p.sum()
    mult = rng.choice(m, size=20_000, p=p)
    keys = rng.permutation(np.repeat(np.arange(1, len(mult) + 1, dtype=np.uint64), mult))
    n = len(keys)
    vals = rng.integers(0, 1 << 40, size=n, dtype=np.uint64)
    distinct = len(mult)
    pool = int(n * 2.5) + 64
    t = BucketListHashTable(int(np.ceil(distinct / 0.8)), pool, growth=GrowthPolicy(s0, lam), key_bits=32)
    st = t.insert_device(keys, vals).cpu().numpy()
    assert (st == 0).all()
    ref = orc.OracleBucket(int(np.ceil(distinct / 0.8)), pool, s0=s0, factor=lam, key_bits=32)
    ref.insert_bulk(keys, vals)
    q = np.arange(1, distinct + 3, dtype=np.uint64)
    offsets, flat = t.retrieve_device(q)
    offsets = offsets.cpu().numpy()
    flat = flat.cpu().numpy().view(np.uint64)
    roff, rflat = ref.retrieve_bulk(q)
    assert (offsets == roff).all()
    seg = np.repeat(np.arange(len(q)), np.diff(offsets))
    assert (flat[np.lexsort((flat, seg))] == rflat[np.lexsort((rflat, seg))]).all()
    assert t.pool.allocated == ref.stats()["allocated"]


def test_reference_protocol_cases():         # test_bucket_list.py:124-265
    t = BucketListHashTable(100, 4096, growth=GrowthPolicy(1, 2))
    for v in range(6):
        assert t.insert(10, v) == INSERTED
    assert t.chain_sizes(10) == [1, 2, 4] and t.count(10) == 6
    assert sorted(t.retrieve(10)) == list(range(6))
    t2 = BucketListHashTable(100, 4096)
    t2.insert(4, 40)
    state, count, _ = unpack_handle(t2.key_store.slots.load_value(t2.key_store.slot_of(4)))
    assert state == HandleState.READY and count == 1
    assert t2.retrieve(404) == [] and t2.count(404) == 0
    ex = BucketListHashTable(100, 4, growth=GrowthPolicy(1, 2))
    assert [ex.insert(1, v) for v in (10, 11, 12)] == [INSERTED] * 3
    assert ex.insert(1, 13) == InsertStatus.OUT_OF_MEMORY and ex.insert(1, 14) == InsertStatus.OUT_OF_MEMORY
    state, count, _ = unpack_handle(ex.key_store.slots.load_value(ex.key_store.slot_of(1)))
    assert state == HandleState.FULL and count == 3 and sorted(ex.retrieve(1)) == [10, 11, 12]
    pk = BucketListHashTable(100, 5, growth=GrowthPolicy(1, 2))
    pk.insert(1, 0)
    pk.insert(1, 1)
    assert pk.insert(1, 2) == INSERTED and pk.insert(1, 3) == InsertStatus.OUT_OF_MEMORY
    assert pk.insert(2, 99) == INSERTED and pk.retrieve(2) == [99]
    ksf = BucketListHashTable(32, 1000)
    for k in range(1, 65):
        assert ksf.insert(k, k) == INSERTED
    assert ksf.insert(999, 1) == InsertStatus.TABLE_FULL
    e = ksf.key_store.slots.sentinels.empty_key
    assert ksf.insert(e, 1) == InsertStatus.INVALID_KEY
    ob = BucketListHashTable(100, 1000)
    for k, n in ((1, 3), (2, 2), (3, 1)):
        for i in range(n):
            ob.insert(k, 10 * k + i)
    offsets, flat = ob.retrieve_bulk([1, 2, 3])
    assert offsets == [0, 3, 5, 6] and flat == [v for k in (1, 2, 3) for v in ob.retrieve(k)]
    assert ob.retrieve_bulk([]) == ([0], [])


def test_same_key_appends_and_quiescent_handles():  # test_bucket_list.py:190-228, acceptance 7
    total = 10_000
    for _ in range(3):
        t = BucketListHashTable(64, 4 * total, growth=GrowthPolicy(1, "1.1"))
        st = t.insert_bulk([(99, v) for v in range(total)])
        assert all(s == INSERTED for s in st)
        assert t.count(99) == total and sorted(t.retrieve(99)) == list(range(total))
    t = BucketListHashTable(500, 50_000)
    rng = random.Random(3)
    t.insert_bulk([(rng.randrange(1, 64), i) for i in range(16_000)])
    for _, _, word in t.key_store.slots.iter_items():
        assert unpack_handle(word)[0] in (HandleState.READY, HandleState.FULL)


def test_exact_policy_maximizes_density():   # test_bucket_list.py:306-319
    r, keys = 8, list(range(1, 65))
    dens = {}
    for name, (s0, lam) in {"exact": (r, "1.0"), "default": (1, "1.1"), "doubling": (1, "2.0")}.items():
        t = BucketListHashTable(100, 4096, growth=GrowthPolicy(s0, lam))
        t.insert_bulk([(k, i) for k in keys for i in range(r)])
        dens[name] = t.storage_density()
    assert dens["exact"] == max(dens.values())


def test_blocked_handle_raises_contention_timeout():
    """A handle left BLOCKED (bucket_list.py:300-318) never becomes ready; the walk flags it
    and the list API raises ContentionTimeout, like the reference after its retry budget."""
    from paper_2009_07914_b200 import ContentionTimeout, pack_handle
    t = BucketListHashTable(64, 256, key_bits=32, value_bits=32)
    t.insert_bulk([(5, 50), (5, 51), (9, 90)])
    assert sorted(t.retrieve(5)) == [50, 51]
    slot = t.key_store.slot_of(5)
    t.slots.store_value(slot, pack_handle(1, 2, 0))   # BLOCKED, count 2
    assert t.retrieve(9) == [90]                        # other keys are unaffected
    with pytest.raises(ContentionTimeout):
        t.retrieve_bulk([5, 9])
