"""GPU parity: single-value tables (K0-K3) against the reference goldens and the oracle.

Sequential (element-at-a-time) replays must reproduce the reference's slot
placement, statuses, probe statistics and counters exactly; bulk batches run
concurrently on the GPU and are checked for the reference's semantics
(SURVEY.md §8c): exact statuses for distinct keys, one INSERTED per new key,
bit-exact values and found flags.
"""
import zlib
from collections import Counter

import numpy as np
import pytest
import torch

import oracle as orc
from gold import STATUS_NAMES, ints, load

pytestmark = pytest.mark.gpu

from paper_2009_07914_b200 import (InsertStatus, LayoutKind, SingleValueHashTable,  # noqa: E402
                                   probing)

INSERTED, DUP = InsertStatus.INSERTED, InsertStatus.DUPLICATE_KEY


def table_from(sc):
    e, t = int(sc["empty"]), int(sc["tomb"])
    from paper_2009_07914_b200 import Sentinels
    return SingleValueHashTable(sc["min_capacity"], layout=sc["layout"], key_bits=sc["key_bits"],
                                value_bits=32 if sc["layout"] == "packed" else 64,
                                group_width=sc["group_width"], max_outer_attempts=sc["max_outer_attempts"],
                                sentinels=Sentinels(e, t))


# ------------------------------------------------ sequential replay: slot-exact

@pytest.mark.parametrize("idx", range(11))
def test_sequential_replay_is_slot_exact(idx):
    sc = load("single.json")["scenarios"][idx]
    t = table_from(sc)
    assert t.capacity == sc["capacity"]
    for step in sc["steps"]:
        if step["op"] == "insert_bulk":
            got = [t.insert(k, v).value for k, v in zip(ints(step["keys"]), ints(step["vals"]))]
            assert got == step["status"]
        elif step["op"] == "erase":
            assert [t.erase(k) for k in ints(step["keys"])] == step["result"]
        elif step["op"] == "retrieve_bulk":
            got = t.retrieve_bulk(ints(step["keys"]))
            assert got == [None if r is None else int(r) for r in step["result"]]
        elif step["op"] == "stats":
            for key, att, win, slot in step["probe"]:
                _, stats = t.retrieve_with_stats(int(key))
                assert (stats.attempts, stats.windows_visited) == (att, win), key
                assert t.slot_of(int(key)) == slot, key
    keys = [t.slots.load_key(i) for i in range(t.capacity)]
    vals = [t.slots.load_value(i) for i in range(t.capacity)]
    assert keys == ints(sc["final_keys"])
    assert vals == ints(sc["final_vals"])
    assert (t.occupied, t.tombstones) == (sc["occupied"], sc["tombstones"])
    c = t.probe_counters()
    assert (c.ops, c.attempts, c.windows_visited) == \
        (sc["counters"]["ops"], sc["counters"]["attempts"], sc["counters"]["windows"])


# ------------------------------------------------ bulk replay: semantic parity

@pytest.mark.parametrize("loc", ["off", "on", "staged"])
@pytest.mark.parametrize("idx", range(11))
def test_bulk_replay_semantics(idx, loc):
    sc = load("single.json")["scenarios"][idx]
    t = table_from(sc)
    t.set_locality(loc)
    model: dict[int, int] = {}
    any_full = False
    for step in sc["steps"]:
        if step["op"] == "insert_bulk":
            keys, vals = ints(step["keys"]), ints(step["vals"])
            got = t.insert_bulk(list(zip(keys, vals)))
            ref = step["status"]
            any_full |= "table_full" in ref or InsertStatus.TABLE_FULL in got
            mult = Counter(keys)
            winners = {}
            for k, v, g, r in zip(keys, vals, got, ref):
                if r == "invalid_key":
                    assert g == InsertStatus.INVALID_KEY
                elif mult[k] == 1 and not any_full:
                    assert g.value == r, k  # distinct keys: exact status
                if g == INSERTED:
                    assert k not in winners, "two INSERTED for one key"
                    winners[k] = v
            if not any_full:
                new_keys = {k for k, r in zip(keys, ref) if r == "inserted"}
                assert set(winners) == new_keys, "new keys must be inserted exactly once"
            model.update(winners)
        elif step["op"] == "erase":
            keys = ints(step["keys"])
            er = t.erase_device(keys).cpu().numpy().astype(bool).tolist()
            # a key listed twice is retired once, by either position
            assert Counter(k for k, hit in zip(keys, er) if hit) == \
                Counter(k for k, hit in zip(keys, step["result"]) if hit) or any_full
            for k, hit in zip(keys, er):
                if hit:
                    model.pop(k)
        elif step["op"] == "retrieve_bulk":
            keys = ints(step["keys"])
            assert t.retrieve_bulk(keys) == [model.get(k) for k in keys]
    assert {k: v for _, k, v in t.slots.iter_items()} == model
    if not any_full:
        assert t.occupied == sc["occupied"]


# ------------------------------------------------ large batches vs the oracle

@pytest.mark.parametrize("layout,kb,vb,g", [
    ("packed", 32, 32, 1), ("packed", 32, 32, 2), ("packed", 32, 32, 4), ("packed", 32, 32, 8),
    ("packed", 32, 32, 16), ("packed", 32, 32, 32),
    ("soa", 64, 64, 4), ("soa", 32, 64, 8), ("soa", 64, 32, 16), ("soa", 32, 32, 32),
    ("aos", 64, 64, 8), ("aos", 32, 32, 4), ("aos", 32, 64, 2), ("aos", 64, 32, 1),
])
@pytest.mark.parametrize("rho,loc", [(0.8, "auto"), (0.95, "auto"), (0.95, "on"), (0.8, "staged"),
                                     (0.95, "staged")])
def test_bulk_unique_vs_oracle(layout, kb, vb, g, rho, loc):
    n = 1 << 18
    rng = np.random.default_rng(zlib.crc32(f"{layout}{kb}{vb}{g}{rho}{loc}".encode()))
    hi = (1 << kb) - 3
    keys = rng.permutation(np.unique(rng.integers(1, hi, size=3 * n, dtype=np.uint64)))
    present, absent = keys[:n], keys[n:2 * n]
    vals = rng.integers(0, (1 << vb) - 1, size=n, dtype=np.uint64)
    cap = int(np.ceil(n / rho))
    t = SingleValueHashTable(cap, layout=layout, key_bits=kb, value_bits=vb, group_width=g)
    t.set_locality(loc)
    st = t.insert_device(present, vals).cpu().numpy()
    assert (st == 0).all()
    assert t.occupied == n
    v, f = t.retrieve_device(present)
    assert f.cpu().numpy().all()
    got = v.cpu().numpy().view(np.uint32 if vb <= 32 else np.uint64).astype(np.uint64)
    assert (got == vals).all()
    v2, f2 = t.retrieve_device(absent)
    assert not f2.cpu().numpy().any()
    assert (v2.cpu().numpy() == 0).all()
    # re-inserting is all duplicates and leaves the values untouched
    st2 = t.insert_device(present, vals ^ np.uint64(1)).cpu().numpy()
    assert (st2 == 1).all()
    # the oracle agrees on occupancy and the hit/miss sets
    ref = orc.OracleSingle(cap, group_width=g, key_bits=kb, packed=layout == "packed")
    ref.insert_bulk(present, vals)
    assert ref.stats()["occupied"] == t.occupied
    rv, rf = ref.retrieve_bulk(present[:4096])
    assert (rv == got[:4096]).all() and rf.all()


def test_retrieve_probe_counts_match_oracle_readonly():
    """Read-only probes are schedule independent: mean attempts equal the oracle's."""
    n = 1 << 16
    rng = np.random.default_rng(3)
    keys = rng.permutation(np.unique(rng.integers(1, (1 << 32) - 3, size=2 * n, dtype=np.uint64)))[:n]
    for g in (1, 4, 32):
        t = SingleValueHashTable(int(n / 0.9), layout="packed", key_bits=32, value_bits=32, group_width=g)
        ref = orc.OracleSingle(int(n / 0.9), group_width=g, key_bits=32, packed=True)
        # sequentially-equivalent placement: insert the oracle's final state directly
        ref.insert_bulk(keys, keys)
        rk, rvals = ref.dump()
        t._dt  # noqa: B018
        from paper_2009_07914_b200 import _lib
        k32 = rk.astype(np.uint32)
        v32 = rvals.astype(np.uint32)
        _lib.check(_lib.lib().ch_write_slots(t._dt.handle, k32.ctypes.data, v32.ctypes.data))
        t._dt.touch()
        before = ref.stats()
        t.reset_probe_counters()
        t.retrieve_device(keys)
        ref.retrieve_bulk(keys)
        after = ref.stats()
        c = t.probe_counters()
        assert c.ops == after["ops"] - before["ops"]
        assert c.attempts == after["attempts"] - before["attempts"]
        assert c.windows_visited == after["windows"] - before["windows"]


# ------------------------------------------------ reference test_single_table.py mirrors

def _table(min_capacity=1000, **kw):
    return SingleValueHashTable(min_capacity, **kw)


def test_singleton_and_duplicate():          # test_single_table.py:19-31
    t = _table()
    assert t.insert(5, 50) == INSERTED
    assert t.retrieve(5) == 50 and t.occupied == 1
    assert t.insert(5, 51) == DUP and t.retrieve(5) == 50


def test_invalid_key_rejected():             # :34-40
    t = _table()
    e = t.slots.sentinels.empty_key
    assert t.insert(e, 1) == InsertStatus.INVALID_KEY
    assert t.insert(t.slots.sentinels.tombstone_key, 1) == InsertStatus.INVALID_KEY
    assert t.retrieve(e) is None and not t.erase(e)


def test_fill_to_high_density():             # :43-50
    t = _table(1000)
    n = int(t.capacity * 0.97)
    st = t.insert_bulk([(k, k + 1) for k in range(1, n + 1)])
    assert all(s == INSERTED for s in st)
    assert t.retrieve_bulk(range(1, n + 1)) == [k + 1 for k in range(1, n + 1)]
    assert t.load_factor() == n / t.capacity


def test_absent_key_stops_after_first_window():  # :53-58
    t = _table()
    value, stats = t.retrieve_with_stats(12345)
    assert value is None and stats.windows_visited == 1 and stats.attempts >= 1


def test_erase_semantics():                  # :61-85
    t = _table()
    assert not t.erase(4)
    t.insert(4, 44)
    assert t.erase(4) and not t.erase(4)
    assert t.retrieve(4) is None
    t.insert(6, 60)
    before, slot = t.occupied, t.slot_of(6)
    assert t.erase(6)
    assert t.insert(6, 61) == INSERTED
    assert t.occupied == before and t.slot_of(6) == slot and t.retrieve(6) == 61


def _colliding_pair(table):
    cfg = table.config
    seen = {}
    for key in range(1, 1 << 20):
        start = cfg.hash.value(key) % cfg.plan.c
        if start in seen:
            return seen[start], key
        seen[start] = key
    raise AssertionError


def test_tombstone_cases():                  # :101-124
    t = _table()
    k1, k2 = _colliding_pair(t)
    t.insert(k1, 100)
    t.erase(k1)
    assert t.insert(k2, 200) == INSERTED and t.retrieve(k2) == 200
    assert sum(1 for _, k, _ in t.slots.iter_items() if k == k2) == 1
    t2 = _table()
    t2.insert(k1, 1)
    t2.insert(k2, 2)
    t2.erase(k1)
    assert t2.insert(k2, 3) == DUP and t2.retrieve(k2) == 2
    # same in one concurrent batch: the duplicate behind the tombstone is still found
    assert t2.insert_bulk([(k2, 4)] * 64) == [DUP] * 64


def test_lowest_index_placement():           # :127-142
    import random
    t = _table(3000)
    rng = random.Random(41)
    keys = rng.sample(range(1, 1 << 30), 2000)
    t.insert_bulk([(k, k) for k in keys])  # concurrent: still no empty before any key
    e = t.slots.sentinels.empty_key
    for k in rng.sample(keys, 200):
        for idx in probing.probe_order(k, t.config):
            cell = t.slots.load_key(idx)
            if cell == k:
                break
            assert cell != e
        else:
            raise AssertionError


@pytest.mark.parametrize("layout,key_bits,ops", [(LayoutKind.SOA, 64, 3000), (LayoutKind.AOS, 64, 2000),
                                                 (LayoutKind.PACKED_AOS, 32, 2000)])
def test_oracle_equivalence_random_ops(layout, key_bits, ops):   # :145-175
    import random
    t = SingleValueHashTable(256, layout=layout, key_bits=key_bits,
                             value_bits=32 if layout == LayoutKind.PACKED_AOS else 64)
    domain = int(t.capacity * 0.7)
    rng = random.Random(97)
    ref = {}
    for step in range(ops):
        key = rng.randrange(1, domain)
        roll = rng.random()
        if roll < 0.5:
            value = rng.randrange(1, 1 << 30)
            st = t.insert(key, value)
            assert st == (DUP if key in ref else INSERTED), step
            ref.setdefault(key, value)
        elif roll < 0.8:
            assert t.retrieve(key) == ref.get(key), step
        else:
            assert t.erase(key) == (ref.pop(key, None) is not None), step
    assert {k: v for _, k, v in t.slots.iter_items()} == ref
    assert t.occupied == len(ref)


def test_in_batch_duplicates():              # :190-197
    t = _table(1000)
    st = t.insert_bulk([(5, 1), (6, 2), (5, 3), (5, 4), (6, 5)])
    assert st.count(INSERTED) == 2 and st.count(DUP) == 3
    assert t.retrieve(5) in (1, 3, 4) and t.retrieve(6) in (2, 5)


@pytest.mark.parametrize("loc", ["off", "on", "staged"])
def test_same_key_storm_single_winner(loc):  # :278-298 (8 threads -> 1M lanes)
    t = SingleValueHashTable(256, layout="packed", key_bits=32, value_bits=32)
    t.set_locality(loc)
    n = 1 << 20
    keys = torch.full((n,), 777, dtype=torch.int32, device="cuda")
    vals = torch.arange(n, dtype=torch.int32, device="cuda")
    st = t.insert_device(keys, vals).cpu().numpy()
    assert (st == 0).sum() == 1 and (st == 1).sum() == n - 1
    assert t.retrieve(777) == int(np.nonzero(st == 0)[0][0])
    assert t.occupied == 1


def test_empty_and_load_factor():            # :200-231
    t = _table(1000)
    assert t.insert_bulk([]) == [] and t.retrieve_bulk([]) == []
    assert t.load_factor() == 0.0
    t.insert_bulk([(k, k) for k in range(1, 11)])
    assert t.load_factor() == 10 / t.capacity
    t.erase(1)
    assert t.load_factor() == 9 / t.capacity and t.tombstones == 1


def test_table_full_after_whole_cycle():     # :234-239
    t = _table(32)
    for k in range(1, 65):
        assert t.insert(k, k) == INSERTED
    assert t.insert(999, 1) == InsertStatus.TABLE_FULL
    assert t.load_factor() == 1.0
    b = _table(32)
    st = b.insert_bulk([(k, k) for k in range(1, 66)])
    assert st.count(INSERTED) == 64 and st.count(InsertStatus.TABLE_FULL) == 1


def test_group_widths_agree_on_final_state():  # :242-252
    import random
    rng = random.Random(61)
    keys = rng.sample(range(1, 1 << 30), 500)
    views = []
    for g in (1, 2, 4, 8, 16, 32):
        t = _table(1000, group_width=g)
        for k in keys:
            t.insert(k, k + 1)
        t.erase(keys[0])
        views.append({k: v for _, k, v in t.slots.iter_items()})
    assert all(v == views[0] for v in views)


def test_for_each_and_for_all():             # :206-220
    t = _table()
    items = {k: k * 7 for k in range(1, 101)}
    t.insert_bulk(list(items.items()))
    seen = {}
    t.for_all(lambda k, v, i: seen.__setitem__(k, v))
    assert seen == items
    hits = []
    t.for_each([1, 2, 999_999], lambda k, v, i: hits.append((k, v)))
    assert hits == [(1, 7), (2, 14)]


def test_find_or_claim():
    t = _table()
    st, slot = t.find_or_claim(42)
    assert st == INSERTED and slot == t.slot_of(42)
    st2, slot2 = t.find_or_claim(42)
    assert st2 == DUP and slot2 == slot


def test_locality_path_at_scale_matches_direct():
    """2^24 keys in a 128 MiB+ table: region-ordered and direct execution agree bit for bit."""
    n = 1 << 24
    rng = np.random.default_rng(11)
    keys = torch.from_numpy(rng.permutation(np.unique(rng.integers(1, (1 << 32) - 3, size=n + n // 4,
                                                                   dtype=np.uint64)))[:n].astype(np.uint32)
                            .view(np.int32)).cuda()
    vals = torch.arange(n, dtype=torch.int32, device="cuda")
    out = []
    for loc in ("off", "on", "staged"):
        t = SingleValueHashTable(int(n / 0.95), layout="packed", key_bits=32, value_bits=32, group_width=8)
        t.set_locality(loc)
        st = t.insert_device(keys, vals)
        assert (st == 0).all().item() and t.occupied == n
        dup = keys[: n // 2]
        st2 = t.insert_device(dup, vals[: n // 2])
        assert (st2 == 1).all().item()
        v, f = t.retrieve_device(keys)
        assert f.bool().all().item() and (v == vals).all().item()
        miss = keys[: 1 << 20] ^ 0x5A5A5A5A
        out.append(t.retrieve_device(miss))
    for o in out[1:]:
        assert torch.equal(out[0][1], o[1]) and torch.equal(out[0][0], o[0])


@pytest.mark.parametrize("rho", [0.8, 0.95, 0.99])
def test_staged_path_mixed_batches_vs_oracle(rho):
    """Staged regions (csrc/staged.cu) on batches mixing new keys, in-batch duplicates,
    keys already present, sentinels and tombstones: statuses, values and found flags
    against the oracle's sequential semantics for the distinct-key parts."""
    n = 1 << 20
    rng = np.random.default_rng(int(rho * 100))
    pool = rng.permutation(np.unique(rng.integers(1, (1 << 32) - 3, size=3 * n, dtype=np.uint64)))
    first, second, absent = pool[:n // 2], pool[n // 2:n], pool[n:2 * n]
    cap = int(np.ceil(n / rho))
    t = SingleValueHashTable(cap, layout="packed", key_bits=32, value_bits=32, group_width=8)
    t.set_locality("staged")
    v1 = rng.integers(0, 1 << 32, size=first.size, dtype=np.uint64)
    st = t.insert_device(first, v1).cpu().numpy()
    assert (st == 0).all() and t.occupied == first.size
    # erase a quarter: tombstones in front of later keys' first empties
    gone = first[: first.size // 4]
    er = t.erase_device(gone).cpu().numpy()
    assert er.all() and t.tombstones == gone.size
    # batch: second half new keys (+ a duplicated tail), old keys again, sentinels
    dup = second[: 4096]
    keys = np.concatenate([second, dup, first[first.size // 4:first.size // 4 + 8192],
                           np.array([(1 << 32) - 1, (1 << 32) - 2], dtype=np.uint64)])
    perm = rng.permutation(keys.size)
    keys = keys[perm]
    vals = rng.integers(0, 1 << 32, size=keys.size, dtype=np.uint64)
    st = t.insert_device(keys, vals).cpu().numpy()
    inv = keys >= (1 << 32) - 2
    assert (st[inv] == 3).all()
    ins = st == 0
    ks, cnt = np.unique(keys[ins], return_counts=True)
    assert (cnt == 1).all(), "two INSERTED for one key"
    assert set(ks.tolist()) == set(second.tolist())
    old = np.isin(keys, first)
    assert (st[old] == 1).all()
    winner = dict(zip(keys[ins].tolist(), vals[ins].tolist()))
    model = dict(zip(first[first.size // 4:].tolist(), v1[first.size // 4:].tolist()))
    model.update(winner)
    assert t.occupied == len(model)
    q = np.concatenate([np.array(list(model.keys()), dtype=np.uint64), gone, absent[: n // 2]])
    q = q[rng.permutation(q.size)]
    v, f = t.retrieve_device(q)
    v = v.cpu().numpy().view(np.uint32).astype(np.uint64)
    f = f.cpu().numpy().astype(bool)
    want_f = np.isin(q, np.array(list(model.keys()), dtype=np.uint64))
    assert (f == want_f).all()
    want_v = np.array([model.get(int(k), 0) for k in q[f]], dtype=np.uint64)
    assert (v[f] == want_v).all() and (v[~f] == 0).all()
    # the staged lookup agrees with the direct one bit for bit
    t.set_locality("off")
    dv, df = t.retrieve_device(q)
    assert (dv.cpu().numpy().view(np.uint32).astype(np.uint64) == v).all()
    assert (df.cpu().numpy().astype(bool) == f).all()


def test_staged_counters_match_direct_readonly():
    """Read-only staged lookups count ops / attempts / windows exactly like direct probes."""
    n = 1 << 20
    rng = np.random.default_rng(5)
    keys = rng.permutation(np.unique(rng.integers(1, (1 << 32) - 3, size=2 * n, dtype=np.uint64)))
    present, absent = keys[:n], keys[n:2 * n]
    t = SingleValueHashTable(int(n / 0.95), layout="packed", key_bits=32, value_bits=32, group_width=4)
    t.insert_device(present, present)
    q = np.concatenate([present, absent])
    res = []
    for loc in ("off", "staged"):
        t.set_locality(loc)
        t.reset_probe_counters()
        t.retrieve_device(q)
        c = t.probe_counters()
        res.append((c.ops, c.attempts, c.windows_visited))
    assert res[0] == res[1]


def test_host_pipeline_matches_device_path():
    """insert_host / retrieve_host (chunked H2D / kernel / D2H overlap) == the device API."""
    n = (1 << 22) + 12345
    rng = np.random.default_rng(21)
    keys = rng.permutation(np.unique(rng.integers(1, (1 << 32) - 3, size=n + n // 4, dtype=np.uint64)))[:n]
    vals = rng.integers(0, 1 << 32, size=n, dtype=np.uint64)
    t = SingleValueHashTable(int(n / 0.9), layout="packed", key_bits=32, value_bits=32, group_width=8)
    st = t.insert_host(keys, vals, chunk=1 << 20)
    assert (st.numpy() == 0).all() and t.occupied == n
    st2 = t.insert_host(keys[:1000], vals[:1000], chunk=300)
    assert (st2.numpy() == 1).all()
    v, f = t.retrieve_host(np.concatenate([keys, keys[:10] ^ np.uint64(0xFFFF)]), chunk=1 << 19)
    v = v.numpy().view(np.uint32)
    f = f.numpy()
    assert f[:n].all() and (v[:n] == vals.astype(np.uint32)).all()
    dv, df = t.retrieve_device(keys[:4096])
    assert (dv.cpu().numpy().view(np.uint32) == v[:4096]).all()
    # async insert_host then retrieve_host, repeatedly through the same staging buffers
    from paper_2009_07914_b200 import _lib
    import torch
    for rep in range(3):
        _lib.check(_lib.lib().ch_clear(t._dt.handle, torch.cuda.current_stream().cuda_stream))
        kk = keys[rep::3]
        vv = (vals[rep::3] + rep) % (1 << 32)
        st = t.insert_host(kk, vv, chunk=1 << 18, sync=False)
        v, f = t.retrieve_host(kk, chunk=1 << 18)
        assert (st.numpy() == 0).all() and f.numpy().all()
        assert (v.numpy().view(np.uint32) == vv.astype(np.uint32)).all()


@pytest.mark.parametrize("switches", [{"CH_STAGED_ROUND2": "1", "CH_STAGED_FB_CTAS": "1"},
                                      {"CH_STAGED_COUNT": "1"}])
def test_staged_round2_and_fallback_caps_match_direct(tmp_path, switches):
    """The optional staged window-1 round (CH_STAGED_ROUND2=1), a capped COPS pass
    (CH_STAGED_FB_CTAS=1) and the count-based partition (CH_STAGED_COUNT=1, the path of
    batches >= 2^30 keys) give the same statuses / values / found flags as direct probes
    (run in a child process: the switches are read when the library loads)."""
    import subprocess
    import sys
    script = tmp_path / "r2.py"
    script.write_text(
        "import sys, numpy as np, torch\n"
        f"sys.path.insert(0, {str(__import__('os').getcwd())!r})\n"
        "from paper_2009_07914_b200 import SingleValueHashTable\n"
        "n = 1 << 20\n"
        "rng = np.random.default_rng(77)\n"
        "pool = rng.permutation(np.unique(rng.integers(1, (1 << 32) - 3, size=3 * n, dtype=np.uint64)))\n"
        "keys, absent = pool[:n], pool[n:2 * n]\n"
        "vals = rng.integers(0, 1 << 32, size=n, dtype=np.uint64)\n"
        "out = []\n"
        "for loc in ('staged', 'off'):\n"
        "    t = SingleValueHashTable(int(n / 0.97), layout='packed', key_bits=32, value_bits=32, group_width=8)\n"
        "    t.set_locality(loc)\n"
        "    st = t.insert_device(keys, vals).cpu().numpy()\n"
        "    q = np.concatenate([keys, absent])\n"
        "    v, f = t.retrieve_device(q)\n"
        "    out.append((st, v.cpu().numpy(), f.cpu().numpy(), t.occupied))\n"
        "a, b = out\n"
        "assert (a[0] == 0).all() and (b[0] == 0).all() and a[3] == b[3] == n\n"
        "assert (a[1] == b[1]).all() and (a[2] == b[2]).all() and a[2][:n].all() and not a[2][n:].any()\n"
        "print('ok')\n")
    import os
    env = dict(os.environ, **switches)
    r = subprocess.run([sys.executable, str(script)], env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and "ok" in r.stdout, r.stdout + r.stderr


@pytest.mark.parametrize("min_cap", [(1 << 31) - (1 << 20), (1 << 31) + (1 << 20)])
def test_probe_start_matches_reference_hash_at_2g_slots(min_cap):
    """Window starts h = mix64(k) mod c on both sides of c = 2^31 (the device takes a
    32-bit remainder below 2^31, probing.py HashFn(0) % c): in a sparse table almost every
    key sits at h, and every key sits inside window 0."""
    from paper_2009_07914_b200.probing import mix64
    t = SingleValueHashTable(min_cap, layout="packed", key_bits=32, value_bits=32, group_width=8)
    c = t.capacity
    assert (c < (1 << 31)) == (min_cap < (1 << 31))
    rng = np.random.default_rng(11)
    keys = np.unique(rng.integers(1, (1 << 32) - 2, size=200_000, dtype=np.uint64)).astype(np.uint32)
    kt = torch.from_numpy(keys.view(np.int32)).cuda()
    assert (t.insert_device(kt, kt).cpu() == 0).all()
    slots, _, _, _ = t.find_device(kt)
    slots = slots.cpu().numpy()
    h = np.array([mix64(int(k)) % c for k in keys], dtype=np.int64)
    off = (slots - h) % c
    assert (off < 32).all()
    assert (off == 0).mean() > 0.99
    del t
    torch.cuda.empty_cache()


@pytest.mark.parametrize("skew", ["super", "region"])
def test_staged_overflowing_partition_areas(skew):
    """Skewed batches overflow the staged schedule's fixed partition areas (csrc/staged.cu,
    Part): a super-region holding most of the batch re-runs the exact level-1 partition,
    and over-full regions hand their runs to the COPS kernels.  Statuses, values and
    found flags match the direct probes."""
    from paper_2009_07914_b200.probing import mix64_array
    rng = np.random.default_rng(3 if skew == "super" else 4)
    cap = 4_300_000
    t = SingleValueHashTable(cap, layout="packed", key_bits=32, value_bits=32, group_width=8)
    c = t.capacity
    cand = np.unique(rng.integers(1, (1 << 32) - 3, size=12_000_000, dtype=np.uint64))
    h = mix64_array(cand) % np.uint64(c)
    if skew == "super":  # 90 % of the batch in super-region 0 (regions 0..255)
        hot = cand[(h >> np.uint64(21)) == 0][:900_000]
    else:  # three regions over-full, the rest uniform
        hot = cand[np.isin(h >> np.uint64(13), [5, 6, 300])][:24_000]
    cold = rng.permutation(cand[(h >> np.uint64(21)) != 0])[:100_000]
    keys = np.concatenate([hot, cold, hot[:5000]])  # + in-batch duplicates
    keys = keys[rng.permutation(keys.size)]
    vals = rng.integers(0, 1 << 32, size=keys.size, dtype=np.uint64)
    ref = SingleValueHashTable(cap, layout="packed", key_bits=32, value_bits=32, group_width=8)
    ref.set_locality("off")
    t.set_locality("staged")
    st, st_ref = t.insert_device(keys, vals).cpu().numpy(), ref.insert_device(keys, vals).cpu().numpy()
    assert t.occupied == ref.occupied == np.unique(keys).size
    u, cnt = np.unique(keys, return_counts=True)
    single = np.isin(keys, u[cnt == 1])
    assert (st[single] == 0).all() and (st_ref[single] == 0).all()
    ins = keys[st == 0]
    assert np.unique(ins).size == ins.size == u.size  # every key inserted exactly once
    absent = np.setdiff1d(cand[:200_000], keys)[:50_000]
    q = np.concatenate([keys, absent])
    v, f = t.retrieve_device(q)
    vr, fr = ref.retrieve_device(q)
    f, fr = f.cpu().numpy(), fr.cpu().numpy()
    assert (f == fr).all() and f[:keys.size].all() and not f[keys.size:].any()
    # values: the winner's value per key; both tables hold a value of one of the key's copies
    vv = v.cpu().numpy().view(np.uint32)[:keys.size]
    got = dict(zip(keys[single].tolist(), vv[single].tolist()))
    want = dict(zip(keys[single].tolist(), vals[single].astype(np.uint32).tolist()))
    assert got == want


@pytest.mark.parametrize("rho", [0.9, 0.97])
def test_staged_misses_and_erase_vs_direct(rho):
    """Misses (absent keys walk until an empty, mostly past window 0 at high load) through
    the fingerprint kernels agree with the word-scanning direct kernels on the same table
    -- values, found flags and probe counters -- before and after an erase."""
    n = 1 << 20
    rng = np.random.default_rng(int(rho * 1000))
    pool = rng.permutation(np.unique(rng.integers(1, (1 << 32) - 3, size=3 * n, dtype=np.uint64)))
    present, absent = pool[:n], pool[n:2 * n]
    t = SingleValueHashTable(int(n / rho), layout="packed", key_bits=32, value_bits=32, group_width=8)
    t.set_locality("staged")
    t.insert_device(present, present ^ np.uint64(7))
    q = np.concatenate([absent, present[::3]])

    def both(keys):
        out = []
        for mode in ("staged", "off"):
            t.set_locality(mode)
            t.reset_probe_counters()
            v, f = t.retrieve_device(keys)
            c = t.probe_counters()
            out.append((v.cpu().numpy(), f.cpu().numpy(), (c.ops, c.attempts, c.windows_visited)))
        return out

    a, b = both(q)
    for x, y in zip(a, b):
        assert np.array_equal(np.asarray(x), np.asarray(y))
    assert not a[1][:n].any() and a[1][n:].all()
    er = t.erase_device(present[::5]).cpu().numpy()
    assert er.all() and t.tombstones == er.size
    a, b = both(np.concatenate([present, absent[:1000]]))
    for x, y in zip(a, b):
        assert np.array_equal(np.asarray(x), np.asarray(y))
    gone = np.zeros(n, dtype=bool)
    gone[::5] = True
    assert (a[1][:n].astype(bool) == ~gone).all()


def _placement_is_valid_linearisation(t):
    """No erases happened: every live key's window-0 slots before it are occupied (it took the first
    free cell when it was inserted), and a key stored past window 0 has a full window 0."""
    from paper_2009_07914_b200.probing import mix64_array
    k, _, sl = t.for_all_device()
    k = k.cpu().numpy().view(np.uint32).astype(np.uint64)
    sl = sl.cpu().numpy().astype(np.int64)
    c = t.capacity
    occ = np.zeros(2 * c, dtype=np.int64)
    occ[sl] = 1
    occ[sl + c] = 1  # windows wrap around the end of the table
    pre = np.concatenate([[0], np.cumsum(occ)])
    h = (mix64_array(k) % np.uint64(c)).astype(np.int64)
    off = (sl - h) % c
    span = np.minimum(off, 32)  # slots of window 0 before the key (all of it when past window 0)
    return bool(((pre[h + span] - pre[h]) == span).all())


@pytest.mark.parametrize("rho", [0.9, 0.95])
def test_sorted_greedy_insert_semantics(rho):
    """The sorted-greedy region insert (csrc/staged.cu k_st_insert_sg): a fresh table filled by one
    batch keeps almost every key in window 0 (the greedy's point); later batches into the partly
    filled table, with in-batch duplicates of several multiplicities (regions holding one are handed
    to k_st_insert_q), keys already stored and sentinels: one INSERTED per new key with its value
    stored, DUPLICATE_KEY for the other copies and for stored keys, INVALID_KEY for sentinels, and
    every placement a valid sequential insert."""
    n = 1 << 21
    rng = np.random.default_rng(int(rho * 100) + 11)
    pool = rng.permutation(np.unique(rng.integers(1, (1 << 32) - 3, size=3 * n, dtype=np.uint64)))
    cap = int(np.ceil(n / rho))
    t = SingleValueHashTable(cap, layout="packed", key_bits=32, value_bits=32, group_width=8)
    t.set_locality("staged")
    model = {}

    def batch(new, old, ndup):
        dup = np.concatenate([np.repeat(new[:ndup], 2), np.repeat(new[ndup:ndup + ndup // 8], 5)])
        keys = np.concatenate([new, dup, old, np.array([(1 << 32) - 1, (1 << 32) - 2], dtype=np.uint64)])
        keys = keys[rng.permutation(keys.size)]
        vals = rng.integers(0, 1 << 32, size=keys.size, dtype=np.uint64)
        st = t.insert_device(keys, vals).cpu().numpy()
        assert (st[keys >= (1 << 32) - 2] == 3).all()
        assert (st[np.isin(keys, old)] == 1).all()
        ins = st == 0
        ks, cnt = np.unique(keys[ins], return_counts=True)
        assert (cnt == 1).all() and set(ks.tolist()) == set(new.tolist())
        assert ((st == 0) | (st == 1) | (st == 3)).all()
        model.update(zip(keys[ins].tolist(), vals[ins].tolist()))
        assert t.occupied == len(model)

    def past_window0():
        from paper_2009_07914_b200.probing import mix64_array
        k, _, sl = t.for_all_device()
        h = (mix64_array(k.cpu().numpy().view(np.uint32).astype(np.uint64)) % np.uint64(t.capacity)).astype(np.int64)
        return ((sl.cpu().numpy() - h) % t.capacity >= 32).mean()

    fresh = pool[: (3 * n) // 4]
    batch(fresh, np.zeros(0, dtype=np.uint64), 0)  # one fresh batch: empty tiles, sorted placement
    assert _placement_is_valid_linearisation(t)
    assert past_window0() < 0.001, past_window0()
    batch(pool[(3 * n) // 4: (7 * n) // 8], fresh[:50_000], 0)  # partly filled tiles, stored keys
    assert _placement_is_valid_linearisation(t)
    batch(pool[(7 * n) // 8: n], fresh[50_000:60_000], 2000)  # + in-batch duplicates
    assert _placement_is_valid_linearisation(t)
    q = np.concatenate([np.array(list(model.keys()), dtype=np.uint64), pool[n: n + 100_000]])
    v, f = t.retrieve_device(q)
    v = v.cpu().numpy().view(np.uint32).astype(np.uint64)
    f = f.cpu().numpy().astype(bool)
    assert f[: len(model)].all() and not f[len(model):].any()
    assert (v[: len(model)] == np.array(list(model.values()), dtype=np.uint64)).all()
    t.set_locality("off")  # the direct (COPS) lookups agree
    dv, df = t.retrieve_device(q)
    assert (dv.cpu().numpy().view(np.uint32).astype(np.uint64) == v).all()
    assert (df.cpu().numpy().astype(bool) == f).all()


def test_deferred_clear_semantics():
    """ch_clear of a staged-size packed table defers the memset (api.cu pending_clear): the next
    staged insert starts every region empty; any other operation -- lookups, a small (direct)
    insert, slot reads -- sees an empty table."""
    from paper_2009_07914_b200 import _lib
    rng = np.random.default_rng(21)
    pool = rng.permutation(np.unique(rng.integers(1, (1 << 32) - 3, size=1 << 24, dtype=np.uint64)))
    t = SingleValueHashTable(34_000_000, layout="packed", key_bits=32, value_bits=32, group_width=8)
    assert t.capacity * 8 >= 256 << 20
    keys = pool[: 1 << 22]
    vals = keys ^ np.uint64(0x5A5A5A5A)
    stream = torch.cuda.current_stream().cuda_stream

    def clear():
        _lib.check(_lib.lib().ch_clear(t._dt.handle, stream), "clear")

    assert t.batch_schedule(keys.size) == "staged"
    assert (t.insert_device(keys, vals).cpu().numpy() == 0).all()
    clear()  # then lookups: nothing found
    v, f = t.retrieve_device(keys[:100_000])
    assert not f.cpu().numpy().any() and t.occupied == 0
    clear()  # then a small direct insert
    small = pool[-1000:]
    assert t.batch_schedule(small.size) != "staged"
    assert (t.insert_device(small, small).cpu().numpy() == 0).all()
    v, f = t.retrieve_device(np.concatenate([small, keys[:1000]]))
    f = f.cpu().numpy()
    assert f[:1000].all() and not f[1000:].any() and t.occupied == 1000
    clear()  # then slot reads
    assert t.slots.load_key(0) == (1 << 32) - 1 and t.slots.load_key(t.capacity - 1) == (1 << 32) - 1
    clear()  # then a staged insert into the pending-clear table, twice in a row
    for _ in range(2):
        st = t.insert_device(keys, vals).cpu().numpy()
        assert (st == 0).all() and t.occupied == keys.size
        assert _placement_is_valid_linearisation(t)
        clear()
    st = t.insert_device(keys[: 1 << 21], vals[: 1 << 21]).cpu().numpy()  # staged (covers c / 16)
    assert (st == 0).all()
    v, f = t.retrieve_device(keys)
    f = f.cpu().numpy()
    assert f[: 1 << 21].all() and not f[1 << 21:].any()
    assert (v.cpu().numpy().view(np.uint32)[: 1 << 21] == vals[: 1 << 21].astype(np.uint32)).all()


@pytest.mark.parametrize("rho", [0.9, 0.97])
def test_staged_erase_matches_direct(rho):
    """Bulk erase on the staged schedule (csrc/staged.cu k_st_lookup_q<true>: region pass retiring
    by shared-memory CAS, COPS erase for the keys past window 0 or crossing the region end)
    against the direct COPS erase on a cell-for-cell copy of the same table: erased flags, the
    table afterwards (tombstones in the same cells), ops / attempts / windows / occupied /
    tombstone deltas -- then in-batch duplicate erases (exactly one copy erases) and erasing
    over existing tombstones."""
    from paper_2009_07914_b200 import _lib
    n = 1 << 20
    rng = np.random.default_rng(int(rho * 100) + 5)
    pool = rng.permutation(np.unique(rng.integers(1, (1 << 32) - 3, size=3 * n, dtype=np.uint64)))
    present, absent = pool[:n], pool[n:2 * n]

    def table():
        return SingleValueHashTable(int(n / rho), layout="packed", key_bits=32, value_bits=32, group_width=8)

    a, b = table(), table()
    a.set_locality("staged")
    a.insert_device(present, present ^ np.uint64(3))
    ks, vs = a._dt.read_slots()
    _lib.check(_lib.lib().ch_write_slots(b._dt.handle, ks.ctypes.data, vs.ctypes.data), "write slots")
    b.set_locality("off")

    def erase_both(keys):
        res = []
        for t in (a, b):
            t.reset_probe_counters()
            o0, t0 = t.occupied, t.tombstones
            e = t.erase_device(keys).cpu().numpy()
            c = t.probe_counters()
            res.append((e, (c.ops, c.attempts, c.windows_visited, t.occupied - o0, t.tombstones - t0)))
        return res

    q = rng.permutation(np.concatenate([present[::3], absent[: n // 4], np.array([0xFFFFFFFF], dtype=np.uint64)]))
    (ea, ca), (eb, cb) = erase_both(q)
    assert np.array_equal(ea, eb) and ca == cb
    assert ea.sum() == present[::3].size
    assert np.array_equal(a._dt.read_slots()[0], b._dt.read_slots()[0])
    # erasing next to tombstones, and in-batch duplicates (one copy of each key erases)
    q2 = rng.permutation(np.concatenate([present[1::3], present[1::3][:5000], present[::3][:1000]]))
    (ea, ca), (eb, cb) = erase_both(q2)
    for e in (ea, eb):
        got = {}
        for k, f in zip(q2.tolist(), e.tolist()):
            got[k] = got.get(k, 0) + f
        assert all(got[k] == 1 for k in present[1::3].tolist())
        assert all(got[k] == 0 for k in present[::3][:1000].tolist())
    assert ca[3:] == cb[3:]
    assert np.array_equal(a._dt.read_slots()[0], b._dt.read_slots()[0])
    v, f = a.retrieve_device(present)
    f = f.cpu().numpy().astype(bool)
    assert (f == (np.arange(n) % 3 == 2)).all()
