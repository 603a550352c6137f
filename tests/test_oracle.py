"""Pin the CPU oracle (oracle/oracle.c) to the reference's own outputs.

tests/golden/*.json were produced by tests/golden/make_golden.py, which ran
the reference package (coophash) itself.  Every comparison here is exact:
hash values, capacity plans, steps, statuses, probe counters, slot-exact
table states, multi-value segments (probe order), bucket arenas and chains.
CPU only.
"""
import json
import os
from fractions import Fraction

import numpy as np
import pytest

import oracle as orc

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def load(name):
    with open(os.path.join(GOLD, name)) as fh:
        return json.load(fh)


STATUS = {name: code for code, name in enumerate(orc.STATUS_NAMES)}


def ints(xs):
    return [int(x) for x in xs]


# ------------------------------------------------------------------ probing

def test_mix64_and_stephash_golden():
    g = load("probing.json")
    keys = ints(g["keys"])
    assert [orc.mix64(k) for k in keys] == ints(g["mix64"])
    assert orc.mix64(0) == 0x9CA066F1A4AB2EEA  # test_probing.py:16
    step_seed = 0x9E3779B97F4A7C15
    assert orc.mix64_array(keys, step_seed).tolist() == ints(g["stephash"])


def test_capacity_plans_and_steps_golden():
    g = load("probing.json")
    for m, (p, c) in g["plans"].items():
        assert orc.choose_p(int(m)) == p and 32 * p == c, m
    keys = ints(g["keys"])[:100]
    for p, steps in g["steps"].items():
        assert [orc.dh_step(k, int(p)) for k in keys] == steps, p
    assert [orc.is_prime(int(n)) for n in g["primes"]] == g["prime_flags"]


# ------------------------------------------------------------ single-value

@pytest.mark.parametrize("idx", range(11))
def test_single_scenarios_slot_exact(idx):
    g = load("single.json")
    sc = g["scenarios"][idx]
    e, t = int(sc["empty"]), int(sc["tomb"])
    tab = orc.OracleSingle(sc["min_capacity"], group_width=sc["group_width"], key_bits=sc["key_bits"],
                           packed=sc["layout"] == "packed", max_outer_attempts=sc["max_outer_attempts"] or 0,
                           sentinels=(e, t))
    assert tab.capacity == sc["capacity"] and tab.p == sc["p"]
    for step in sc["steps"]:
        if step["op"] == "insert_bulk":
            st = tab.insert_bulk(ints(step["keys"]), ints(step["vals"]))
            assert [orc.STATUS_NAMES[s] for s in st] == step["status"]
        elif step["op"] == "erase":
            assert [bool(x) for x in tab.erase_bulk(ints(step["keys"]))] == step["result"]
        elif step["op"] == "retrieve_bulk":
            v, f = tab.retrieve_bulk(ints(step["keys"]))
            assert [int(x) if hit else None for x, hit in zip(v, f)] == \
                [None if r is None else int(r) for r in step["result"]]
        elif step["op"] == "stats":
            for key, att, win, slot in step["probe"]:
                s1, a1, w1 = tab.find(int(key))
                assert (a1, w1) == (att, win), key
                s2, _, _ = tab.find(int(key))
                assert s2 == slot, key
    keys, vals = tab.dump()
    assert keys.tolist() == ints(sc["final_keys"])
    assert vals.tolist() == ints(sc["final_vals"])
    st = tab.stats()
    assert (st["occupied"], st["tombstones"]) == (sc["occupied"], sc["tombstones"])
    assert (st["ops"], st["attempts"], st["windows"]) == \
        (sc["counters"]["ops"], sc["counters"]["attempts"], sc["counters"]["windows"])


def test_single_full_table_p2():
    g = load("single.json")["full"]
    tab = orc.OracleSingle(32)
    st = [int(tab.insert_bulk([k], [k])[0]) for k in range(1, 66)]
    assert [orc.STATUS_NAMES[s] for s in st] == g["status"]
    assert tab.capacity == g["capacity"] == 64
    c = tab.stats()
    assert (c["occupied"], c["ops"], c["attempts"], c["windows"]) == \
        (g["occupied"], g["counters"]["ops"], g["counters"]["attempts"], g["counters"]["windows"])


# ------------------------------------------------------------- multi-value

@pytest.mark.parametrize("idx", range(5))
def test_multi_scenarios_exact(idx):
    sc = load("multi.json")["scenarios"][idx]
    tab = orc.OracleMulti(sc["min_capacity"], group_width=sc["group_width"], key_bits=sc["key_bits"],
                          packed=sc["layout"] == "packed")
    assert tab.capacity == sc["capacity"]
    st = tab.insert_bulk(ints(sc["keys"]), ints(sc["vals"]))
    assert [orc.STATUS_NAMES[s] for s in st] == sc["status"]
    q = ints(sc["queries"])
    assert tab.count_bulk(q).tolist() == sc["counts"]
    offsets, flat = tab.retrieve_bulk(q)
    assert offsets.tolist() == sc["offsets"]
    assert flat.tolist() == ints(sc["flat"])  # probe order, exactly
    keys, vals = tab.dump()
    assert keys.tolist() == ints(sc["final_keys"]) and vals.tolist() == ints(sc["final_vals"])
    c = tab.stats()
    assert (c["occupied"], c["ops"], c["attempts"], c["windows"]) == \
        (sc["occupied"], sc["counters"]["ops"], sc["counters"]["attempts"], sc["counters"]["windows"])


def test_multi_full_and_prefix_sum():
    g = load("multi.json")
    tab = orc.OracleMulti(32)
    st = [int(tab.insert_bulk([1], [i])[0]) for i in range(64)]
    st += [int(tab.insert_bulk([1], [64])[0]), int(tab.insert_bulk([2], [0])[0])]
    assert [orc.STATUS_NAMES[s] for s in st] == g["full_status"]
    assert [orc.exclusive_prefix_sum(c).tolist() for c in ([], [5], [2, 0, 3])] == g["prefix_sum"]


# -------------------------------------------------------------- bucket list

@pytest.mark.parametrize("idx", range(6))
def test_bucket_scenarios_exact(idx):
    sc = load("bucket.json")["scenarios"][idx]
    tab = orc.OracleBucket(sc["min_keys"], sc["pool"], s0=sc["s0"], factor=sc["factor"],
                           group_width=sc["group_width"])
    st = tab.insert_bulk(ints(sc["keys"]), ints(sc["vals"]))
    assert [orc.STATUS_NAMES[s] for s in st] == sc["status"]
    q = ints(sc["queries"])
    assert tab.count_bulk(q).tolist() == sc["counts"]
    offsets, flat = tab.retrieve_bulk(q)
    assert offsets.tolist() == sc["offsets"]
    assert flat.tolist() == ints(sc["flat"])  # head-first chain order, exactly
    for k, chain in sc["chains"].items():
        assert tab.chain_sizes(int(k)) == chain
    s = tab.stats()
    assert (s["occupied_keys"], s["total_values"], s["allocated"]) == \
        (sc["occupied_keys"], sc["total_values"], sc["allocated"])
    assert tab.arena()[: sc["allocated"]].tolist() == ints(sc["arena"])
    keys, handles = tab.key_store.dump()
    assert keys.tolist() == ints(sc["final_keys"]) and handles.tolist() == ints(sc["final_handles"])


def test_growth_tables_and_handles():
    g = load("bucket.json")
    for spec, sizes in g["growth"].items():
        s0, lam = spec.split(":")
        assert orc.growth_sizes(int(s0), Fraction(lam), len(sizes)).tolist() == sizes
    for s, c, t, word in g["handles"]:
        assert orc.pack_handle(s, c, t) == int(word)


# ------------------------------------------------------------ distribution

def test_routes_and_splits_golden():
    g = load("distributed.json")
    keys = ints(g["keys"])
    for s, routes in g["routes"].items():
        assert [orc.route(k, int(s)) for k in keys] == routes
    for s, plan in g["splits"].items():
        perm, offsets = orc.multi_split(keys, int(s))
        assert perm.tolist() == plan["perm"] and offsets.tolist() == plan["offsets"]


def test_distributed_single_sequential_order():
    """Shard t receives (i mod S, i)-ordered pairs (distributed.py:111-127)."""
    g = load("distributed.json")
    pairs = g["pairs"]
    for s_str, exp in g["single"].items():
        S = int(s_str)
        shards = [orc.OracleSingle(4096) for _ in range(S)]
        status = [None] * len(pairs)
        for t in range(S):
            idx = [i for src in range(S) for i in range(src, len(pairs), S)
                   if orc.route(pairs[i][0], S) == t]
            st = shards[t].insert_bulk([pairs[i][0] for i in idx], [pairs[i][1] for i in idx])
            for i, c in zip(idx, st):
                status[i] = orc.STATUS_NAMES[c]
        assert status == exp["status"]
        got = []
        for k in range(3005):
            v, f = shards[orc.route(k, S)].retrieve_bulk([k])
            got.append(int(v[0]) if f[0] else None)
        assert got == exp["retrieve"]
