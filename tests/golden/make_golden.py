"""Generate golden vectors by running the REFERENCE package itself.

Run here (the reference is importable only in the build container):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

It imports ``coophash`` from /root/reference/pkg/src (read-only; bytecode
writing disabled) and records, for small seeded workloads, the reference's
outputs: hash / capacity / step / probe-order values, full slot-exact table
states after sequences of bulk and element operations, statuses, probe
counters, multi-value segments, bucket-list arenas and handles, and
distribution plans.  The JSON files in this directory are committed; the
GPU box never sees /root/reference.  tests/test_oracle.py pins the CPU
oracle (oracle/oracle.c) to these files and the GPU parity tests use the
same workloads.
"""
from __future__ import annotations

import json
import os
import random
import sys

sys.dont_write_bytecode = True
sys.path.insert(0, "/root/reference/pkg/src")

import coophash as ch  # noqa: E402
from coophash.bench import WorkloadSpec, gen_multiplicity, gen_unique  # noqa: E402
from coophash.probing import STEP_SEED, mix64_array  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))


def dump(name: str, obj) -> None:
    path = os.path.join(HERE, name)
    with open(path, "w") as fh:
        json.dump(obj, fh, separators=(",", ":"))
    print(f"wrote {path} ({os.path.getsize(path)} bytes)")


def status_names(sts):
    return [s.value for s in sts]


# ---------------------------------------------------------------- probing

def gen_probing():
    rng = random.Random(2009)
    keys = [0, 1, 2, 3, 0xDEADBEEF, (1 << 32) - 1, (1 << 32) - 2, (1 << 64) - 1,
            (1 << 64) - 2] + [rng.getrandbits(64) for _ in range(200)] + \
           [rng.getrandbits(32) for _ in range(200)]
    mins = [32, 33, 63, 64, 65, 100, 1000, 1024, 4096, 12345, 1_310_720, 282_564_700,
            298_261_800, 335_544_320, 167_772_160] + [rng.randrange(32, 1 << 34) for _ in range(50)]
    plans = {str(m): [ch.choose_capacity(m).p, ch.choose_capacity(m).c] for m in mins}
    ps = sorted({v[0] for v in plans.values()} | {2, 3, 5, 37, 101})
    steps = {str(p): [ch.dh_step(k, ch.CapacityPlan(p=p, c=32 * p)) for k in keys[:100]] for p in ps}
    primes = [n for n in range(0, 3000)] + [rng.randrange(1 << 40) for _ in range(200)] + \
             [2_147_483_647, (1 << 61) - 1, 18446744073709551557]
    prime_flags = [ch.is_prime(n) for n in primes]
    # probe orders / window starts for every scheme at a small plan
    plan = ch.choose_capacity(1000)
    orders = {}
    for scheme in ch.ProbingScheme:
        cfg = ch.ProbingConfig(plan=plan, scheme=scheme)
        orders[scheme.value] = {str(k): list(ch.window_starts(k, cfg)) for k in keys[:8]}
    cfg4 = ch.ProbingConfig(plan=plan, group_width=4, max_outer_attempts=3)
    cops = {str(k): [ch.cops_positions(k, cfg4, i) for i in range(0, 96, 4)] for k in keys[:8]}
    porder = {str(k): ch.probing.probe_order(k, ch.ProbingConfig(plan=plan), limit=100)
              for k in keys[:8]}
    dump("probing.json", {
        "keys": [str(k) for k in keys],
        "mix64": [str(ch.mix64(k)) for k in keys],
        "stephash": [str(ch.HashFn(STEP_SEED).value(k)) for k in keys],
        "mix64_array_first": [str(int(x)) for x in mix64_array(
            __import__("numpy").array(keys[:64], dtype="uint64"))],
        "plans": plans,
        "steps": steps,
        "primes": [str(n) for n in primes],
        "prime_flags": prime_flags,
        "window_starts": orders,
        "cops_g4": cops,
        "probe_order": porder,
        "plan_1000": [plan.p, plan.c],
    })


# ---------------------------------------------------------- single-value

def table_state(t):
    s = t.slots
    keys = [s.load_key(i) for i in range(s.capacity)]
    vals = [s.load_value(i) for i in range(s.capacity)]
    return [str(k) for k in keys], [str(v) for v in vals]


def counters(t):
    c = t.probe_counters()
    return {"ops": c.ops, "attempts": c.attempts, "windows": c.windows_visited}


def single_scenario(name, min_cap, *, layout="soa", key_bits=64, group_width=32,
                    max_outer=None, seed=0, n_keys=800, domain=None):
    rng = random.Random(seed)
    vb = 32 if layout == "packed" else 64
    t = ch.SingleValueHashTable(min_cap, layout=layout, key_bits=key_bits, value_bits=vb,
                                group_width=group_width, max_outer_attempts=max_outer)
    e, tomb = t.slots.sentinels.empty_key, t.slots.sentinels.tombstone_key
    hi = domain or min((1 << key_bits) - 3, (1 << 31))
    vmax = (1 << 32) - 1 if vb == 32 else (1 << 40)
    steps = []
    # phase 1: bulk insert with duplicates and sentinels sprinkled in
    keys = [rng.randrange(1, hi) for _ in range(n_keys)]
    keys += keys[: n_keys // 10]  # in-batch duplicates (sequential: first wins)
    keys[5] = e
    keys[7] = tomb
    vals = [rng.randrange(0, vmax) for _ in keys]
    st = t.insert_bulk(list(zip(keys, vals)))
    steps.append({"op": "insert_bulk", "keys": [str(k) for k in keys],
                  "vals": [str(v) for v in vals], "status": status_names(st)})
    # phase 2: element erases (present, absent, sentinel)
    er_keys = keys[: n_keys // 4] + [hi, e]  # hi is never drawn and is no sentinel
    er = [t.erase(k) for k in er_keys]
    steps.append({"op": "erase", "keys": [str(k) for k in er_keys], "result": er})
    # phase 3: reinsert half of the erased keys with new values + new keys
    re_keys = er_keys[: n_keys // 8] + [rng.randrange(1, hi) for _ in range(n_keys // 8)]
    re_vals = [rng.randrange(0, vmax) for _ in re_keys]
    st2 = t.insert_bulk(list(zip(re_keys, re_vals)))
    steps.append({"op": "insert_bulk", "keys": [str(k) for k in re_keys],
                  "vals": [str(v) for v in re_vals], "status": status_names(st2)})
    # phase 4: retrieve present + absent + sentinel
    q = keys[: n_keys // 2] + re_keys + [rng.randrange(1, hi) for _ in range(50)] + [e, tomb]
    got = t.retrieve_bulk(q)
    steps.append({"op": "retrieve_bulk", "keys": [str(k) for k in q],
                  "result": [None if v is None else str(v) for v in got]})
    # phase 5: per-key stats for a few keys
    probe = []
    for k in q[:40]:
        v, stats = t.retrieve_with_stats(k)
        probe.append([str(k), stats.attempts, stats.windows_visited, t.slot_of(k)])
    steps.append({"op": "stats", "probe": probe})
    ks, vs = table_state(t)
    return {"name": name, "min_capacity": min_cap, "layout": layout, "key_bits": key_bits,
            "group_width": group_width, "max_outer_attempts": max_outer,
            "p": t.config.plan.p, "capacity": t.capacity, "empty": str(e), "tomb": str(tomb),
            "steps": steps, "final_keys": ks, "final_vals": vs, "occupied": t.occupied,
            "tombstones": t.tombstones, "counters": counters(t)}


def full_scenario():
    t = ch.SingleValueHashTable(32)  # p = 2, c = 64
    st = [t.insert(k, k) for k in range(1, 66)]
    return {"name": "p2_full", "status": [s.value for s in st], "capacity": t.capacity,
            "occupied": t.occupied, "counters": counters(t)}


def gen_single():
    scen = []
    for g in (1, 2, 4, 8, 16, 32):
        scen.append(single_scenario(f"soa64_g{g}", 1000, group_width=g, seed=11 + g))
    scen.append(single_scenario("packed32_g4", 1000, layout="packed", key_bits=32,
                                group_width=4, seed=7))
    scen.append(single_scenario("packed32_g32_dense", 1200, layout="packed", key_bits=32,
                                group_width=32, seed=8, n_keys=1100, domain=5000))
    scen.append(single_scenario("aos64_g8", 3000, layout="aos", group_width=8, seed=9,
                                n_keys=2500))
    scen.append(single_scenario("soa32_maxouter2", 500, key_bits=32, group_width=16,
                                max_outer=2, seed=10, n_keys=600))
    scen.append(single_scenario("soa64_bigkeys", 2000, group_width=8, seed=12, n_keys=1500,
                                domain=(1 << 64) - 3))
    dump("single.json", {"scenarios": scen, "full": full_scenario()})


# ----------------------------------------------------------- multi-value

def gen_multi():
    scen = []
    for name, n, r, g, layout, kb, seed in [
            ("r4_g32", 3000, 4, 32, "soa", 64, 21), ("r16_g4", 3000, 16, 4, "soa", 64, 22),
            ("r1_g8_packed", 2000, 1, 8, "packed", 32, 23),
            ("r64_g1", 2500, 64, 1, "soa", 64, 24), ("r300_g16_aos", 2000, 300, 16, "aos", 64, 25)]:
        rng = random.Random(seed)
        vb = 32 if layout == "packed" else 64
        t = ch.MultiValueHashTable(int(n / 0.8), layout=layout, key_bits=kb, value_bits=vb,
                                   group_width=g)
        keys = [rng.randrange(1, max(2, n // r) + 1) for _ in range(n)]
        vals = list(range(1, n + 1))
        st = t.insert_bulk(list(zip(keys, vals)))
        queries = list(range(0, n // r + 5)) + [t.slots.sentinels.empty_key]
        counts = t.count_bulk(queries)
        offsets, flat = t.retrieve_bulk(queries)
        ks, vs = table_state(t)
        scen.append({"name": name, "min_capacity": int(n / 0.8), "layout": layout,
                     "key_bits": kb, "group_width": g, "capacity": t.capacity,
                     "keys": [str(k) for k in keys], "vals": vals, "status": status_names(st),
                     "queries": [str(q) for q in queries], "counts": counts,
                     "offsets": offsets, "flat": [str(v) for v in flat],
                     "final_keys": ks, "final_vals": vs, "occupied": t.occupied,
                     "counters": counters(t)})
    # full table: capacity 64
    t = ch.MultiValueHashTable(32)
    st = [t.insert(1, i) for i in range(64)] + [t.insert(1, 64), t.insert(2, 0)]
    dump("multi.json", {"scenarios": scen, "full_status": [s.value for s in st],
                        "prefix_sum": [ch.exclusive_prefix_sum([]),
                                       ch.exclusive_prefix_sum([5]),
                                       ch.exclusive_prefix_sum([2, 0, 3])]})


# ----------------------------------------------------------- bucket list

def gen_bucket():
    scen = []
    for name, min_keys, pool, s0, lam, n, dom, g, seed in [
            ("default_r16", 400, 12000, 1, "1.1", 4000, 250, 32, 31),
            ("doubling", 200, 6000, 1, "2", 3000, 60, 4, 32),
            ("s2_l15", 100, 100000, 2, "1.5", 20000, 49, 8, 33),
            ("exact8", 100, 4096, 8, "1.0", 512, 64, 16, 34),
            ("exhaust", 100, 300, 1, "2", 500, 20, 32, 35),
            ("l1_s1", 64, 5000, 1, "1.0", 2000, 30, 1, 36)]:
        rng = random.Random(seed)
        t = ch.BucketListHashTable(min_keys, pool, growth=ch.GrowthPolicy(s0, lam),
                                   group_width=g)
        keys = [rng.randrange(1, dom + 1) for _ in range(n)]
        vals = [rng.randrange(0, 1 << 40) for _ in range(n)]
        st = t.insert_bulk(list(zip(keys, vals)))
        queries = list(range(0, dom + 3))
        counts = t.count_bulk(queries)
        offsets, flat = t.retrieve_bulk(queries)
        chains = {str(k): t.chain_sizes(k) for k in queries[:20]}
        ks, hs = table_state(t.key_store)
        scen.append({"name": name, "min_keys": min_keys, "pool": pool, "s0": s0, "factor": lam,
                     "group_width": g, "keys": [str(k) for k in keys],
                     "vals": [str(v) for v in vals], "status": status_names(st),
                     "queries": [str(q) for q in queries], "counts": counts,
                     "offsets": offsets, "flat": [str(v) for v in flat], "chains": chains,
                     "arena": [str(v) for v in t.pool.arena[:t.pool.allocated]], "allocated": t.pool.allocated,
                     "occupied_keys": t.occupied_keys, "total_values": t.total_values,
                     "key_capacity": t.capacity, "final_keys": ks, "final_handles": hs,
                     "storage_density": t.storage_density()})
    growth = {}
    for s0, lam in [(1, "1.1"), (1, "2"), (5, "1.0"), (2, "1.5"), (3, "1.25"), (1, "1.01")]:
        p = ch.GrowthPolicy(s0, lam)
        growth[f"{s0}:{lam}"] = [p.bucket_size(i) for i in range(60)]
    bf = ch.GrowthPolicy(1, 2)
    dump("bucket.json", {"scenarios": scen, "growth": growth,
                         "buckets_for_doubling": [bf.buckets_for(c) for c in range(0, 40)],
                         "handles": [[s, c, tl, str(ch.pack_handle(s, c, tl))] for s, c, tl in
                                     [(0, 0, 0), (1, 0, 0), (2, 1, 5), (3, 3, 7),
                                      (2, (1 << 20) - 1, (1 << 42) - 1)]]})


# ----------------------------------------------------------- distribution

def gen_distributed():
    rng = random.Random(41)
    keys = [rng.getrandbits(64) for _ in range(300)] + list(range(0, 100))
    routes = {str(s): [ch.ShardRouter(s).route(k) for k in keys] for s in range(1, 9)}
    splits = {}
    for s in (1, 2, 3, 4, 8):
        plan = ch.multi_split(keys, ch.ShardRouter(s))
        splits[str(s)] = {"perm": plan.permutation, "offsets": plan.offsets}
    # distributed single-value with in-batch duplicates (first in (i mod S, i) order wins)
    pairs = [(5, 1), (6, 2), (5, 3), (5, 4), (6, 5)] + \
            [(rng.randrange(1, 3000), rng.randrange(1, 1 << 30)) for _ in range(2000)]
    dist = {}
    for s in (1, 2, 3, 4):
        with ch.DistributedTable(s, lambda _: ch.SingleValueHashTable(4096)) as dt:
            st = dt.insert_bulk(pairs)
            q = list(range(0, 3005))
            got = dt.retrieve_bulk(q)
            dist[str(s)] = {"status": status_names(st),
                            "retrieve": [None if v is None else v for v in got]}
    dump("distributed.json", {"keys": [str(k) for k in keys], "routes": routes,
                              "splits": splits, "pairs": pairs, "single": dist})


def gen_workloads():
    out = {}
    for n, kb, seed in [(1000, 32, 42), (1 << 16, 32, 10_010), (5000, 64, 12)]:
        out[f"unique_{n}_{kb}_{seed}"] = [str(k) for k in gen_unique(
            WorkloadSpec(n=n, key_bits=kb, seed=seed))[:64]]
    for n, r, seed in [(1000, 4, 77), (1 << 14, 16, 42), (1000, 1, 4)]:
        out[f"mult_{n}_{r}_{seed}"] = [str(k) for k in gen_multiplicity(
            WorkloadSpec(n=n, r=r, seed=seed))[:64]]
    dump("workloads.json", out)


def gen_kmer():
    """Canonical k-mers, window sketches and read classification of the reference's k-mer
    demo (kmer.py:63-137) on seeded random sequences with non-ACGT gaps, lower case and
    short tails."""
    from coophash import kmer as km
    rng = random.Random(63)
    alphabet = "ACGTACGTACGTACGTacgtN"

    def seq(n):
        return "".join(rng.choice(alphabet) for _ in range(n))

    seqs = [seq(n) for n in (5, 17, 40, 127, 128, 129, 300, 1000, 2500)] + ["ACGT" * 40, "N" * 50, "acgtnACGT" * 30]
    out = {"seqs": seqs, "cases": []}
    for k, window, sketch in [(16, 128, 16), (5, 20, 4), (31, 64, 8), (32, 100, 3), (1, 8, 2), (11, 11, 100)]:
        p = km.KmerParams(k=k, window=window, sketch_size=sketch)
        out["cases"].append({
            "k": k, "window": window, "sketch": sketch,
            "canonical": [[str(x) for x in km.canonical_kmers(s_, k)] for s_ in seqs[:6]],
            "sketches": [[str(x) for x in km.sketch_sequence(s_, p)] for s_ in seqs],
        })
    # an index of 6 references, classification of 8 reads (multi-value backend, 64-bit keys)
    refs = [km.ReferenceRecord(target_id=i, sequence=seq(3000 + 700 * i)) for i in range(6)]
    reads = []
    for j in range(8):
        r = refs[j % 6].sequence
        a = rng.randrange(0, len(r) - 400)
        reads.append(r[a:a + 250 + 20 * j] + seq(30))
    reads.append(seq(500))
    p = km.KmerParams()
    table = km.make_backend("oa", km.expected_sketch_volume(refs, p))
    inserted = km.build_index(refs, p, table)
    out["index"] = {"refs": [r.sequence for r in refs], "reads": reads, "inserted": inserted,
                    "volume": km.expected_sketch_volume(refs, p),
                    "classify": [[list(x) for x in km.classify(r, p, table)] for r in reads]}
    dump("kmer.json", out)


if __name__ == "__main__":
    gen_kmer()
    gen_probing()
    gen_single()
    gen_multi()
    gen_bucket()
    gen_distributed()
    gen_workloads()
